"""Per-kernel-class device time of one forward + backward (EM statistics) on a
benchmark config: python scripts/class_times.py [CONFIG] [BATCH] (default C3
16384). CUDA-event classes of the library profiler (einet_profile_*)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2004_06231_b200 as E  # noqa: E402
from paper_2004_06231_b200 import _native, engine  # noqa: E402
from paper_2004_06231_b200.data import config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
rg, fam, k, gen = config(cfg)
c = E.compile_graph(rg, k)
x = torch.from_numpy(gen(B, seed=3).astype(np.float32)).cuda()
ein, mix, phi = engine.init_parameters_host(c, fam, seed=0, data=gen(512, seed=1))
p = engine.Parameters.from_numpy(c, fam, ein, mix, phi)
for _ in range(3):
    tr = E.forward(c, p, fam, x)
    E.backward(c, p, fam, tr)
torch.cuda.synchronize()
_native.profile_enable(True)
for _ in range(5):
    tr = E.forward(c, p, fam, x)
    E.backward(c, p, fam, tr)
torch.cuda.synchronize()
prof = _native.profile_read()
_native.profile_enable(False)
print(json.dumps({k: round(v[0] / 5 * 1e3, 1) for k, v in prof.items()}))
