"""W-statistics unit timeline (EINET_WS_TRACE=1) on the C5 shape:
python scripts/ws_trace_c5.py K B (one eager EM step; the trace goes to stderr)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ.setdefault("EINET_WS_TRACE", "1")
from paper_2004_06231_b200 import engine, trainer  # noqa: E402
from paper_2004_06231_b200.compiler import compile_graph  # noqa: E402
from paper_2004_06231_b200.builders import make_family  # noqa: E402
from paper_2004_06231_b200.model import EinetModel  # noqa: E402
from paper_2004_06231_b200.structures import StructureConfig, random_binary_tree  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 128
b = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
fam = make_family("gaussian", image_mode=False)
rg = random_binary_tree(16, StructureConfig(depth=2, replicas=32, seed=0))
circuit = compile_graph(rg, k)
x = np.random.default_rng(0).normal(0.0, 1.0, size=(b, 16))
ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=x[:256])
model = EinetModel(circuit, engine.Parameters.from_numpy(circuit, fam, ein, mix, phi), fam)
xd = engine.as_device_batch(x)
trainer.em_stochastic_step(model, xd, 0.0)
torch.cuda.synchronize()
