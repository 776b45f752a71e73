import sys, os, json, numpy as np, torch
sys.path.insert(0, ".")
import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import engine, _native
from paper_2004_06231_b200.data import config
rg, fam, k, gen = config("C3")
c = E.compile_graph(rg, k)
x = torch.from_numpy(gen(16384, seed=3).astype(np.float32)).cuda()
ein, mix, phi = engine.init_parameters_host(c, fam, seed=0, data=gen(512, seed=1))
p = engine.Parameters.from_numpy(c, fam, ein, mix, phi)
for _ in range(3):
    tr = E.forward(c, p, fam, x); E.backward(c, p, fam, tr)
torch.cuda.synchronize()
_native.profile_enable(True)
for _ in range(5):
    tr = E.forward(c, p, fam, x); E.backward(c, p, fam, tr)
torch.cuda.synchronize()
prof = _native.profile_read(); _native.profile_enable(False)
print(json.dumps({k: round(v[0] / 5 * 1e3, 1) for k, v in prof.items()}))
