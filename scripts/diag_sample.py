import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import sampling, engine, _native
from paper_2004_06231_b200.data import config
rg, fam, k, gen = config("C3")
x = gen(4096, seed=3)
m = E.build_model(rg, fam, k=k, seed=0, data=x)
n = 16384
m.sample(n, 1)
torch.cuda.synchronize()
# device-only timing: replicate _run without the .cpu()
eng = engine.get_engine(m.circuit, fam, 1)
lib = eng._lib
out = torch.empty((n, m.circuit.d_vars), dtype=torch.float64, device="cuda")
scratch = torch.empty(int(lib.einet_sample_scratch_bytes(eng.handle, n)), dtype=torch.uint8, device="cuda")
status = eng.new_status()
p = engine._ptr
def dev():
    lib.einet_sample(eng.handle, p(m.params.flat), None, 0, None, None, n, 1, p(scratch), p(out), p(status), engine._stream())
for f, name in [(dev, "device kernels")]:
    f(); torch.cuda.synchronize()
    t = time.perf_counter(); f(); torch.cuda.synchronize(); print(name, (time.perf_counter()-t)*1e3, "ms")
t = time.perf_counter(); h = out.cpu(); print("D2H pageable", (time.perf_counter()-t)*1e3, "ms")
hp = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
t = time.perf_counter(); hp.copy_(out); torch.cuda.synchronize(); print("D2H pinned (preallocated)", (time.perf_counter()-t)*1e3, "ms")
t = time.perf_counter(); hp2 = torch.empty(out.shape, dtype=out.dtype, pin_memory=True); print("pinned alloc", (time.perf_counter()-t)*1e3, "ms")
t = time.perf_counter(); a = m.sample(n, 1); print("m.sample total", (time.perf_counter()-t)*1e3, "ms")
