"""Host submission cost vs device time of the pipelined EM steps (diagnostic):
python scripts/host_overhead.py CONFIG BATCH"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2004_06231_b200 as E  # noqa: E402
from paper_2004_06231_b200 import engine, trainer  # noqa: E402
from paper_2004_06231_b200.data import config  # noqa: E402

cfg, B = sys.argv[1], int(sys.argv[2])
rg, fam, k, gen = config(cfg)
c = E.compile_graph(rg, k)
x = engine.as_device_batch(gen(B, seed=3))
ein, mix, phi = engine.init_parameters_host(c, fam, seed=0, data=gen(512, seed=1))
model = E.EinetModel(c, engine.Parameters.from_numpy(c, fam, ein, mix, phi), fam)
trainer.em_stochastic_steps(model, [x] * 5, 0.5, chunk=B)
torch.cuda.synchronize()
n = 200
marks = {}
orig = trainer._finish_steps


def finish(*a, **kw):
    marks["submitted"] = time.perf_counter()
    return orig(*a, **kw)


trainer._finish_steps = finish
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
trainer.em_stochastic_steps(model, [x] * n, 0.5, chunk=B)
t1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
print(f"{cfg} B={B}: device {e0.elapsed_time(e1) / n * 1e3:.1f} us/step, host submission "
      f"{(marks['submitted'] - t0) / n * 1e6:.1f} us/step")
