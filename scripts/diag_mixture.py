"""Where does a train_many step spend its time? (diagnostic)"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_06231_b200 import engine, trainer  # noqa: E402
from paper_2004_06231_b200.compiler import compile_graph  # noqa: E402
from paper_2004_06231_b200.data import config  # noqa: E402
from paper_2004_06231_b200.model import EinetModel  # noqa: E402

rg, fam, k, gen = config("C3")
circuit = compile_graph(rg, k)
d = gen(5810, seed=1)
ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=d[:512])
m = EinetModel(circuit, engine.Parameters.from_numpy(circuit, fam, ein, mix, phi), fam)
xd = engine.as_device_batch(d)
idx = torch.randperm(5810, device="cuda")
xb = torch.empty((500, xd.shape[1]), dtype=torch.float32, device="cuda")
logs = torch.empty((240, 4), dtype=torch.int32, device="cuda")
sums = torch.empty(240, dtype=torch.float64, device="cuda")
N = 100


def timed(name, fn):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(N):
        fn(i)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:28s} host {1e6 * (t1 - t) / N:8.1f} us/step  total {1e6 * (t2 - t) / N:8.1f} us/step",
          flush=True)


def step(i):
    trainer._enqueue_step(m, xb, 0.5, 1e-12, 4096)


timed("graph step only", step)
timed("+ index_select", lambda i: (torch.index_select(xd, 0, idx[:500], out=xb), step(i)))
timed("+ status copy", lambda i: (step(i), logs[i].copy_(m.step_buffers(500)[3])))
timed("+ flat sum", lambda i: (step(i), sums.__setitem__(i, m.params.flat.sum())))
out = torch.empty(5810, dtype=torch.float64, device="cuda")
timed("epoch LL pass (per comp)", lambda i: trainer._enqueue_ll(m, xd, 500, out))
timed("compute_for", lambda i: m.params.compute_for(m.step_buffers(500)[0]))
timed("step_buffers", lambda i: m.step_buffers(500))

models = [m]
for c in range(1, 4):
    e2, m2, p2 = engine.init_parameters_host(circuit, fam, seed=c, data=d[:512])
    models.append(EinetModel(circuit, engine.Parameters.from_numpy(circuit, fam, e2, m2, p2), fam))
streams = [torch.cuda.Stream() for _ in models]


def inter(i, use_streams):
    for c, mm in enumerate(models):
        if use_streams:
            with torch.cuda.stream(streams[c]):
                trainer._enqueue_step(mm, xb, 0.5, 1e-12, 4096)
        else:
            trainer._enqueue_step(mm, xb, 0.5, 1e-12, 4096)


timed("4 models, one stream (x4)", lambda i: inter(i, False))
timed("4 models, 4 streams (x4)", lambda i: inter(i, True))
cfg = trainer.TrainerConfig(epochs=1, batch_size=500, step_size=0.5, seed=0)
for nm in (1, 4):
    trainer.train_many(models[:nm], [d] * nm, cfg)
    torch.cuda.synchronize()
    t = time.perf_counter()
    trainer.train_many(models[:nm], [d] * nm, cfg)
    torch.cuda.synchronize()
    print(f"train_many {nm} models x 12 steps: {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
