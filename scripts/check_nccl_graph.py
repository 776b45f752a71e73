"""One-rank NCCL group through the graph path (E-step graph, all-reduce, M-step
graph) vs the single-device graph: identical parameters. Diagnostics."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import trainer
from paper_2004_06231_b200.structures import StructureConfig

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
rng = np.random.default_rng(0)
x = rng.normal(0.5, 0.2, (256, 16))
ms = [E.build_model(E.random_binary_tree(16, StructureConfig(depth=2, replicas=2, seed=1)),
                    E.GaussianFamily(), k=8, seed=2, data=x) for _ in range(2)]
xd = torch.from_numpy(x.astype(np.float32)).cuda()
for step in range(3):
    a = trainer.em_stochastic_step(ms[0], xd, 0.5, chunk=128, process_group=dist.group.WORLD)
    b = trainer.em_stochastic_step(ms[1], xd, 0.5, chunk=128)
    print(step, a, b, torch.equal(ms[0].params.flat, ms[1].params.flat))
print("graphs:", [len(k) for k in ms[0]._graphs.values()])
dist.destroy_process_group()
