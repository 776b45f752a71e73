"""The NCCL paths on one device: a world-size-1 NCCL group runs the E-step
graph, the all-reduces of the statistics and error words, and the M-step
graph -- the multi-GPU step -- and must equal the single-device step bitwise
(sum over one rank is the identity). Covers ``em_stochastic_step`` and the
pipelined ``em_stochastic_steps`` (no host wait between steps), including the
stop at the first failing step."""

import os
import socket

import numpy as np
import pytest
import torch

import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import trainer
from paper_2004_06231_b200.data import config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def group():
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


def _models(cfg, n=2, seed=0):
    rg, fam, k, gen = config(cfg)
    x = gen(256, seed=seed)
    return [E.build_model(rg, fam, k=k, seed=0, data=x) for _ in range(n)], gen


def test_nccl_step_equals_single_device(group):
    ms, gen = _models("C2")
    xs = [gen(256, seed=s) for s in range(3)]
    for x in xs:
        a = trainer.em_stochastic_step(ms[0], x, 0.5, chunk=128, process_group=group)
        b = trainer.em_stochastic_step(ms[1], x, 0.5, chunk=128)
        assert a == b
    assert torch.equal(ms[0].params.flat, ms[1].params.flat)


def test_nccl_pipelined_steps_equal_single_device(group):
    ms, gen = _models("C2")
    xs = [np.rint(gen(256, seed=s) * 255).astype(np.uint8) for s in range(4)]
    hosts = [torch.from_numpy(x).pin_memory() for x in xs]
    a = trainer.em_stochastic_steps(ms[0], hosts, 0.5, chunk=128, process_group=group)
    b = trainer.em_stochastic_steps(ms[1], hosts, 0.5, chunk=128)
    assert a == b
    assert torch.equal(ms[0].params.flat, ms[1].params.flat)


def test_nccl_pipelined_steps_stop_at_first_failure(group):
    ms, gen = _models("C1")
    xs = [gen(64, seed=s).astype(np.float32) for s in range(3)]
    xs[1][3, 2] = 7.0
    with pytest.raises(E.UnsupportedValueError, match="variable 2"):
        trainer.em_stochastic_steps(ms[0], [torch.from_numpy(x).pin_memory() for x in xs], 0.5,
                                    process_group=group)
    trainer.em_stochastic_step(ms[1], xs[0], 0.5)
    assert torch.equal(ms[0].params.flat, ms[1].params.flat)
