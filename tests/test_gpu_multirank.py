"""The data-parallel product step on TWO ranks: two processes
share cuda:0 through a gloo group (NCCL refuses two ranks on one device; the
step code is the same for both backends: E-step graph, ONE all-reduce of the
statistics buffer, M-step graph). Each rank runs ``distributed.em_stochastic_step(s)``
on its contiguous shard of a global batch; the result must equal the
single-device step on the whole batch (chunked at the shard boundary, so the
statistics are summed in the same order) and every step must issue exactly one
collective. Also: a rank with an empty shard, and the stop at the first failing
step when only one rank sees the bad value."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

B = 256


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup(cfg, seed=0):
    import paper_2004_06231_b200 as E
    from paper_2004_06231_b200.data import config
    rg, fam, k, gen = config(cfg)
    x0 = gen(B, seed=seed)
    return E.build_model(rg, fam, k=k, seed=0, data=x0), gen


def _worker(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []
    real = dist.all_reduce

    def counting(t, *a, **k):
        calls.append((tuple(t.shape), str(t.dtype)))
        return real(t, *a, **k)

    dist.all_reduce = counting
    out = {}
    try:
        import paper_2004_06231_b200 as E
        from paper_2004_06231_b200 import distributed as D
        model, gen = _setup(cfg)
        xs = [gen(B, seed=s) for s in range(1, 4)]
        # 1) single steps (graph path)
        out["ll_single"] = [D.em_stochastic_step(model, x, 0.5, chunk=B // world) for x in xs]
        out["calls_single"] = len(calls)
        # 2) pipelined steps from pinned host u8 batches
        calls.clear()
        u8 = [torch.from_numpy(np.rint(gen(B, seed=s) * 255).astype(np.uint8)).pin_memory()
              for s in range(4, 7)]
        out["ll_steps"] = D.em_stochastic_steps(model, u8, 0.5, chunk=B // world)
        out["calls_steps"] = len(calls)
        out["params"] = model.params.flat.cpu().numpy()
        # 3) a global batch of one sample: rank 1's shard is empty
        calls.clear()
        one = gen(1, seed=9)
        out["ll_one"] = D.em_stochastic_step(model, one, 0.5)
        out["calls_one"] = len(calls)
        out["params_one"] = model.params.flat.cpu().numpy()
        # 4) only rank 1 sees a non-finite value in the second of three steps
        calls.clear()
        bad = [gen(B, seed=s).astype(np.float32) for s in range(10, 13)]
        bad[1][B - 3, 17] = np.nan  # row B-3 lies in rank 1's shard
        try:
            D.em_stochastic_steps(model, [torch.from_numpy(b) for b in bad], 0.5,
                                  chunk=B // world)
            out["err"] = None
        except E.UnsupportedValueError as e:
            out["err"] = str(e)
        out["calls_bad"] = len(calls)
        out["params_bad"] = model.params.flat.cpu().numpy()
        q.put((rank, out))
        dist.barrier()
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, {"exception": repr(e)}))
        raise
    finally:
        dist.all_reduce = real
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_two_rank_product_step_equals_single_device(cfg):
    import torch.multiprocessing as mp

    import paper_2004_06231_b200 as E
    from paper_2004_06231_b200 import trainer

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    for r in range(world):
        assert "exception" not in res[r], res[r]

    # single device, whole batch, chunked at the shard boundary
    model, gen = _setup(cfg)
    xs = [gen(B, seed=s) for s in range(1, 4)]
    ll_single = [trainer.em_stochastic_step(model, x, 0.5, chunk=B // world) for x in xs]
    u8 = [torch.from_numpy(np.rint(gen(B, seed=s) * 255).astype(np.uint8)).pin_memory()
          for s in range(4, 7)]
    ll_steps = trainer.em_stochastic_steps(model, u8, 0.5, chunk=B // world)
    params = model.params.flat.cpu().numpy()
    ll_one = trainer.em_stochastic_step(model, gen(1, seed=9), 0.5)
    params_one = model.params.flat.cpu().numpy()

    for r in range(world):
        got = res[r]
        # one collective per EM update: the fp64 statistics all-reduce
        assert got["calls_single"] == 3 and got["calls_steps"] == 3 and got["calls_one"] == 1
        np.testing.assert_allclose(got["ll_single"], ll_single, rtol=1e-12)
        np.testing.assert_allclose(got["ll_steps"], ll_steps, rtol=1e-12)
        np.testing.assert_allclose(got["params"], params, rtol=1e-11, atol=1e-15)
        np.testing.assert_allclose(got["ll_one"], ll_one, rtol=1e-12)
        np.testing.assert_allclose(got["params_one"], params_one, rtol=1e-11, atol=1e-15)
        # the failing step raises on BOTH ranks with the parameters left as after
        # the first (good) step: 3 stats all-reduces + 1 MIN of the error logs
        assert got["err"] == "variable 17: non-finite value"
        assert got["calls_bad"] == 4
    # ranks stay bitwise identical
    assert np.array_equal(res[0]["params"], res[1]["params"])
    assert np.array_equal(res[0]["params_bad"], res[1]["params_bad"])
    bad = [gen(B, seed=s).astype(np.float32) for s in range(10, 13)]
    trainer.em_stochastic_step(model, bad[0], 0.5, chunk=B // world)
    np.testing.assert_allclose(res[0]["params_bad"], model.params.flat.cpu().numpy(),
                               rtol=1e-11, atol=1e-15)
    print(f"{cfg}: 2-rank params bitwise equal to single device: "
          f"{np.array_equal(res[0]['params'], params)}")
