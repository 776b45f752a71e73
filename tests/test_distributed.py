"""Multi-process (gloo, world size 2, CPU) checks of the data-parallel EM
host logic: contiguous shards (including empty ones), the
packed statistics layout, the merge semantics of one all-reduce(sum) with the
replicated M-step (oracle statistics), and the cross-rank error protocol of
``trainer`` (error words cross ranks in a MIN all-reduce only when the summed
failure flag says some rank failed). The product step on two ranks runs in
``tests/test_gpu_multirank.py``."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import _native, trainer
from paper_2004_06231_b200 import distributed as D
from paper_2004_06231_b200.compiler import compile_graph
from paper_2004_06231_b200.engine import init_parameters_host
from paper_2004_06231_b200.expfam import GaussianFamily
from paper_2004_06231_b200.structures import StructureConfig, lift_channels, poon_domingos

from oracle import einet_oracle as O

from .helpers import pack_stats, unpack_stats


def _setup():
    rg = lift_channels(poon_domingos(4, 4, StructureConfig(deltas=(2,), axes="both")), 3)
    fam = GaussianFamily(var_max=1e-2)
    circuit = compile_graph(rg, 4)
    rng = np.random.default_rng(0)
    x = np.round(np.clip(rng.normal(0.5, 0.2, (37, rg.d_vars)), 0, 1) * 255) / 255
    ein, mix, phi = init_parameters_host(circuit, fam, seed=0, data=x)
    return circuit, fam, x, O.OracleParams(ein, mix, phi)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    circuit, fam, x, p = _setup()
    lo, hi = D.shard_range(len(x), rank, world)
    tr = O.forward(circuit, p, fam.to_dict(), x[lo:hi])
    st = O.backward(circuit, p, fam.to_dict(), tr)
    flat = torch.from_numpy(pack_stats(circuit, fam, st.einsum, st.mixing, st.acc_pt, st.acc_p,
                                         st.ll_sum, st.n_samples))
    dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    q.put((rank, flat.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_covers_batch():
    for n in (0, 1, 7, 37, 4096):
        for world in (1, 2, 3, 8):
            spans = [D.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    assert D.shard_range(1, 1, 2) == (1, 1)  # n < world: an empty shard
    with pytest.raises(ValueError):
        D.shard_range(4, 2, 2)
    x = np.arange(10)[:, None]
    assert np.array_equal(np.concatenate([D.local_shard(x, r, 3) for r in range(3)]), x)


def test_pack_unpack_round_trip():
    circuit, fam, x, p = _setup()
    tr = O.forward(circuit, p, fam.to_dict(), x)
    st = O.backward(circuit, p, fam.to_dict(), tr)
    flat = pack_stats(circuit, fam, st.einsum, st.mixing, st.acc_pt, st.acc_p, st.ll_sum,
                        st.n_samples)
    ein, mix, acc_pt, acc_p, ll, n = unpack_stats(circuit, fam, flat)
    for i in st.einsum:
        assert np.array_equal(ein[i], st.einsum[i])
    for i in st.mixing:
        assert np.array_equal(mix[i], st.mixing[i])
    assert np.array_equal(acc_pt, st.acc_pt)
    assert np.array_equal(acc_p, st.acc_p)
    assert ll == st.ll_sum and n == st.n_samples


def test_two_rank_allreduce_equals_full_batch_em():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    # every rank holds the identical merged buffer
    assert np.array_equal(results[0], results[1])
    circuit, fam, x, p = _setup()
    tr = O.forward(circuit, p, fam.to_dict(), x)
    full = O.backward(circuit, p, fam.to_dict(), tr)
    ein, mix, acc_pt, acc_p, ll, n = unpack_stats(circuit, fam, results[0])
    merged = O.OracleStats(ein, mix, acc_p, acc_pt, int(n), ll)
    for i in full.einsum:
        np.testing.assert_allclose(ein[i], full.einsum[i], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(acc_pt, full.acc_pt, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(acc_p, full.acc_p, rtol=1e-12, atol=1e-15)
    assert n == len(x)
    # the replicated M-step on the merged statistics equals the full-batch step
    want_ll, want = O.em_step(circuit, p, fam.to_dict(), x, 0.5)
    got = O.apply_update(circuit, p, fam.to_dict(), merged, 0.5)
    assert abs(ll / n - want_ll) <= 1e-12 * abs(want_ll)
    for i in want.einsum:
        np.testing.assert_allclose(got.einsum[i], want.einsum[i], rtol=1e-10, atol=1e-15)
    np.testing.assert_allclose(got.phi, want.phi, rtol=1e-10, atol=1e-15)


NONE = _native.STATUS_NONE


def _protocol_worker(rank, world, port, q):
    """Each rank holds its own device-style logs of 3 pipelined steps; rank 1
    failed in step 1 (variable 5), rank 0 in step 2 (variable 2). The summed
    failure flag set word 3 on both ranks from step 1 on (sticky). Both ranks
    must raise step 1's error (variable 5) after ONE extra collective; with no
    failure no collective is issued at all."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []
    real = dist.all_reduce

    def counting(t, *a, **k):
        calls.append(tuple(t.shape))
        return real(t, *a, **k)

    dist.all_reduce = counting
    try:
        model = type("M", (), {"family": E.GaussianFamily()})()
        ll = torch.tensor([[-10.0, 4.0], [-12.0, 4.0], [-9.0, 4.0]], dtype=torch.float64)
        ok = torch.full((3, 4), NONE, dtype=torch.int32)
        out = {"ok": trainer._finish_steps(model, ll, ok, dist.group.WORLD),
               "ok_calls": list(calls)}
        bad = torch.full((3, 4), NONE, dtype=torch.int32)
        bad[1:, 3] = 0
        if rank == 1:
            bad[1:, 0] = 5
        else:
            bad[2:, 0] = 2
        try:
            trainer._finish_steps(model, ll, bad, dist.group.WORLD)
            out["err"] = None
        except E.UnsupportedValueError as e:
            out["err"] = str(e)
        out["bad_calls"] = calls[len(out["ok_calls"]):]
        q.put((rank, out))
        dist.barrier()
    finally:
        dist.all_reduce = real
        dist.destroy_process_group()


def test_two_rank_error_protocol():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_protocol_worker, args=(r, world, port, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for r in range(world):
        got = results[r]
        assert got["ok"] == [-2.5, -3.0, -2.25]
        assert got["ok_calls"] == []          # no failure: no collective beyond the stats
        assert got["bad_calls"] == [(3, 4)]   # one MIN all-reduce of the step logs
        assert got["err"] == "variable 5: non-finite value"
