"""Parity AT THE BENCHMARKED CONFIGURATION.

``bench.py`` times C3 (SVHN-shaped 32x32x3 PD EiNet, K=40) at 16384 samples
per step in one chunk. These tests run exactly that step -- B = 16384 with
chunk 16384 and with chunk 4096 -- against the fp64 oracle, sharded over host
processes (forward + back-pass per shard, statistics merged by summation,
engine.py:228-236, then the oracle M-step): per-sample log-likelihoods, the
complete BackwardStats and the parameters after two EM steps (lambda 0.5).
Same for the CelebA-shaped C4 (49152 variables) at B = 1024.

Tolerances (BASELINE.json north star):
* per-sample LL: |d| <= 1e-4 * max(|LL|, 1);
* statistics: rtol 1e-4 + atol 1e-6 * B;
* W after each step: rtol 1e-4 + atol 1e-9 (the 1e-12 projection floor);
* leaf means: rtol 1e-4 + atol 1e-6; leaf VARIANCES sigma^2 = phi_1 - phi_0^2
  (derived in fp64 from the fp64 master parameters) RELATIVELY: rtol
  VAR_RTOL, no absolute floor (image-mode variances
  go down to 1e-6, so an absolute floor on phi would hide them).
Every comparison prints its worst relative error.
"""

import multiprocessing as mp
import os

import numpy as np
import pytest

import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import engine, trainer
from paper_2004_06231_b200.data import config

from oracle import einet_oracle as O

from tests.helpers import device_values

pytestmark = pytest.mark.gpu

LL_RTOL = 1e-4
P_RTOL = 1e-4
VAR_RTOL = 1e-4

_G = {}


def _init(circuit, fam, x):
    _G["m"] = (circuit, fam, x)


def _shard(args):
    params, lo, hi, sub = args
    circuit, fam, x = _G["m"]
    st, roots = None, []
    for a in range(lo, hi, sub):
        tr = O.forward(circuit, params, fam, x[a:min(hi, a + sub)])
        roots.append(tr.root[:, 0])
        part = O.backward(circuit, params, fam, tr)
        st = part if st is None else st.merge(part)
    return st, np.concatenate(roots)


def oracle_estep(circuit, fam, x, params, sub):
    """Sharded fp64 E-step: (per-sample LL, merged OracleStats)."""
    procs = max(1, min(len(os.sched_getaffinity(0)), 64))
    n = len(x)
    bounds = np.linspace(0, n, procs + 1).astype(int)
    spans = [(int(bounds[i]), int(bounds[i + 1])) for i in range(procs)
             if bounds[i + 1] > bounds[i]]
    with mp.get_context("fork").Pool(len(spans), initializer=_init,
                                     initargs=(circuit, fam, x)) as pool:
        parts = pool.map(_shard, [(params, lo, hi, sub) for lo, hi in spans])
    st = parts[0][0]
    for p, _ in parts[1:]:
        st.merge(p)
    return np.concatenate([r for _, r in parts]), st


def worst_rel(got, want, atol=0.0):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want) / (np.abs(want) + atol + 1e-300)))


def check(name, got, want, rtol, atol, report):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    err = np.abs(got - want) - (rtol * np.abs(want) + atol)
    report.append(f"{name}: worst rel {worst_rel(got, want):.3e}, "
                  f"worst tol use {np.max(np.abs(got - want) / (rtol * np.abs(want) + atol)):.3f}")
    assert err.max() <= 0, report[-1]


def check_phi(name, got, want, report):
    """Leaf means with atol 1e-6; variances relative only."""
    check(name + ".mu", got[..., 0], want[..., 0], P_RTOL, 1e-6, report)
    vg = got[..., 1] - got[..., 0] ** 2
    vw = want[..., 1] - want[..., 0] ** 2
    check(name + ".var", vg, vw, VAR_RTOL, 0.0, report)


def _setup(cfg, n, seed, init_n=None):
    rg, fam, k, gen = config(cfg)
    circuit = E.compile_graph(rg, k)
    # the oracle sees what the device evaluates: image data on the 1/255 grid
    # at u / 255 exactly (helpers.device_values)
    x = device_values(gen(n, seed=seed).astype(np.float32))
    data = x if init_n is None else x[:init_n]
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=data)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    op = O.OracleParams({i: f32(w) for i, w in ein.items()},
                        {i: f32(w) for i, w in mix.items()}, f32(phi))
    return circuit, fam, x, op


_CACHE = {}


def _oracle_run(cfg, n, seed, sub):
    """Oracle LLs + stats at init, then the parameters after steps 1 and 2."""
    key = (cfg, n, seed)
    if key not in _CACHE:
        circuit, fam, x, op = _setup(cfg, n, seed)
        fd = fam.to_dict()
        ll0, st0 = oracle_estep(circuit, fd, x, op, sub)
        p1 = O.apply_update(circuit, op, fd, st0, 0.5)
        ll1, st1 = oracle_estep(circuit, fd, x, p1, sub)
        p2 = O.apply_update(circuit, p1, fd, st1, 0.5)
        _CACHE[key] = dict(circuit=circuit, fam=fam, x=x, op=op, ll0=ll0, st0=st0, p1=p1,
                           p2=p2, mean=[st0.ll_sum / n, st1.ll_sum / n])
    return _CACHE[key]


def _run(cfg, n, seed, chunk, sub):
    R = _oracle_run(cfg, n, seed, sub)
    circuit, fam, x, op = R["circuit"], R["fam"], R["x"], R["op"]
    report = [f"{cfg} B={n} chunk={chunk}"]
    p = engine.Parameters.from_numpy(circuit, fam, op.einsum, op.mixing, op.phi)
    # per-sample LL and the complete statistics of the first E-step
    xs = x.astype(np.float32)
    stats = None
    lls = []
    for lo in range(0, n, chunk):
        tr = E.forward(circuit, p, fam, xs[lo:lo + chunk])
        lls.append(tr.log_likelihood)
        part = E.backward(circuit, p, fam, tr)
        if stats is None:
            stats = {"einsum": part.einsum, "mixing": part.mixing, "acc_p": part.acc_p,
                     "acc_pt": part.acc_pt}
        else:
            for i in stats["einsum"]:
                stats["einsum"][i] = stats["einsum"][i] + part.einsum[i]
            for i in stats["mixing"]:
                stats["mixing"][i] = stats["mixing"][i] + part.mixing[i]
            stats["acc_p"] = stats["acc_p"] + part.acc_p
            stats["acc_pt"] = stats["acc_pt"] + part.acc_pt
    ll = np.concatenate(lls)
    bound = LL_RTOL * np.maximum(np.abs(R["ll0"]), 1.0)
    err = np.abs(ll - R["ll0"])
    report.append(f"LL: worst rel {worst_rel(ll, R['ll0']):.3e}, worst tol use "
                  f"{(err / bound).max():.3f}")
    assert (err <= bound).all(), report[-1]
    st0 = R["st0"]
    atol = 1e-6 * n
    for i in st0.einsum:
        check(f"stats.einsum[{i}]", stats["einsum"][i], st0.einsum[i], P_RTOL, atol, report)
    for i in st0.mixing:
        check(f"stats.mixing[{i}]", stats["mixing"][i], st0.mixing[i], P_RTOL, atol, report)
    check("stats.acc_p", stats["acc_p"], st0.acc_p, P_RTOL, atol, report)
    check("stats.acc_pt", stats["acc_pt"], st0.acc_pt, P_RTOL, atol, report)
    # Two EM steps through the public step at this chunk size. Each step
    # starts from the ORACLE's parameters before that step (fp64 masters
    # loaded as they are), so the check measures one update's error. Feeding
    # the GPU's own step-1 result into step 2 measures EM's amplification of
    # a 1e-5 difference instead: with 768 (C3) or 12288 (C4) variables per
    # leaf scope a relative change of 1e-5 in a mean moves a leaf
    # log-density by O(1) nat, so posteriors (and the next targets) move by
    # O(1e-4) in the oracle itself. That compounded drift is printed below.
    chained = E.EinetModel(circuit, engine.Parameters.from_numpy(
        circuit, fam, op.einsum, op.mixing, op.phi), fam)
    starts = (op, R["p1"])
    for s, want in enumerate((R["p1"], R["p2"])):
        src = starts[s]
        ps = engine.Parameters.from_numpy(circuit, fam, src.einsum, src.mixing, src.phi)
        model = E.EinetModel(circuit, ps, fam)
        mean = trainer.em_stochastic_step(model, xs, 0.5, chunk=chunk)
        wm = R["mean"][s]
        report.append(f"step {s + 1} mean LL rel {abs(mean - wm) / abs(wm):.3e}")
        assert abs(mean - wm) <= LL_RTOL * max(abs(wm), 1.0)
        e2, m2, phi2 = ps.to_numpy()
        for i in e2:
            check(f"step{s + 1}.W[{i}]", e2[i], want.einsum[i], P_RTOL, 1e-9, report)
        for i in m2:
            check(f"step{s + 1}.mix[{i}]", m2[i], want.mixing[i], P_RTOL, 1e-9, report)
        check_phi(f"step{s + 1}.phi", phi2, want.phi, report)
        trainer.em_stochastic_step(chained, xs, 0.5, chunk=chunk)
    e2, _, phi2 = chained.params.to_numpy()
    drift = max(worst_rel(e2[i], R["p2"].einsum[i], 1e-9) for i in e2)
    report.append(f"compounded (GPU step 1 -> GPU step 2) W drift vs oracle: {drift:.3e}")
    print("\n".join(report))


@pytest.mark.parametrize("chunk", [16384, 4096])
def test_c3_benchmarked_step_vs_oracle(chunk):
    _run("C3", 16384, 21, chunk, sub=128)


def test_c4_b1024_vs_oracle():
    _run("C4", 1024, 22, 1024, sub=16)
