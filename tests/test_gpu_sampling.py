"""Batched GPU sampling (csrc/sample.cu) vs the oracle and the reference.

Parity: the device draws with a Philox4x32-10 stream keyed by (seed, sample,
decision site); ``oracle.einet_oracle.sample_philox`` restates the reference
descent (engine.py:339-388) with the same uniforms, so unconditional samples
must agree draw for draw (discrete values exactly, Gaussian values to 1e-10
relative: the device's log/cos/sqrt differ from numpy's by a few ulp).
Conditional sampling weights the branches by the evidence posterior of a
forward pass whose per-slab offsets the device keeps in fp32, so a branch
whose cumulative boundary lies within ~1e-7 of the uniform may flip: at
least 99% of the samples must agree. Against the reference's own sampler
(numpy generators) parity is statistical: moments within 5 standard errors
of tests/golden/sampling.npz (the max over up to ~1200 mean and second-moment
entries per case).
"""

import time

import numpy as np
import pytest

import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import engine
from paper_2004_06231_b200.data import config

from tests.helpers import Case, moment_z, oracle_samples, sampling_cases

pytestmark = pytest.mark.gpu

G_TOL = 1e-10


def device_params(case):
    p = case.params("init")
    return engine.Parameters.from_numpy(case.circuit, case.family, p.einsum, p.mixing, p.phi)


def run(case, evidence, n, seed):
    p = device_params(case)
    if evidence:
        return E.conditional_sample(case.circuit, p, case.family, case.x[0], evidence, n, seed)
    return E.sample(case.circuit, p, case.family, n, seed)


def rows_equal(a, b, gaussian):
    if gaussian:
        return np.all(np.abs(a - b) <= G_TOL * np.maximum(np.abs(b), 1.0), axis=1)
    return np.all(a == b, axis=1)


def test_unconditional_matches_oracle_draw_for_draw():
    g, cases = sampling_cases()
    for i, case, ev in cases:
        if ev:
            continue
        got = run(case, ev, 1000, seed=5)
        want = oracle_samples(case, ev, 1000, seed=5)
        assert got.shape == want.shape
        assert not np.isnan(got).any()
        ok = rows_equal(got, want, case.fam_doc["family"] == "gaussian")
        assert ok.all(), (case.name, np.nonzero(~ok)[0][:5])


def test_conditional_matches_oracle():
    g, cases = sampling_cases()
    for i, case, ev in cases:
        if not ev:
            continue
        got = run(case, ev, 2000, seed=9)
        want = oracle_samples(case, ev, 2000, seed=9)
        assert (got[:, ev] == case.x[0][ev]).all()
        ok = rows_equal(got, want, case.fam_doc["family"] == "gaussian")
        assert ok.mean() >= 0.99, (case.name, ok.mean())


def test_samples_match_reference_moments():
    g, cases = sampling_cases()
    for i, case, ev in cases:
        s = run(case, ev, int(g["n"]), seed=21)
        z = moment_z(s, g, f"case{i}")
        assert z < 5.0, (case.name, ev, z)


def test_sampling_is_deterministic_and_independent_of_n():
    case = Case("rat_categorical4")
    a = run(case, [], 300, seed=3)
    b = run(case, [], 300, seed=3)
    c = run(case, [], 120, seed=3)
    d = run(case, [], 300, seed=4)
    assert np.array_equal(a, b)
    assert np.array_equal(a[:120], c)
    assert not np.array_equal(a, d)


def test_empty_evidence_is_unconditional():
    case = Case("rat_gaussian")
    p = device_params(case)
    a = E.sample(case.circuit, p, case.family, 64, 2)
    b = E.conditional_sample(case.circuit, p, case.family, case.x[0], [], 64, 2)
    assert np.array_equal(a, b)


def test_sampling_edge_cases():
    case = Case("rat_gaussian")
    p = device_params(case)
    assert E.sample(case.circuit, p, case.family, 0, 0).shape == (0, case.circuit.d_vars)
    kr = Case("rat_gaussian_kroot3")
    with pytest.raises(engine.EngineError):
        E.sample(kr.circuit, device_params(kr), kr.family, 4, 0)


def test_model_api_samples_c3():
    """C3 (SVHN-shaped lifted PD, K=40): a batch of 4096 unconditional samples
    and an image completion (left half observed) through the model API."""
    rg, fam, k, gen = config("C3")
    m = E.build_model(rg, fam, k=k, seed=0, data=gen(256))
    t = time.perf_counter()
    s = m.sample(4096, seed=1)
    dt = time.perf_counter() - t
    assert s.shape == (4096, 3072) and np.isfinite(s).all()
    print(f"C3 sample 4096: {dt * 1e3:.1f} ms")
    x_e = np.random.default_rng(0).random(3072)
    ev = [v for v in range(3072) if (v // 3) % 32 < 16]
    c = m.conditional_sample(x_e, ev, 512, seed=2)
    assert np.isfinite(c).all()
    assert (c[:, ev] == x_e[ev]).all()
    # a sample's value depends on (seed, index) only
    assert np.array_equal(m.sample(16, seed=1), s[:16])
