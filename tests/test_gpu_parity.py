"""CUDA engine vs the reference (golden vectors) and the CPU oracle.

Tolerances (north star, BASELINE.json): per-sample log-likelihoods within
1e-4 relative (|d| <= 1e-4 * max(|LL|, 1)), backward statistics
rtol 1e-4 + atol 1e-6 * B, EM-updated parameters rtol 1e-4 (W with atol 1e-9
for the 1e-12 floor; leaf phi with atol PHI_ATOL = 1e-6 on unit-scale data,
because the 3xTF32 leaf statistics carry ~2^-21 relative product error, which
a mean close to 0 relative to the data spread turns into an absolute error).
The device computes the leaf terms in fp64, contractions in 3xTF32/fp32, with
fp64 statistics, fp64 master parameters and an fp64 M-step.
"""

import numpy as np
import pytest
import torch

import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import _native, engine, trainer
from paper_2004_06231_b200.data import config
from paper_2004_06231_b200.structures import StructureConfig, random_binary_tree

from oracle import einet_oracle as O
from tests.helpers import CASES, Case, close, summarize

pytestmark = pytest.mark.gpu

LL_RTOL = 1e-4
P_RTOL = 1e-4
PHI_ATOL = 1e-6


def device_params(case, prefix="init"):
    p = case.params(prefix)
    return engine.Parameters.from_numpy(case.circuit, case.family, p.einsum, p.mixing, p.phi)


def ll_close(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), fin)
    err = np.abs(got[fin] - want[fin])
    bound = LL_RTOL * np.maximum(np.abs(want[fin]), 1.0)
    assert (err <= bound).all(), (err / bound).max()


def stats_close(case, st, B):
    atol = 1e-6 * B
    for i in case.einsum_layers():
        want = case.z[f"stats_einsum_{i}"]
        got = st.einsum[i]
        if not case.full:
            got = summarize(got)
        close(got, want, P_RTOL, atol)
    for i in case.mixing_layers():
        close(st.mixing[i], case.z[f"stats_mixing_{i}"], P_RTOL, atol)
    for key, got in (("stats_acc_p", st.acc_p), ("stats_acc_pt", st.acc_pt)):
        if not case.full:
            got = summarize(got)
        close(got, case.z[key], P_RTOL, atol)


@pytest.mark.parametrize("name", CASES)
def test_forward_matches_reference(name):
    case = Case(name)
    if case.full:
        p = device_params(case)
    else:
        ein, mix, phi = engine.init_parameters_host(case.circuit, case.family, 0, case.x)
        f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
        p = engine.Parameters.from_numpy(case.circuit, case.family,
                                         {i: f32(w) for i, w in ein.items()},
                                         {i: f32(w) for i, w in mix.items()}, f32(phi))
    tr = engine.forward(case.circuit, p, case.family, case.x, marg_mask=case.mask)
    ll_close(tr.root, case.z["root"])
    st = engine.backward(case.circuit, p, case.family, tr)
    stats_close(case, st, len(case.x))


FULL_BATCH_SKIP = ("rat_gaussian_masked", "rat_gaussian_kroot3")


@pytest.mark.parametrize("name", [c for c in CASES if c not in FULL_BATCH_SKIP])
def test_em_steps_match_reference(name):
    case = Case(name)
    if case.full:
        p = device_params(case)
    else:
        ein, mix, phi = engine.init_parameters_host(case.circuit, case.family, 0, case.x)
        f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
        p = engine.Parameters.from_numpy(case.circuit, case.family,
                                         {i: f32(w) for i, w in ein.items()},
                                         {i: f32(w) for i, w in mix.items()}, f32(phi))
    model = E.EinetModel(case.circuit, p, case.family)
    for s in range(case.steps()):
        ll = trainer.em_stochastic_step(model, case.x, case.lam, chunk=10 if
                                        name == "rat_categorical4" else 4096)
        want_ll = case.z["step_mean_ll"][s]
        assert abs(ll - want_ll) <= LL_RTOL * max(abs(want_ll), 1.0)
        ein, mix, phi = p.to_numpy()
        for i, w in ein.items():
            want = case.z[f"step{s + 1}_einsum_{i}"]
            close(w if case.full else summarize(w), want, P_RTOL, 1e-9)
        for i, w in mix.items():
            close(w, case.z[f"step{s + 1}_mixing_{i}"], P_RTOL, 1e-9)
        close(phi if case.full else summarize(phi), case.z[f"step{s + 1}_phi"], P_RTOL, PHI_ATOL)


def _random_model(seed, family_kind="gaussian"):
    rng = np.random.default_rng(seed)
    d = int(rng.integers(2, 9))
    depth = int(rng.integers(1, min(3, int(np.floor(np.log2(d)))) + 1))
    rg = random_binary_tree(d, StructureConfig(depth=depth, replicas=int(rng.integers(1, 4)),
                                               seed=int(rng.integers(1 << 30))))
    k = int(rng.integers(1, 6))
    if family_kind == "gaussian":
        fam = E.GaussianFamily()
        data = rng.normal(size=(16, d))
    else:
        fam = E.CategoricalFamily(int(rng.integers(2, 5)))
        data = rng.integers(0, fam.num_states, size=(16, d)).astype(float)
    data = data.astype(np.float32).astype(np.float64)
    circuit = E.compile_graph(rg, k)
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=seed, data=data)
    return circuit, fam, data, (ein, mix, phi)


@pytest.mark.parametrize("seed", range(12))
def test_random_fixtures_vs_oracle(seed):
    circuit, fam, data, (ein, mix, phi) = _random_model(seed, ["gaussian", "categorical"][seed % 2])
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    op = O.OracleParams({i: f32(w) for i, w in ein.items()}, {i: f32(w) for i, w in mix.items()},
                        f32(phi))
    p = engine.Parameters.from_numpy(circuit, fam, op.einsum, op.mixing, op.phi)
    tr = engine.forward(circuit, p, fam, data)
    otr = O.forward(circuit, op, fam.to_dict(), data)
    ll_close(tr.log_likelihood, otr.log_likelihood)
    st = engine.backward(circuit, p, fam, tr)
    ost = O.backward(circuit, op, fam.to_dict(), otr)
    for i in ost.einsum:
        close(st.einsum[i], ost.einsum[i], P_RTOL, 1e-6 * len(data))
    close(st.acc_p, ost.acc_p, P_RTOL, 1e-6 * len(data))
    close(st.acc_pt, ost.acc_pt, P_RTOL, 1e-6 * len(data))


def _random_tc_model(seed):
    """Random structures on the tensor-core / DMMA paths: K a multiple of 8,
    RAT or PD graphs, all three families, ragged batch sizes."""
    rng = np.random.default_rng(1000 + seed)
    k = int(rng.choice([8, 16, 24, 32, 40, 48, 56, 64]))
    if seed % 3 == 2:
        h, w = int(rng.integers(2, 5)), int(rng.integers(2, 5))
        rg = E.poon_domingos(h, w, StructureConfig(deltas=(1,), axes="both"))
    else:
        d = int(rng.integers(4, 33))
        depth = min(int(rng.integers(1, 4)), int(np.floor(np.log2(d))))
        rg = random_binary_tree(d, StructureConfig(depth=depth,
                                                   replicas=int(rng.integers(1, 4)),
                                                   seed=int(rng.integers(1 << 30))))
    d = rg.d_vars
    b = int(rng.integers(33, 300))
    kind = ["gaussian", "categorical", "binomial"][seed % 3 if seed % 3 != 2 else 0]
    if kind == "gaussian":
        fam = E.GaussianFamily()
        data = rng.normal(0.3, 0.5, size=(b, d))
    elif kind == "categorical":
        fam = E.CategoricalFamily(int(rng.integers(2, 5)))
        data = rng.integers(0, fam.num_states, size=(b, d)).astype(float)
    else:
        fam = E.BinomialFamily(int(rng.integers(1, 9)))
        data = rng.integers(0, fam.n_trials + 1, size=(b, d)).astype(float)
    data = data.astype(np.float32).astype(np.float64)
    circuit = E.compile_graph(rg, k)
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=seed, data=data)
    mask = rng.random(d) < 0.25 if seed % 4 == 1 else None
    return circuit, fam, data, (ein, mix, phi), mask


@pytest.mark.parametrize("seed", range(16))
def test_random_tensor_core_paths_vs_oracle(seed):
    circuit, fam, data, (ein, mix, phi), mask = _random_tc_model(seed)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    op = O.OracleParams({i: f32(w) for i, w in ein.items()}, {i: f32(w) for i, w in mix.items()},
                        f32(phi))
    p = engine.Parameters.from_numpy(circuit, fam, op.einsum, op.mixing, op.phi)
    tr = engine.forward(circuit, p, fam, data, marg_mask=mask)
    otr = O.forward(circuit, op, fam.to_dict(), data, mask)
    ll_close(tr.log_likelihood, otr.log_likelihood)
    st = engine.backward(circuit, p, fam, tr)
    ost = O.backward(circuit, op, fam.to_dict(), otr)
    for i in ost.einsum:
        close(st.einsum[i], ost.einsum[i], P_RTOL, 1e-6 * len(data))
    close(st.acc_p, ost.acc_p, P_RTOL, 1e-6 * len(data))
    close(st.acc_pt, ost.acc_pt, P_RTOL, 1e-6 * len(data))
    if mask is None:
        want_ll, op = O.em_step(circuit, op, fam.to_dict(), data, 0.5)
        ll = trainer.em_stochastic_step(E.EinetModel(circuit, p, fam), data, 0.5)
        assert abs(ll - want_ll) <= LL_RTOL * max(abs(want_ll), 1.0)
        e2, m2, phi2 = p.to_numpy()
        for i in e2:
            close(e2[i], op.einsum[i], P_RTOL, 1e-9)
        close(phi2, op.phi, P_RTOL, PHI_ATOL)


def test_c3_full_batch_vs_oracle():
    """The headline configuration at B=64 through the whole EM step."""
    rg, fam, k, gen = config("C3")
    circuit = E.compile_graph(rg, k)
    x = gen(64, seed=5).astype(np.float32).astype(np.float64)
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=x)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    op = O.OracleParams({i: f32(w) for i, w in ein.items()}, {i: f32(w) for i, w in mix.items()},
                        f32(phi))
    p = engine.Parameters.from_numpy(circuit, fam, op.einsum, op.mixing, op.phi)
    model = E.EinetModel(circuit, p, fam)
    for step in range(2):
        want_ll, op = O.em_step(circuit, op, fam.to_dict(), x, 0.5)
        ll = trainer.em_stochastic_step(model, x, 0.5)
        assert abs(ll - want_ll) <= LL_RTOL * abs(want_ll)
        e2, m2, phi2 = p.to_numpy()
        for i in e2:
            close(e2[i], op.einsum[i], P_RTOL, 1e-9)
        close(phi2, op.phi, P_RTOL, PHI_ATOL)


def test_c4_celeba_shape_vs_oracle():
    """BASELINE.json configs[3]: the CelebA-shaped 128x128x3 PD EiNet (delta 32
    vertical, K=40, 49152 variables in 4 leaf regions of 12288) through
    forward, back-pass statistics and two EM steps at B=8."""
    rg, fam, k, gen = config("C4")
    circuit = E.compile_graph(rg, k)
    x = gen(8, seed=6).astype(np.float32).astype(np.float64)
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=gen(64, seed=7))
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    op = O.OracleParams({i: f32(w) for i, w in ein.items()}, {i: f32(w) for i, w in mix.items()},
                        f32(phi))
    p = engine.Parameters.from_numpy(circuit, fam, op.einsum, op.mixing, op.phi)
    tr = O.forward(circuit, op, fam.to_dict(), x)
    got = E.forward(circuit, p, fam, x)
    ll_close(got.log_likelihood, tr.root[:, 0])
    st = O.backward(circuit, op, fam.to_dict(), tr)
    gs = E.backward(circuit, p, fam, got)
    for i in st.einsum:
        close(gs.einsum[i], st.einsum[i], P_RTOL, 1e-6 * 8)
    close(gs.acc_pt, st.acc_pt, P_RTOL, 1e-6 * 8)
    model = E.EinetModel(circuit, p, fam)
    for step in range(2):
        want_ll, op = O.em_step(circuit, op, fam.to_dict(), x, 0.5)
        ll = trainer.em_stochastic_step(model, x, 0.5)
        assert abs(ll - want_ll) <= LL_RTOL * abs(want_ll)
        e2, m2, phi2 = p.to_numpy()
        for i in e2:
            close(e2[i], op.einsum[i], P_RTOL, 1e-9)
        close(phi2, op.phi, P_RTOL, PHI_ATOL)


@pytest.mark.parametrize("k", [72, 96, 128])
def test_large_k_paths_vs_oracle(k):
    """K > 64 (BASELINE.json configs[4] sweeps K up to 128): K = 96 and 128 run
    the tile-stationary tcgen05 contraction (contract_big.cu) and the tcgen05
    W statistics, K = 72 the CUDA-core kernels: forward and one EM step vs
    oracle."""
    rg = E.random_binary_tree(12, StructureConfig(depth=2, replicas=2, seed=4))
    x = np.random.default_rng(k).normal(0.4, 0.3, (48, 12)).astype(np.float32).astype(np.float64)
    fam = E.GaussianFamily()
    circuit = E.compile_graph(rg, k)
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=1, data=x)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    op = O.OracleParams({i: f32(w) for i, w in ein.items()}, {i: f32(w) for i, w in mix.items()},
                        f32(phi))
    p = engine.Parameters.from_numpy(circuit, fam, op.einsum, op.mixing, op.phi)
    ll_close(E.forward(circuit, p, fam, x).log_likelihood,
             O.forward(circuit, op, fam.to_dict(), x).root[:, 0])
    want_ll, op = O.em_step(circuit, op, fam.to_dict(), x, 0.5)
    ll = trainer.em_stochastic_step(E.EinetModel(circuit, p, fam), x, 0.5)
    assert abs(ll - want_ll) <= LL_RTOL * abs(want_ll)
    e2, m2, phi2 = p.to_numpy()
    for i in e2:
        close(e2[i], op.einsum[i], P_RTOL, 1e-9)
    close(phi2, op.phi, P_RTOL, PHI_ATOL)


# ---------------------------------------------------------------------------
# reference properties (test_trainer.py, test_engine.py, test_acceptance.py)
# ---------------------------------------------------------------------------

def _gauss_model(seed=0, d=4, k=3, replicas=2, data=None):
    rg = E.random_binary_tree(d, StructureConfig(depth=2, replicas=replicas, seed=seed))
    return E.build_model(rg, E.GaussianFamily(), k=k, seed=seed + 1, data=data)


def test_lambda_zero_is_bitwise_noop():
    data = np.random.default_rng(1).normal(size=(50, 4))
    m = _gauss_model(1, data=data)
    before = m.params.flat.clone()
    trainer.em_stochastic_step(m, data, lam=0.0)
    assert torch.equal(before, m.params.flat)


def test_lambda_one_equals_full_step_bitwise():
    data = np.random.default_rng(2).normal(size=(80, 4))
    a, b = _gauss_model(2, data=data), _gauss_model(2, data=data)
    trainer.em_full_step(a, data)
    trainer.em_stochastic_step(b, data, lam=1.0)
    assert torch.equal(a.params.flat, b.params.flat)


def test_training_is_deterministic():
    data = np.random.default_rng(5).normal(size=(120, 4))
    cfg = trainer.TrainerConfig(mode="stochastic", step_size=0.5, batch_size=40, epochs=3,
                                seed=11)
    a, b = _gauss_model(5, data=data), _gauss_model(5, data=data)
    ma, mb = trainer.train(a, data, cfg), trainer.train(b, data, cfg)
    assert [m.train_ll for m in ma] == [m.train_ll for m in mb]
    assert torch.equal(a.params.flat, b.params.flat)


def test_full_em_monotone():
    rng = np.random.default_rng(3)
    data = np.concatenate([rng.normal(-2, 0.5, (150, 4)), rng.normal(2, 0.5, (150, 4))])
    m = _gauss_model(3, data=data)
    lls = [trainer.em_full_step(m, data) for _ in range(30)]
    lls.append(m.mean_log_likelihood(data))
    assert np.all(np.diff(lls) >= -1e-4)


def test_single_gaussian_one_step():
    rng = np.random.default_rng(0)
    data = rng.normal(2.0, 1.5, size=(200, 4))
    rg = E.random_binary_tree(4, StructureConfig(depth=2, replicas=1, seed=0))
    m = E.build_model(rg, E.GaussianFamily(), k=1, seed=1, data=data)
    trainer.em_full_step(m, data)
    phi = m.params.phi
    mu = phi[:, 0, 0, 0]
    var = phi[:, 0, 0, 1] - mu ** 2
    x32 = data.astype(np.float32).astype(np.float64)
    assert np.allclose(mu, x32.mean(axis=0), atol=1e-6)
    assert np.allclose(var, x32.var(axis=0), rtol=1e-5)


def test_chunked_equals_unchunked():
    data = np.random.default_rng(7).normal(size=(300, 4))
    a, b = _gauss_model(7, data=data), _gauss_model(7, data=data)
    la = trainer.em_stochastic_step(a, data, 0.5, chunk=4096)
    lb = trainer.em_stochastic_step(b, data, 0.5, chunk=64)
    # fp32 partial sums restart per chunk; the fp64 merge itself is exact
    assert abs(la - lb) <= 1e-7 * abs(la)
    assert torch.allclose(a.params.flat, b.params.flat, rtol=1e-5, atol=1e-9)


def test_all_marginalised_is_zero():
    data = np.random.default_rng(8).normal(size=(6, 4))
    m = _gauss_model(8, data=data)
    ll = m.forward(data, marg_mask=np.ones(4, dtype=bool)).log_likelihood
    assert np.max(np.abs(ll)) < 1e-6


def test_categorical_normalises():
    rg = E.random_binary_tree(6, StructureConfig(depth=2, replicas=2, seed=4))
    fam = E.CategoricalFamily(2)
    m = E.build_model(rg, fam, k=3, seed=4)
    grid = np.array(np.meshgrid(*[[0, 1]] * 6)).reshape(6, -1).T.astype(float)
    ll = m.log_likelihood(grid)
    assert abs(np.exp(ll).sum() - 1.0) < 1e-5


def test_root_responsibility_mass_is_batch():
    data = np.random.default_rng(9).normal(size=(33, 4))
    m = _gauss_model(9, data=data)
    tr = m.forward(data)
    st = E.backward(m.circuit, m.params, m.family, tr)
    top = max(st.einsum)
    assert abs(st.einsum[top].sum() - 33) < 1e-4
    assert st.n_samples == 33


def test_unsupported_values_raise():
    m = _gauss_model(10, data=np.zeros((4, 4)))
    x = np.zeros((3, 4))
    x[1, 2] = np.nan
    with pytest.raises(E.UnsupportedValueError, match="variable 2"):
        m.forward(x)
    before = m.params.flat.clone()
    with pytest.raises(E.UnsupportedValueError):
        trainer.em_stochastic_step(m, x, 0.5)
    assert torch.equal(before, m.params.flat)
    rg = E.random_binary_tree(3, StructureConfig(depth=1, replicas=2, seed=0))
    mc = E.build_model(rg, E.CategoricalFamily(3), k=2, seed=1)
    with pytest.raises(E.UnsupportedValueError, match="outside"):
        mc.forward(np.array([[0.0, 3.0, 1.0]]))


def test_unsupported_values_raise_dmma_path():
    """K % 8 == 0 Gaussian leaves take the FP64 tensor-core forward, which has
    no per-value check on unmasked data: the non-finite row flag must still
    raise for the lowest offending variable, and the EM step must not update."""
    rg = E.random_binary_tree(16, StructureConfig(depth=2, replicas=2, seed=3))
    m = E.build_model(rg, E.GaussianFamily(), k=8, seed=2, data=np.zeros((4, 16)))
    x = np.zeros((40, 16))
    x[33, 11] = np.inf
    x[7, 5] = np.nan
    with pytest.raises(E.UnsupportedValueError, match="variable 5"):
        m.forward(x)
    before = m.params.flat.clone()
    with pytest.raises(E.UnsupportedValueError, match="variable 5"):
        trainer.em_stochastic_step(m, x, 0.5)
    assert torch.equal(before, m.params.flat)
    x[7, 5] = 0.0
    with pytest.raises(E.UnsupportedValueError, match="variable 11"):
        trainer.em_stochastic_step(m, x, 0.5)
    x[33, 11] = 0.0
    trainer.em_stochastic_step(m, x, 0.5)


def test_pipelined_steps_equal_sequential_steps():
    """trainer.em_stochastic_steps (copy of batch i+1 overlapping step i) is the
    same computation as em_stochastic_step per batch: bitwise equal results."""
    rng = np.random.default_rng(4)
    batches = [torch.from_numpy(rng.normal(0.5, 0.2, (96, 16)).astype(np.float32)).pin_memory()
               for _ in range(3)]
    ms = []
    for _ in range(2):
        rg = E.random_binary_tree(16, StructureConfig(depth=2, replicas=2, seed=3))
        ms.append(E.build_model(rg, E.GaussianFamily(), k=8, seed=2,
                                data=batches[0].numpy().astype(np.float64)))
    lls_a = trainer.em_stochastic_steps(ms[0], batches, 0.5, chunk=64)
    lls_b = [trainer.em_stochastic_step(ms[1], b, 0.5, chunk=64) for b in batches]
    assert lls_a == lls_b
    assert torch.equal(ms[0].params.flat, ms[1].params.flat)


def test_device_resident_pipelined_steps_equal_sequential_steps():
    """em_stochastic_steps on device-resident fp32 and u8 batches (no copies,
    no host wait) equals em_stochastic_step per batch bitwise."""
    rg, fam, k, gen = config("C2")
    xs = [gen(256, seed=s) for s in range(3)]
    for kind in ("f32", "u8"):
        if kind == "f32":
            dev = [torch.from_numpy(x.astype(np.float32)).cuda() for x in xs]
        else:
            dev = [torch.from_numpy(np.rint(x * 255).astype(np.uint8)).cuda() for x in xs]
        ma = E.build_model(rg, fam, k=k, seed=0, data=xs[0])
        mb = E.build_model(rg, fam, k=k, seed=0, data=xs[0])
        la = trainer.em_stochastic_steps(ma, dev, 0.5, chunk=128)
        lb = [trainer.em_stochastic_step(mb, b, 0.5, chunk=128) for b in dev]
        assert la == lb
        assert torch.equal(ma.params.flat, mb.params.flat)


def test_pipelined_steps_stop_at_the_first_failing_step():
    """A pipelined sequence whose third batch leaves the support raises the
    reference exception (lowest bad variable of that batch) and leaves the
    parameters exactly as after the first two steps."""
    rg, fam, k, gen = config("C1")
    good = [gen(64, seed=s).astype(np.float32) for s in range(4)]
    bad = good[2].copy()
    bad[7, 9] = 3.0
    bad[20, 4] = 2.0
    later = good[3].copy()
    later[1, 1] = 5.0  # a later failure with a lower index must not win
    seq = [good[0], good[1], bad, later]
    ma = E.build_model(rg, fam, k=k, seed=0, data=good[0])
    mb = E.build_model(rg, fam, k=k, seed=0, data=good[0])
    with pytest.raises(E.UnsupportedValueError, match="variable 4"):
        trainer.em_stochastic_steps(ma, [torch.from_numpy(b).pin_memory() for b in seq], 0.5)
    for b in seq[:2]:
        trainer.em_stochastic_step(mb, b, 0.5)
    assert torch.equal(ma.params.flat, mb.params.flat)


def test_shape_mismatch_raises():
    m = _gauss_model(11, data=np.zeros((4, 4)))
    with pytest.raises(E.EngineError):
        m.forward(np.zeros((2, 5)))


def test_log_einsum_exp_device_known_answers():
    out = E.log_einsum_exp(np.zeros((1, 1)), np.zeros((1, 1)), np.ones((1, 1, 1, 1)))
    assert abs(out[0, 0]) < 1e-15
    w = np.full((1, 2, 2, 2), 0.25)
    half = np.log(0.5) * np.ones((1, 2))
    assert np.allclose(E.log_einsum_exp(half, half, w), np.log(0.25), atol=1e-12)
    out = E.log_einsum_exp(np.array([[-np.inf, -np.inf]]), np.array([[0.0, 0.0]]),
                           np.full((1, 1, 2, 2), 0.25))
    assert np.isneginf(out).all()
    left, right = np.array([[-1000.0, -1001.0]]), np.array([[-1000.0, -1000.0]])
    want = O.log_einsum_exp(left, right, w)
    assert np.allclose(E.log_einsum_exp(left, right, w), want, atol=1e-10)


def test_ef_log_prob_matches_oracle():
    rng = np.random.default_rng(12)
    fam = E.GaussianFamily()
    phi = fam.init_phi((5, 3, 2), rng)
    x = rng.normal(size=(4, 5)).astype(np.float32).astype(np.float64)
    mask = np.array([False, True, False, False, True])
    e = E.ef_log_prob(fam, phi, x, marg_mask=mask)
    assert np.all(e[:, 1] == 0.0) and np.all(e[:, 4] == 0.0)
    for d in (0, 2, 3):
        want = O.log_density(fam.to_dict(), phi[d], x[:, d])
        assert np.allclose(e[:, d], want, rtol=1e-12)


def test_launch_counter_moves():
    before = _native.launch_count()
    data = np.random.default_rng(13).normal(size=(8, 4))
    _gauss_model(13, data=data).forward(data)
    assert _native.launch_count() > before


def test_u8_batches_decode_like_the_reference_normalisation():
    """EIND1 u8 payloads (modelio.py:145-166): x = float64(v) / 255 (or raw
    with normalize=False); the device decode equals fp32 staging of that
    array bit for bit, including odd lengths and unaligned slices."""
    rng = np.random.default_rng(0)
    for n in (1, 15, 16, 17, 4099, 1 << 20):
        v = rng.integers(0, 256, n).astype(np.uint8)
        dev = torch.from_numpy(v).cuda()
        got = engine.decode_u8(dev).cpu().numpy()
        assert np.array_equal(got, (v.astype(np.float64) / 255.0).astype(np.float32))
        raw = engine.decode_u8(dev, normalize=False).cpu().numpy()
        assert np.array_equal(raw, v.astype(np.float32))
    big = torch.from_numpy(rng.integers(0, 256, 5000).astype(np.uint8)).cuda()
    got = engine.decode_u8(big[3:4003]).cpu().numpy()
    assert np.array_equal(got, (big[3:4003].cpu().numpy() / 255.0).astype(np.float32))


def test_u8_em_steps_equal_float_steps():
    """A u8 host batch through em_stochastic_step / em_stochastic_steps gives
    bitwise the same parameters and LLs as its float64 normalisation."""
    rg, fam, k, gen = config("C2")
    x = gen(512, seed=3)
    xu = np.rint(x * 255.0).astype(np.uint8)
    assert np.array_equal(xu / 255.0, x)
    circuit = E.compile_graph(rg, k)
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=x)
    ma = E.EinetModel(circuit, engine.Parameters.from_numpy(circuit, fam, ein, mix, phi), fam)
    mb = E.EinetModel(circuit, engine.Parameters.from_numpy(circuit, fam, ein, mix, phi), fam)
    la = [trainer.em_stochastic_step(ma, x, 0.5, chunk=256)]
    lb = [trainer.em_stochastic_step(mb, torch.from_numpy(xu).pin_memory(), 0.5, chunk=256)]
    la += trainer.em_stochastic_steps(ma, [x, x[::-1].copy()], 0.5, chunk=256)
    lb += trainer.em_stochastic_steps(mb, [xu, xu[::-1].copy()], 0.5, chunk=256)
    assert la == lb
    assert torch.equal(ma.params.flat, mb.params.flat)


def _twin_models(cfg, x):
    rg, fam, k, _ = config(cfg)
    circuit = E.compile_graph(rg, k)
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=x)
    return [E.EinetModel(circuit, engine.Parameters.from_numpy(circuit, fam, ein, mix, phi), fam)
            for _ in range(2)]


@pytest.mark.parametrize("kind", ["image", "counts", "off_grid", "mixed"])
def test_f64_numpy_em_steps_equal_fp32_tensor_steps(kind):
    """float64 NumPy batches (the reference caller's type, trainer.py:104) are
    packed on the host (einet_pack_f64: bytes on the u8 grid, else fp32) and
    pipelined; parameters and LLs equal those of the same batches handed over
    as pinned fp32 tensors, bit for bit."""
    cfg = "C1" if kind == "counts" else "C2"
    rg, fam, k, gen = config(cfg)
    xs = [gen(300, seed=s) for s in (3, 4, 5)]
    if kind == "counts":
        xs = [np.random.default_rng(s).integers(0, 2, x.shape).astype(np.float64) * 1.0
              for s, x in enumerate(xs)]
    if kind == "off_grid":
        xs = [x + 1e-3 for x in xs]
    if kind == "mixed":
        xs[1] = xs[1] + 1e-3
    ma, mb = _twin_models(cfg, xs[0])
    la = [trainer.em_stochastic_step(ma, xs[0], 0.5, chunk=256)]
    lb = [trainer.em_stochastic_step(mb, torch.from_numpy(xs[0].astype(np.float32)).pin_memory(),
                                     0.5, chunk=256)]
    la += trainer.em_stochastic_steps(ma, xs + xs[::-1], 0.5, chunk=256)
    lb += trainer.em_stochastic_steps(
        mb, [torch.from_numpy(x.astype(np.float32)).pin_memory() for x in xs + xs[::-1]], 0.5,
        chunk=256)
    assert la == lb
    assert torch.equal(ma.params.flat, mb.params.flat)


def test_f64_numpy_raw_count_grid():
    """Counts above 1 (categorical states) pack as raw bytes (divisor 1)."""
    rg, fam, k, gen = config("C1")
    from paper_2004_06231_b200 import builders
    fam = builders.make_family("categorical", num_states=4)
    circuit = E.compile_graph(rg, k)
    x = np.random.default_rng(9).integers(0, 4, (200, circuit.d_vars)).astype(np.float64)
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=x)
    ms = [E.EinetModel(circuit, engine.Parameters.from_numpy(circuit, fam, ein, mix, phi), fam)
          for _ in range(2)]
    la = trainer.em_stochastic_steps(ms[0], [x, x[::-1].copy()], 0.5, chunk=128)
    lb = trainer.em_stochastic_steps(ms[1], [torch.from_numpy(x.astype(np.float32)),
                                             torch.from_numpy(x[::-1].astype(np.float32))],
                                     0.5, chunk=128)
    assert la == lb
    assert torch.equal(ms[0].params.flat, ms[1].params.flat)


def test_f64_numpy_bad_value_raises_like_fp32():
    """A NaN in a float64 batch goes the fp32 way and raises the reference's
    exception at that step, parameters as after the steps before it."""
    rg, fam, k, gen = config("C2")
    xs = [gen(128, seed=s) for s in (1, 2, 3)]
    xs[1] = xs[1].copy()
    xs[1][5, 7] = np.nan
    ma, mb = _twin_models("C2", xs[0])
    errs = []
    for m, batches in ((ma, xs), (mb, [torch.from_numpy(x.astype(np.float32)) for x in xs])):
        with pytest.raises(Exception) as ei:
            trainer.em_stochastic_steps(m, batches, 0.5, chunk=128)
        errs.append((type(ei.value), str(ei.value)))
    assert errs[0] == errs[1]
    assert torch.equal(ma.params.flat, mb.params.flat)


COND_CASES = [
    ("rat_gaussian", [1, 2], [0, 3, 5]),
    ("rat_categorical4", [0], [1, 2, 6]),
    ("rat_binomial", [2, 3, 4], []),
    ("pd_lift_gaussian_image", list(range(0, 48, 5)), list(range(1, 48, 5)))]


@pytest.mark.parametrize("name,query,evidence", COND_CASES)
def test_conditional_log_density_matches_oracle(name, query, evidence):
    """log p(x_q | x_e) (engine.py:198-215) = two marginalised forwards."""
    case = Case(name)
    p = device_params(case)
    got = E.conditional_log_density(case.circuit, p, case.family, case.x, query, evidence)
    d = case.circuit.d_vars
    num = np.array([i not in query and i not in evidence for i in range(d)])
    den = np.array([i not in evidence for i in range(d)])
    op = case.params()
    want = (O.forward(case.circuit, op, case.fam_doc, case.x, num).root[:, 0] -
            O.forward(case.circuit, op, case.fam_doc, case.x, den).root[:, 0])
    ll_close(got, want)
    with pytest.raises(ValueError):
        E.conditional_log_density(case.circuit, p, case.family, case.x, [0], [0])


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_reprepared_compute_equals_fused_mstep(cfg):
    """The fused M-step rewrites the compute copies in place; preparing them
    again from the master parameters (a reloaded model) gives the same LLs
    bit for bit."""
    rg, fam, k, gen = config(cfg)
    x = gen(128, seed=5)
    m = E.build_model(rg, fam, k=k, seed=0, data=x)
    trainer.em_stochastic_step(m, x, 0.5)
    a = m.log_likelihood(x)
    m.params.touch()
    b = m.log_likelihood(x)
    assert np.array_equal(a, b)
