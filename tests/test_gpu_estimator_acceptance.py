"""The reference's estimator tests (pkg/tests/test_estimator.py) and the
acceptance criteria on normalisation, conditional inference and persistence
(pkg/tests/test_acceptance.py criteria 02, 07, 10), restated on the GPU
engine. Enumeration over all joint states stands in for the reference's
exhaustive circuit oracle."""

import itertools

import numpy as np
import pytest

import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import engine, modelio
from paper_2004_06231_b200.estimator import EinsumNetwork
from paper_2004_06231_b200.structures import StructureConfig

pytestmark = pytest.mark.gpu


def _data(seed=0, n=120, d=4):
    rng = np.random.default_rng(seed)
    return np.concatenate([rng.normal(-1, 0.5, (n // 2, d)), rng.normal(1, 0.5, (n // 2, d))])


def test_estimator_fit_score_sample():
    """test_estimator.py:15-61."""
    data = _data()
    est = EinsumNetwork(depth=2, replicas=2, k=4, mode="full", epochs=5, seed=0).fit(data)
    assert est.n_features_in_ == 4 and len(est.metrics_) == 5
    assert est.metrics_[-1].train_ll >= est.metrics_[0].train_ll
    ll = est.score_samples(data[:10])
    assert ll.shape == (10,)
    assert abs(est.score(data) - est.score_samples(data).mean()) < 1e-12
    a, b = est.sample(6, seed=1), est.sample(6, seed=1)
    assert a.shape == (6, 4) and np.array_equal(a, b)
    out = est.conditional_sample(data[0], [0, 1], n_samples=4, seed=2)
    assert np.array_equal(out[:, :2], np.tile(data[0][:2], (4, 1)))


def test_estimator_sklearn_protocol():
    """test_estimator.py:32-82: NotFittedError, get/set_params, GridSearchCV,
    Poon-Domingos through the estimator."""
    from sklearn.exceptions import NotFittedError
    from sklearn.model_selection import GridSearchCV
    with pytest.raises(NotFittedError):
        EinsumNetwork().score_samples(np.zeros((2, 4)))
    params = EinsumNetwork(k=7, epochs=2).get_params()
    assert EinsumNetwork().set_params(**params).get_params() == params
    gs = GridSearchCV(EinsumNetwork(mode="full", epochs=2, replicas=1, depth=1), {"k": [1, 2]},
                      cv=2)
    gs.fit(_data(seed=4, n=60))
    assert gs.best_params_["k"] in (1, 2)
    x = np.random.default_rng(5).normal(0.5, 0.1, size=(50, 16))
    est = EinsumNetwork(structure="pd", height=4, width=4, deltas=(2,), k=2, mode="full",
                        epochs=2).fit(x)
    assert np.isfinite(est.score(x))


@pytest.mark.parametrize("seed", range(6))
def test_acceptance_normalisation(seed):
    """Criterion 02: all variables marginalised gives log 1; a categorical
    circuit's probabilities over every joint state sum to 1."""
    rng = np.random.default_rng(200 + seed)
    d = int(rng.integers(3, 8))
    depth = min(int(rng.integers(1, 3)), int(np.floor(np.log2(d))))
    rg = E.random_binary_tree(d, StructureConfig(depth=depth,
                                                 replicas=int(rng.integers(1, 3)), seed=seed))
    fam = E.CategoricalFamily(int(rng.integers(2, 4)))
    k = int(rng.choice([2, 3, 8, 16]))
    circuit = E.compile_graph(rg, k)
    params = E.init_parameters(circuit, fam, seed=seed)
    grid = np.array(list(itertools.product(range(fam.num_states), repeat=d)), dtype=np.float64)
    ll = E.forward(circuit, params, fam, grid, marg_mask=np.ones(d, bool)).log_likelihood
    assert np.max(np.abs(ll)) <= 1e-6
    ll = E.forward(circuit, params, fam, grid).log_likelihood
    assert abs(np.exp(ll).sum() - 1.0) <= 1e-5


def test_acceptance_conditional_inference():
    """Criterion 07: conditional densities against enumeration of the joint,
    and the empirical conditional distribution of 1e5 conditional samples."""
    rg = E.random_binary_tree(3, StructureConfig(depth=1, replicas=2, seed=1))
    circuit = E.compile_graph(rg, k=3)
    fam = E.CategoricalFamily(2)
    params = E.init_parameters(circuit, fam, seed=2)

    def joint(x):
        return float(np.exp(E.forward(circuit, params, fam, np.array([x])).log_likelihood[0]))

    for xq in (0.0, 1.0):
        x = np.array([xq, 1.0, 0.0])
        got = E.conditional_log_density(circuit, params, fam, x, query=[0], evidence=[1, 2])[0]
        want = np.log(joint(x) / sum(joint(np.array([s, 1.0, 0.0])) for s in (0.0, 1.0)))
        assert abs(got - want) <= 1e-6
    draws = E.conditional_sample(circuit, params, fam, np.array([0.0, 1.0, 0.0]), [1, 2],
                                 10 ** 5, seed=3)
    assert np.all(draws[:, 1] == 1.0) and np.all(draws[:, 2] == 0.0)
    norm = sum(joint(np.array([s, 1.0, 0.0])) for s in (0.0, 1.0))
    tv = 0.5 * sum(abs(np.mean(draws[:, 0] == s) - joint(np.array([s, 1.0, 0.0])) / norm)
                   for s in (0.0, 1.0))
    assert tv <= 0.02


@pytest.mark.parametrize("seed", range(10))
def test_acceptance_persistence(seed, tmp_path):
    """Criterion 10: save / load keeps every log-likelihood bit for bit."""
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.integers(2, 12))
    rg = E.random_binary_tree(d, StructureConfig(depth=1, replicas=int(rng.integers(1, 4)),
                                                 seed=seed))
    kind = seed % 3
    if kind == 0:
        fam, x = E.GaussianFamily(), rng.normal(size=(40, d))
    elif kind == 1:
        fam = E.CategoricalFamily(3)
        x = rng.integers(0, 3, (40, d)).astype(float)
    else:
        fam = E.BinomialFamily(4)
        x = rng.integers(0, 5, (40, d)).astype(float)
    model = E.build_model(rg, fam, k=int(rng.choice([2, 5, 8, 16])), seed=seed, data=x)
    path = str(tmp_path / f"m{seed}.einm")
    modelio.save_model(path, model)
    again = modelio.load_model(path)
    assert np.array_equal(model.log_likelihood(x), again.log_likelihood(x))


@pytest.mark.parametrize("seed", range(8))
def test_acceptance_gradient_identity(seed):
    """Criterion 03 (test_acceptance.py:56-89): the device EM statistics are
    the reference's gradient identity -- acc / (w * B) = d mean LL / d w for
    einsum and mixing weights, acc_p / B = d mean LL / d (leaf log offset) --
    checked against fp64 central differences of the oracle's forward pass."""
    from oracle import einet_oracle as O
    rng = np.random.default_rng(300 + seed)
    d = int(rng.integers(2, 8))
    depth = min(int(rng.integers(1, 3)), int(np.floor(np.log2(d))))
    rg = E.random_binary_tree(d, StructureConfig(depth=depth, replicas=int(rng.integers(1, 4)),
                                                 seed=seed))
    if seed % 2:
        fam = E.CategoricalFamily(3)
        x = rng.integers(0, 3, (24, d)).astype(float)
    else:
        fam = E.GaussianFamily()
        x = rng.normal(size=(24, d)).astype(np.float32).astype(np.float64)
    circuit = E.compile_graph(rg, int(rng.choice([2, 3, 8])))
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=seed, data=x)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    op = O.OracleParams({i: f32(w) for i, w in ein.items()}, {i: f32(w) for i, w in mix.items()},
                        f32(phi))
    p = engine.Parameters.from_numpy(circuit, fam, op.einsum, op.mixing, op.phi)
    st = E.backward(circuit, p, fam, E.forward(circuit, p, fam, x))
    doc, B, h = fam.to_dict(), len(x), 1e-6

    def mean_ll(params, offset=None):
        return float(np.mean(O.forward(circuit, params, doc, x,
                                       leaf_log_offset=offset).root[:, 0]))

    def check(want, plus, minus):
        got = (plus - minus) / (2 * h)
        assert abs(got - want) <= 1e-3 * max(abs(want), 1e-3), (got, want)

    for _ in range(2):
        li = list(st.einsum)[int(rng.integers(len(st.einsum)))]
        idx = tuple(int(rng.integers(s)) for s in st.einsum[li].shape)
        want = st.einsum[li][idx] / (op.einsum[li][idx] * B)
        a, b = op.copy(), op.copy()
        a.einsum[li][idx] += h
        b.einsum[li][idx] -= h
        check(want, mean_ll(a), mean_ll(b))
    for li, acc in st.mixing.items():
        m, c = (int(v) for v in np.argwhere(circuit.layers[li].mask)[0])
        want = acc[m, c] / (op.mixing[li][m, c] * B)
        a, b = op.copy(), op.copy()
        a.mixing[li][m, c] += h
        b.mixing[li][m, c] -= h
        check(want, mean_ll(a), mean_ll(b))
        break
    dd, kk, rr = (int(rng.integers(s)) for s in st.acc_p.shape)
    off = np.zeros(op.phi.shape[:3])
    off[dd, kk, rr] = h
    check(st.acc_p[dd, kk, rr] / B, mean_ll(op, off), mean_ll(op, -off))
