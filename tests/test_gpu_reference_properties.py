"""Reference behaviours of the widened API on the GPU: the properties the
reference's own tests check for sampling, conditionals, training and mixtures
(/root/reference/pkg/tests/test_engine.py:94-236, test_trainer.py:59-192),
restated against this package. Parity with the reference's numbers is in
test_gpu_sampling.py / test_mixture.py; these are the behavioural checks."""

import numpy as np
import pytest

import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import engine, trainer
from paper_2004_06231_b200.builders import make_family, make_structure
from paper_2004_06231_b200.structures import StructureConfig

pytestmark = pytest.mark.gpu


def _tiny_discrete(seed=0, d_vars=3, k=3, replicas=2, num_states=2):
    rg = E.random_binary_tree(d_vars, StructureConfig(depth=1, replicas=replicas, seed=seed))
    circuit = E.compile_graph(rg, k=k)
    family = E.CategoricalFamily(num_states)
    return circuit, E.init_parameters(circuit, family, seed=seed + 1), family


def _gaussian_model(seed=0, d_vars=4, k=3, replicas=2, data=None):
    rg = make_structure("rat", d_vars=d_vars, depth=2, replicas=replicas, seed=seed)
    return E.build_model(rg, make_family("gaussian"), k=k, seed=seed + 1, data=data)


def test_sample_joint_matches_forward():
    """test_engine.py:205-216: empirical joint of 20000 samples vs exp(forward)."""
    circuit, params, family = _tiny_discrete(seed=19, d_vars=2, k=2)
    n = 20000
    draws = E.sample(circuit, params, family, n, seed=1)
    tv = 0.0
    for a in range(2):
        for b in range(2):
            want = float(np.exp(E.forward(circuit, params, family,
                                          np.array([[a, b]], float)).log_likelihood[0]))
            tv += 0.5 * abs(np.mean(np.all(draws == [a, b], axis=1)) - want)
    assert tv < 0.02


def test_sample_gaussian_mean():
    """test_engine.py:193-202."""
    rg = E.random_binary_tree(2, StructureConfig(depth=1, replicas=1, seed=0))
    circuit = E.compile_graph(rg, k=1)
    family = E.GaussianFamily()
    params = E.init_parameters(circuit, family, seed=0)
    phi = params.phi
    phi[..., 0] = 1.5
    phi[..., 1] = 1.5 ** 2 + 1.0
    params.phi = phi
    n = 4000
    draws = E.sample(circuit, params, family, n, seed=3)
    assert np.all(np.abs(draws.mean(axis=0) - 1.5) < 3.0 / np.sqrt(n))


def test_conditional_sample_evidence_cases():
    """test_engine.py:219-236: full evidence is copied, empty evidence equals
    sample(), evidence outside the support raises."""
    circuit, params, family = _tiny_discrete(seed=23)
    x_e = np.array([1.0, 0.0, 1.0])
    out = E.conditional_sample(circuit, params, family, x_e, [0, 1, 2], 10, seed=0)
    assert np.array_equal(out, np.tile(x_e, (10, 1)))
    a = E.conditional_sample(circuit, params, family, np.zeros(3), [], 15, seed=4)
    assert np.array_equal(a, E.sample(circuit, params, family, 15, seed=4))
    with pytest.raises(Exception):
        E.conditional_sample(circuit, params, family, np.array([5.0, 0.0, 0.0]), [0], 5, seed=0)


def test_conditional_empty_evidence_is_log_likelihood():
    """test_engine.py:94-100."""
    circuit, params, family = _tiny_discrete(seed=3)
    x = np.array([[1.0, 0.0, 1.0], [0.0, 0.0, 0.0]])
    ll = E.forward(circuit, params, family, x).log_likelihood
    cond = E.conditional_log_density(circuit, params, family, x, query=[0, 1, 2], evidence=[])
    assert np.allclose(cond, ll, atol=1e-12)


def test_two_component_mixture_recovers_means():
    """test_trainer.py:70-80."""
    rng = np.random.default_rng(9)
    data = np.concatenate([rng.normal(-3, 0.4, (300, 2)), rng.normal(3, 0.4, (300, 2))])
    rg = make_structure("rat", d_vars=2, depth=1, replicas=1, seed=0)
    model = E.build_model(rg, make_family("gaussian"), k=2, seed=4, data=data)
    for _ in range(30):
        E.em_full_step(model, data)
    mus = np.sort(model.params.phi[0, :, 0, 0])
    assert abs(mus[0] + 3) < 0.05 and abs(mus[1] - 3) < 0.05


def test_train_determinism_full_mode_and_empty():
    """test_trainer.py:118-145."""
    rng = np.random.default_rng(5)
    data = rng.normal(size=(120, 4))
    cfg = trainer.TrainerConfig(mode="stochastic", step_size=0.5, batch_size=40, epochs=4,
                                seed=11)
    ma = trainer.train(_gaussian_model(seed=5, data=data), data, cfg, valid=data[:20])
    mb = trainer.train(_gaussian_model(seed=5, data=data), data, cfg, valid=data[:20])
    assert len(ma) == 4
    assert [m.train_ll for m in ma] == [m.train_ll for m in mb]
    assert [m.valid_ll for m in ma] == [m.valid_ll for m in mb]
    full = trainer.train(_gaussian_model(seed=6, data=data[:100]), data[:100],
                         trainer.TrainerConfig(mode="full", epochs=10))
    assert np.all(np.diff([m.train_ll for m in full]) >= -1e-8)
    with pytest.raises(ValueError):
        trainer.train(_gaussian_model(seed=7), np.zeros((0, 4)), trainer.TrainerConfig(epochs=1))


def test_mixture_properties():
    """test_trainer.py:148-192: k-means separates blobs; a one-cluster mixture
    is the model itself; the weights are the cluster proportions."""
    rng = np.random.default_rng(8)
    data = np.concatenate([rng.normal(-5, 0.3, (100, 3)), rng.normal(5, 0.3, (100, 3))])
    labels, centers = trainer.kmeans(data, 2, seed=0)
    assert max(np.mean(labels[:100] == 0), np.mean(labels[:100] == 1)) >= 0.95
    assert len(centers) == 2

    data = np.random.default_rng(10).normal(size=(80, 4))
    cfg = trainer.TrainerConfig(mode="full", epochs=3)
    factory = lambda c, subset: _gaussian_model(seed=20, data=subset)  # noqa: E731
    mix = trainer.train_mixture(data, 1, factory, cfg, seed=0)
    assert isinstance(mix, trainer.MixtureModel)
    assert abs(np.exp(mix.log_pi).sum() - 1.0) < 1e-12
    single = factory(0, data)
    trainer.train(single, data, cfg)
    assert np.allclose(mix.log_likelihood(data), single.log_likelihood(data), atol=1e-12)

    rng = np.random.default_rng(12)
    data = np.concatenate([rng.normal(-4, 0.3, (60, 2)), rng.normal(4, 0.3, (140, 2))])

    def factory2(c, subset):
        rg = make_structure("rat", d_vars=2, depth=1, replicas=1, seed=0)
        return E.build_model(rg, make_family("gaussian"), k=1, seed=c, data=subset)

    mix = trainer.train_mixture(data, 2, factory2, trainer.TrainerConfig(mode="full", epochs=2),
                                seed=1)
    assert np.allclose(np.sort(np.exp(mix.log_pi)), [0.3, 0.7], atol=0.02)
