"""Host-side API pieces: family utilities (reference tests/test_expfam.py
known answers), configuration validation, the estimator's sklearn contract."""

import numpy as np
import pytest

import paper_2004_06231_b200 as E
from paper_2004_06231_b200.builders import make_family, make_structure
from paper_2004_06231_b200.expfam import ExponentialFamily
from paper_2004_06231_b200.trainer import TrainerConfig


def test_gaussian_known_answers():
    fam = E.GaussianFamily()
    assert abs(fam.log_prob(np.array([0.0, 1.0]), 0.0) - (-0.9189385)) < 1e-6
    phi = E.GaussianFamily(var_min=1e-2).project(np.array([[2.0, 4.0]]))
    assert phi[0, 0] == 2.0 and abs(phi[0, 1] - 4.0 - 1e-2) < 1e-15
    with pytest.raises(E.UnsupportedValueError):
        fam.check_support(np.array([0.0, np.nan]), 1)


def test_categorical_and_binomial_known_answers():
    from scipy.stats import binom
    cat = E.CategoricalFamily(2)
    assert abs(cat.log_prob(np.array([0.25, 0.75]), 1) - np.log(0.75)) < 1e-12
    b = E.BinomialFamily(6)
    for x in range(7):
        assert abs(b.log_prob(np.array([1.8]), x) - binom.logpmf(x, 6, 0.3)) < 1e-10
    with pytest.raises(E.UnsupportedValueError):
        E.CategoricalFamily(3).check_support(np.array([0.5]), 0)


def test_em_update_closed_forms():
    fam = E.GaussianFamily(var_min=1e-2)
    new = E.ef_em_update(fam, np.array([[[[0.0, 1.0]]]]), np.array([[[[2.0, 2.0]]]]),
                         np.array([[[2.0]]]))
    assert abs(new[0, 0, 0, 0] - 1.0) < 1e-12
    keep = E.ef_em_update(E.GaussianFamily(), np.array([[[[0.3, 1.09]]]]),
                          np.zeros((1, 1, 1, 2)), np.zeros((1, 1, 1)))
    assert np.allclose(keep, [[[[0.3, 1.09]]]])


def test_family_serialisation_round_trip():
    for fam in (E.GaussianFamily(var_min=1e-3), E.CategoricalFamily(5), E.BinomialFamily(9)):
        again = ExponentialFamily.from_dict(fam.to_dict())
        assert type(again) is type(fam) and again.to_dict() == fam.to_dict()


def test_config_validation():
    with pytest.raises(ValueError):
        TrainerConfig(mode="sgd")
    with pytest.raises(ValueError):
        TrainerConfig(step_size=1.5)
    with pytest.raises(ValueError):
        TrainerConfig(batch_size=0)


def test_builders():
    assert make_family("gaussian", image_mode=True).var_max == 1e-2
    with pytest.raises(ValueError):
        make_family("poisson")
    rg = make_structure("pd", d_vars=48, height=4, width=4, deltas=(2,), channels=3)
    assert rg.d_vars == 48
    with pytest.raises(ValueError):
        make_structure("pd", d_vars=17, height=4, width=4)


def test_estimator_params_round_trip():
    est = E.EinsumNetwork(k=7, epochs=2)
    params = est.get_params()
    assert params["k"] == 7
    assert E.EinsumNetwork().set_params(**params).get_params() == params


def test_weight_projection_simplex():
    w = E.project_einsum_weights(np.random.default_rng(0).random((3, 2, 4, 4)))
    assert np.allclose(w.sum(axis=(2, 3)), 1.0, atol=1e-12) and w.min() >= 1e-12


def test_host_batch_conversions():
    """trainer._host_batch: float32 and uint8 pass through unchanged, float64
    converts (multi-threaded ATen) exactly like numpy's astype(float32)."""
    import numpy as np
    import torch

    from paper_2004_06231_b200 import trainer
    rng = np.random.default_rng(0)
    x64 = rng.normal(size=(300, 70)) * 123.456
    t = trainer._host_batch(x64)
    assert t.dtype == torch.float32 and t.is_contiguous()
    assert np.array_equal(t.numpy(), x64.astype(np.float32))
    x32 = x64.astype(np.float32)
    assert np.array_equal(trainer._host_batch(x32).numpy(), x32)
    u8 = rng.integers(0, 256, (5, 9)).astype(np.uint8)
    tu = trainer._host_batch(u8)
    assert tu.dtype == torch.uint8 and np.array_equal(tu.numpy(), u8)
    assert tuple(trainer._host_batch(x64[0]).shape) == (1, 70)
