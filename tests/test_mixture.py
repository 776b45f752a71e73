"""Cluster-then-mix pipeline (reference trainer.py:165-228).

CPU: ``kmeans`` reproduces the reference's labels and centres exactly
(tests/golden/mixture.npz from gen_mixture.py), including re-seeded empty
clusters, with the distance matrix computed in row blocks.
GPU: ``train_mixture`` matches the reference's run (component parameters
rtol 1e-4, leaf phi atol 1e-6, identical mixture weights, LLs 1e-4 relative);
``train_many`` leaves every model bitwise where sequential ``train`` would.
"""

import json
import os

import numpy as np
import pytest
import torch

import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import trainer
from paper_2004_06231_b200.expfam import ExponentialFamily
from paper_2004_06231_b200.structures import RegionGraph

from tests.helpers import GOLDEN, close

G = dict(np.load(os.path.join(GOLDEN, "mixture.npz")))


@pytest.mark.parametrize("name", [str(n) for n in G["km_names"]])
@pytest.mark.parametrize("block", [None, 7])
def test_kmeans_matches_reference(name, block):
    x = G[f"km_{name}_x"]
    lab, cen = trainer.kmeans(x, int(G[f"km_{name}_k"]), seed=int(G[f"km_{name}_seed"]),
                              block_rows=block)
    assert np.array_equal(lab, G[f"km_{name}_labels"])
    assert np.array_equal(cen, G[f"km_{name}_centers"])


def test_kmeans_errors():
    x = np.zeros((3, 2))
    with pytest.raises(ValueError):
        trainer.kmeans(x, 0)
    with pytest.raises(ValueError):
        trainer.kmeans(x, 4)


def _setup():
    rg = RegionGraph.from_json(str(G["mix_rg_json"]))
    fam = ExponentialFamily.from_dict(json.loads(str(G["mix_family_json"])))
    cfg = trainer.TrainerConfig(epochs=2, batch_size=16, step_size=0.5, seed=0)
    return rg, fam, cfg


@pytest.mark.gpu
@pytest.mark.parametrize("streams", [1, 16])
def test_train_mixture_matches_reference(streams):
    rg, fam, cfg = _setup()
    x = G["mix_x"]
    mix = trainer.train_mixture(x, 3, lambda c, sub: E.build_model(rg, fam, k=4, seed=c,
                                                                  data=sub),
                                cfg, seed=2, streams=streams)
    assert np.array_equal(mix.log_pi, G["mix_log_pi"])
    for c, m in enumerate(mix.components):
        ein, mx, phi = m.params.to_numpy()
        for i in ein:
            close(ein[i], G[f"mix_c{c}_einsum_{i}"], 1e-4, 1e-9)
        for i in mx:
            close(mx[i], G[f"mix_c{c}_mixing_{i}"], 1e-4, 1e-9)
        close(phi, G[f"mix_c{c}_phi"], 1e-4, 1e-6)
    ll = mix.log_likelihood(x)
    want = G["mix_ll"]
    assert (np.abs(ll - want) <= 1e-4 * np.maximum(np.abs(want), 1.0)).all()


@pytest.mark.gpu
def test_train_many_equals_sequential_train():
    from paper_2004_06231_b200.data import config
    rg, fam, k, gen = config("C2")
    datas = [gen(n, seed=s) for s, n in enumerate((700, 333, 1024))]
    cfg = trainer.TrainerConfig(epochs=2, batch_size=256, step_size=0.5, seed=4)
    seq = [E.build_model(rg, fam, k=k, seed=i, data=d) for i, d in enumerate(datas)]
    par = [E.build_model(rg, fam, k=k, seed=i, data=d) for i, d in enumerate(datas)]
    ms = [trainer.train(m, d, cfg) for m, d in zip(seq, datas)]
    mp = trainer.train_many(par, datas, cfg, streams=3)
    for a, b, la, lb in zip(seq, par, ms, mp):
        assert np.array_equal(a.params.flat.cpu().numpy(), b.params.flat.cpu().numpy())
        assert [e.train_ll for e in la] == [e.train_ll for e in lb]


@pytest.mark.gpu
def test_train_many_raises_reference_errors():
    from paper_2004_06231_b200.data import config
    rg, fam, k, gen = config("C1")
    good = gen(64, seed=1)
    bad = gen(64, seed=2)
    bad[5, 3] = 2.0  # outside {0, 1}
    cfg = trainer.TrainerConfig(epochs=1, batch_size=16, step_size=0.5)
    models = [E.build_model(rg, fam, k=k, seed=i, data=good) for i in range(2)]
    with pytest.raises(E.UnsupportedValueError):
        trainer.train_many(models, [good, bad], cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [900, 610])  # 610: the ragged last batch uses another bucket
def test_train_stops_at_failing_batch(n):
    """after a failing batch the epoch's later M-steps are no-ops, so
    the parameters are those after the last good batch, as the reference's
    exception leaves them (trainer.py:146-155)."""
    from paper_2004_06231_b200.data import config
    rg, fam, k, gen = config("C1")
    x = gen(n, seed=3)
    bs = 300
    cfg = trainer.TrainerConfig(epochs=1, batch_size=bs, step_size=0.5, seed=5)
    perm = np.random.default_rng(cfg.seed).permutation(n)
    bad_batch = 1
    x[perm[bad_batch * bs + 2], 4] = 3.0  # outside {0, 1}
    m = E.build_model(rg, fam, k=k, seed=0, data=x)
    ref = E.build_model(rg, fam, k=k, seed=0, data=x)
    with pytest.raises(E.UnsupportedValueError, match="variable 4"):
        trainer.train(m, x, cfg)
    for bi in range(bad_batch):
        trainer.em_stochastic_step(ref, x[perm[bi * bs:(bi + 1) * bs]], 0.5)
    assert np.array_equal(m.params.flat.cpu().numpy(), ref.params.flat.cpu().numpy())


@pytest.mark.gpu
def test_train_after_parameter_change_uses_new_parameters():
    """a cached epoch graph replayed after the parameters were set
    from the host must see the new parameters (compute copies re-derived)."""
    from paper_2004_06231_b200.data import config
    rg, fam, k, gen = config("C2")
    x = gen(300, seed=1)
    cfg = trainer.TrainerConfig(epochs=1, batch_size=100, step_size=0.5, seed=2)
    a = E.build_model(rg, fam, k=k, seed=0, data=x)
    b = E.build_model(rg, fam, k=k, seed=7, data=x)
    trainer.train(a, x, cfg)                       # captures a's epoch graph
    a.params.phi = b.params.phi                    # host setters -> touch()
    for i in b.params.einsum.keys():
        a.params.einsum[i] = b.params.einsum[i]
    for i in b.params.mixing.keys():
        a.params.mixing[i] = b.params.mixing[i]
    assert torch.equal(a.params.flat, b.params.flat)
    ma = trainer.train(a, x, cfg)                  # replays the cached graph
    mb = trainer.train(b, x, cfg)
    assert torch.equal(a.params.flat, b.params.flat)
    assert [e.train_ll for e in ma] == [e.train_ll for e in mb]
