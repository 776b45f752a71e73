"""Generate k-means and mixture-training fixtures from the reference.

Run in the build container (the reference exists only here):
    python tests/golden/gen_mixture.py
``mixture.npz`` holds the reference's ``kmeans`` labels and centres
(trainer.py:165-190) for blob data, tied duplicate points (empty clusters are
re-seeded) and a larger 48-variable case, and one ``train_mixture`` run
(trainer.py:212-228): RAT structure on 8 Gaussian variables, 3 clusters,
2 epochs of batch 16 -- the final parameters of every component, the mixture
weights and the mixture log-likelihoods of the data.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def blobs(n, d, k, seed, spread=3.0):
    rng = np.random.default_rng(seed)
    centres = rng.normal(0.0, spread, (k, d))
    lab = rng.integers(0, k, n)
    return centres[lab] + rng.normal(size=(n, d))


def main():
    sys.path.insert(0, REF)
    from einet import expfam, model, structures, trainer

    out = {}
    km = [("blobs", blobs(300, 5, 3, 0), 3, 0),
          ("wide", blobs(2000, 48, 10, 1, spread=1.0), 10, 3)]
    dup = np.concatenate([np.zeros((10, 2)), np.ones((10, 2))])
    km += [(f"dup{s}", dup, 3, s) for s in range(6)]
    for name, x, k, seed in km:
        lab, cen = trainer.kmeans(x, k, seed=seed)
        out[f"km_{name}_x"] = x
        out[f"km_{name}_k"] = np.array(k)
        out[f"km_{name}_seed"] = np.array(seed)
        out[f"km_{name}_labels"] = lab
        out[f"km_{name}_centers"] = cen
    out["km_names"] = np.array([n for n, *_ in km])

    x = blobs(150, 8, 3, 7, spread=2.5)
    rg = structures.random_binary_tree(8, structures.StructureConfig(depth=2, replicas=2,
                                                                    seed=1))
    fam = expfam.GaussianFamily()
    cfg = trainer.TrainerConfig(epochs=2, batch_size=16, step_size=0.5, seed=0)
    mix = trainer.train_mixture(
        x, 3, lambda c, sub: model.build_model(rg, fam, k=4, seed=c, data=sub), cfg, seed=2)
    out["mix_x"] = x
    out["mix_rg_json"] = np.array(rg.to_json())
    out["mix_family_json"] = np.array(json.dumps(fam.to_dict()))
    out["mix_log_pi"] = mix.log_pi
    out["mix_ll"] = mix.log_likelihood(x)
    for c, m in enumerate(mix.components):
        for i, w in m.params.einsum.items():
            out[f"mix_c{c}_einsum_{i}"] = w
        for i, w in m.params.mixing.items():
            out[f"mix_c{c}_mixing_{i}"] = w
        out[f"mix_c{c}_phi"] = m.params.phi
    np.savez_compressed(os.path.join(HERE, "mixture.npz"), **out)
    print("saved mixture.npz", mix.log_pi)


if __name__ == "__main__":
    main()
