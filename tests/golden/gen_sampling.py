"""Generate sampling moment fixtures from the reference sampler.

Run in the build container (the reference exists only here):
    python tests/golden/gen_sampling.py
For a few golden circuits (their fp32 ``init`` parameters from the .npz
fixtures made by gen_golden.py) it draws n samples with the reference's own
``engine.sample`` / ``engine.conditional_sample`` (engine.py:391-423) and
stores their first and second moments (and per-state frequencies for
discrete families) in ``sampling.npz``. The reference draws with per-sample
numpy generators, the device with a Philox4x32-10 stream, so parity with the
reference is statistical: tests/test_oracle_golden.py checks the oracle's
Philox restatement (oracle/einet_oracle.py: sample_philox) against these
moments, and the GPU tests check the device against that restatement draw
for draw.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
N = 6000

# (fixture, evidence variables or None); evidence values are the fixture's x[0]
CASES = [
    ("rat_gaussian", None),
    ("rat_gaussian", [0, 3, 5]),
    ("rat_binomial", None),
    ("rat_categorical4", None),
    ("rat_categorical4", [1, 2]),
    ("pd_lift_gaussian_image", None),
    ("rat_binomial", [0, 4]),
    ("pd_lift_gaussian_image", list(range(0, 48, 2))),
]


def moments(s, fam):
    out = {"mean": s.mean(axis=0), "m2": (s.T @ s) / s.shape[0]}
    if fam["family"] != "gaussian":
        top = fam["num_states"] if fam["family"] == "categorical" else fam["n_trials"] + 1
        out["freq"] = np.stack([(s == v).mean(axis=0) for v in range(top)], axis=1)
    return out


def main():
    sys.path.insert(0, REF)
    from einet import compiler, engine, expfam, structures

    out = {"n": np.array(N)}
    for ci, (name, evidence) in enumerate(CASES):
        z = dict(np.load(os.path.join(HERE, name + ".npz")))
        rg = structures.RegionGraph.from_json(str(z["rg_json"]))
        circuit = compiler.compile_graph(rg, int(z["k"]), int(z["k_root"]))
        fam_doc = json.loads(str(z["family_json"]))
        family = expfam.ExponentialFamily.from_dict(fam_doc)
        ein = {i: z[f"init_einsum_{i}"] for i, l in enumerate(circuit.layers)
               if type(l).__name__ == "EinsumLayer"}
        mix = {i: z[f"init_mixing_{i}"] for i, l in enumerate(circuit.layers)
               if type(l).__name__ == "MixingLayer"}
        params = engine.Parameters(einsum=ein, mixing=mix, phi=z["init_phi"])
        if evidence is None:
            s = engine.sample(circuit, params, family, N, seed=11)
        else:
            s = engine.conditional_sample(circuit, params, family, z["x"][0], evidence, N,
                                          seed=11)
        key = f"case{ci}"
        out[f"{key}_name"] = np.array(name)
        out[f"{key}_evidence"] = np.array(evidence if evidence else [], dtype=np.int64)
        for m, v in moments(np.asarray(s, dtype=np.float64), fam_doc).items():
            out[f"{key}_{m}"] = v
        print(key, name, evidence, s.shape)
    out["num_cases"] = np.array(len(CASES))
    np.savez_compressed(os.path.join(HERE, "sampling.npz"), **out)
    print("saved sampling.npz")


if __name__ == "__main__":
    main()
