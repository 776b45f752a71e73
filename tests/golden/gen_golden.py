"""Generate golden vectors from the reference package itself.

Run in the build container (the reference exists only here):
    python tests/golden/gen_golden.py
It imports /root/reference/pkg/src/einet (read-only), builds each case with the
reference's own structures/compiler/init/forward/backward/EM functions and
stores inputs and outputs as small .npz fixtures next to this script. The
oracle (oracle/einet_oracle.py) and the host plan producers are pinned
against these files by tests/test_oracle_golden.py; nothing at test time on
the GPU box reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import einet  # noqa: F401
    from einet import builders, compiler, engine, expfam, model, structures, trainer
    return builders, compiler, engine, expfam, model, structures, trainer


def lift3(structures, rg):
    out = structures.RegionGraph(d_vars=3 * rg.d_vars, root=rg.root)
    for rid, r in rg.regions.items():
        out.regions[rid] = structures.Region(
            rid, frozenset(3 * p + c for p in r.scope for c in range(3)))
    out.partitions = dict(rg.partitions)
    return out


def image_data(n, d, seed):
    rng = np.random.default_rng(seed)
    x = rng.normal(0.5, 0.2, size=(n, d)) + rng.normal(0.0, 0.15, size=(n, 1))
    return np.round(np.clip(x, 0.0, 1.0) * 255.0) / 255.0


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def snapshot(prefix, params, out, full=True):
    for i, w in params.einsum.items():
        out[f"{prefix}_einsum_{i}"] = w if full else summarize(w)
    for i, w in params.mixing.items():
        out[f"{prefix}_mixing_{i}"] = w
    out[f"{prefix}_phi"] = params.phi if full else summarize(params.phi)


def summarize(a):
    a = np.asarray(a)
    flat = a.reshape(a.shape[0], -1) if a.ndim > 1 else a[:, None]
    return np.concatenate([flat.sum(axis=1), flat[:, :8].ravel(), [a.sum(), (a * a).sum()]])


def make_case(name, rg, family, k, x, seed, steps=3, lam=0.5, k_root=1, mask=None,
              full=True, chunk=4096):
    builders, compiler, engine, expfam, model, structures, trainer = _ref()
    x = f32(x)
    m = model.build_model(rg, family, k=k, k_root=k_root, seed=seed, data=x)
    # the GPU consumes fp32 parameters: pin the fp32-rounded parameters
    p = m.params
    for i in list(p.einsum):
        p.einsum[i] = f32(p.einsum[i])
    for i in list(p.mixing):
        p.mixing[i] = f32(p.mixing[i])
    p.phi = f32(p.phi)
    out = {"name": np.array(name), "k": np.array(k), "k_root": np.array(k_root),
           "seed": np.array(seed), "lam": np.array(lam), "x": x,
           "rg_json": np.array(rg.to_json()), "plan_json": np.array(m.circuit.plan_json()),
           "family_json": np.array(json.dumps(family.to_dict())), "full": np.array(full)}
    init = model.build_model(rg, family, k=k, k_root=k_root, seed=seed, data=x).params
    snapshot("init_exact", init, out, full)
    snapshot("init", p, out, full)
    tr = engine.forward(m.circuit, p, family, x, marg_mask=mask)
    out["root"] = tr.root
    if mask is not None:
        out["mask"] = np.asarray(mask, dtype=bool)
    st = engine.backward(m.circuit, p, family, tr)
    for i, a in st.einsum.items():
        out[f"stats_einsum_{i}"] = a if full else summarize(a)
    for i, a in st.mixing.items():
        out[f"stats_mixing_{i}"] = a
    out["stats_acc_p"] = st.acc_p if full else summarize(st.acc_p)
    out["stats_acc_pt"] = st.acc_pt if full else summarize(st.acc_pt)
    if mask is None and k_root == 1:
        lls = []
        for s in range(steps):
            lls.append(trainer.em_stochastic_step(m, x, lam, chunk=chunk))
            snapshot(f"step{s + 1}", m.params, out, full)
        out["step_mean_ll"] = np.array(lls)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "saved", sorted(out)[:4], "...")


def main():
    builders, compiler, engine, expfam, model, structures, trainer = _ref()
    S = structures
    rng = np.random.default_rng(1234)
    # C1 (BASELINE.json configs[0]): RAT16 d3 R2 K10 categorical, B=100
    make_case("c1_rat_categorical",
              S.random_binary_tree(16, S.StructureConfig(depth=3, replicas=2, seed=0)),
              expfam.CategoricalFamily(2), 10,
              np.random.default_rng(0).integers(0, 2, (100, 16)).astype(float), seed=0)
    make_case("rat_gaussian",
              S.random_binary_tree(8, S.StructureConfig(depth=2, replicas=3, seed=5)),
              expfam.GaussianFamily(), 4, rng.normal(size=(32, 8)), seed=3)
    make_case("rat_gaussian_masked",
              S.random_binary_tree(8, S.StructureConfig(depth=2, replicas=3, seed=5)),
              expfam.GaussianFamily(), 4, rng.normal(size=(12, 8)), seed=3,
              mask=np.array([0, 1, 0, 0, 1, 1, 0, 0], dtype=bool))
    make_case("rat_gaussian_kroot3",
              S.random_binary_tree(8, S.StructureConfig(depth=2, replicas=1, seed=2)),
              expfam.GaussianFamily(), 3, rng.normal(size=(10, 8)), seed=4, k_root=3)
    make_case("pd_lift_gaussian_image",
              lift3(S, S.poon_domingos(4, 4, S.StructureConfig(deltas=(2,), axes="both"))),
              builders.make_family("gaussian", image_mode=True), 3,
              image_data(16, 48, 7), seed=1)
    make_case("rat_binomial",
              S.random_binary_tree(6, S.StructureConfig(depth=1, replicas=2, seed=3)),
              expfam.BinomialFamily(5), 3,
              np.random.default_rng(3).integers(0, 6, (20, 6)).astype(float), seed=2)
    make_case("rat_categorical4",
              S.random_binary_tree(7, S.StructureConfig(depth=2, replicas=2, seed=9)),
              expfam.CategoricalFamily(4), 5,
              np.random.default_rng(9).integers(0, 4, (24, 7)).astype(float), seed=6,
              chunk=10)
    # C2 (MNIST-shaped PD, delta 7 vertical, K=10), small batch
    make_case("c2_mnist_pd",
              S.poon_domingos(28, 28, S.StructureConfig(deltas=(7,), axes="vertical")),
              builders.make_family("gaussian", image_mode=True), 10,
              image_data(16, 784, 11), seed=0, steps=2)
    # C3 (SVHN-shaped lifted PD, delta 8 vertical, K=40): summaries only
    make_case("c3_svhn_pd",
              lift3(S, S.poon_domingos(32, 32, S.StructureConfig(deltas=(8,),
                                                                 axes="vertical"))),
              builders.make_family("gaussian", image_mode=True), 40,
              image_data(8, 3072, 13), seed=0, steps=2, full=False)
    # plan documents of the benchmark graphs (compiler parity)
    plans = {}
    for name, rg, k in [
        ("C1", S.random_binary_tree(16, S.StructureConfig(depth=3, replicas=2, seed=0)), 10),
        ("C2", S.poon_domingos(28, 28, S.StructureConfig(deltas=(7,), axes="vertical")), 10),
        ("C3", lift3(S, S.poon_domingos(32, 32, S.StructureConfig(deltas=(8,),
                                                                  axes="vertical"))), 40),
        ("C3b", lift3(S, S.poon_domingos(32, 32, S.StructureConfig(deltas=(8,),
                                                                   axes="both"))), 40),
        ("PD_multi", S.poon_domingos(3, 4, S.StructureConfig(deltas=(1, 2), axes="both")), 2),
        ("RAT_big", S.random_binary_tree(64, S.StructureConfig(depth=4, replicas=10,
                                                               seed=7)), 5),
    ]:
        c = compiler.compile_graph(rg, k)
        plans[name] = {"rg": rg.to_json(), "plan": c.plan_json(),
                       "replicas": {str(a): b for a, b in c.replicas.replica_of.items()}}
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(plans, f)
    # known answers of log_einsum_exp (engine.py:91-109)
    cases = {}
    w = np.full((1, 2, 2, 2), 0.25)
    for nm, left, right, ww in [
        ("uniform", np.log(0.5) * np.ones((1, 2)), np.log(0.5) * np.ones((1, 2)), w),
        ("underflow", np.array([[-1000.0, -1001.0]]), np.array([[-1000.0, -1000.0]]), w),
        ("neg_inf", np.array([[-np.inf, -np.inf]]), np.array([[0.0, 0.0]]),
         np.full((1, 1, 2, 2), 0.25)),
        ("random", rng.normal(-50, 5, (6, 3, 4)), rng.normal(-50, 5, (6, 3, 4)),
         engine.project_einsum_weights(rng.random((3, 5, 4, 4)))),
    ]:
        cases[nm] = {"left": left.tolist(), "right": right.tolist(), "w": ww.tolist(),
                     "out": np.where(np.isinf(o := engine.log_einsum_exp(left, right, ww)),
                                     -1e308, o).tolist()}
    with open(os.path.join(HERE, "log_einsum_exp.json"), "w") as f:
        json.dump(cases, f)
    print("done")


if __name__ == "__main__":
    main()
