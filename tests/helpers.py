"""Shared loaders for the golden fixtures (CPU and GPU tests)."""

import json
import os

import numpy as np

from paper_2004_06231_b200.compiler import compile_graph
from paper_2004_06231_b200.expfam import ExponentialFamily
from paper_2004_06231_b200.structures import RegionGraph

from oracle import einet_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

CASES = ["c1_rat_categorical", "rat_gaussian", "rat_gaussian_masked", "rat_gaussian_kroot3",
         "pd_lift_gaussian_image", "rat_binomial", "rat_categorical4", "c2_mnist_pd",
         "c3_svhn_pd"]


class Case:
    def __init__(self, name):
        self.name = name
        self.z = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        z = self.z
        self.rg = RegionGraph.from_json(str(z["rg_json"]))
        self.k = int(z["k"])
        self.k_root = int(z["k_root"])
        self.circuit = compile_graph(self.rg, self.k, self.k_root)
        self.fam_doc = json.loads(str(z["family_json"]))
        self.family = ExponentialFamily.from_dict(self.fam_doc)
        self.x = z["x"]
        self.mask = z.get("mask")
        self.full = bool(z["full"])
        self.lam = float(z["lam"])

    def params(self, prefix="init"):
        ein = {i: self.z[f"{prefix}_einsum_{i}"] for i in self.einsum_layers()}
        mix = {i: self.z[f"{prefix}_mixing_{i}"] for i in self.mixing_layers()}
        return O.OracleParams(ein, mix, self.z[f"{prefix}_phi"])

    def einsum_layers(self):
        return [i for i, l in enumerate(self.circuit.layers) if type(l).__name__ == "EinsumLayer"]

    def mixing_layers(self):
        return [i for i, l in enumerate(self.circuit.layers) if type(l).__name__ == "MixingLayer"]

    def steps(self):
        return len(self.z.get("step_mean_ll", []))


def summarize(a):
    a = np.asarray(a)
    flat = a.reshape(a.shape[0], -1) if a.ndim > 1 else a[:, None]
    return np.concatenate([flat.sum(axis=1), flat[:, :8].ravel(), [a.sum(), (a * a).sum()]])


def close(a, b, rtol, atol):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    both_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
    with np.errstate(invalid="ignore"):
        err = np.where(both_inf, 0.0, np.abs(a - b))
    bound = atol + rtol * np.abs(b)
    bad = ~(err <= bound)
    if bad.any():
        i = np.unravel_index(np.argmax(np.where(bad, err / np.maximum(bound, 1e-300), 0)), a.shape)
        raise AssertionError(f"{bad.sum()} of {a.size} entries differ; worst at {i}: "
                             f"got {a[i]!r} want {b[i]!r} (rtol {rtol}, atol {atol})")


def sampling_cases():
    """(index, Case, evidence list) of tests/golden/sampling.npz."""
    g = dict(np.load(os.path.join(GOLDEN, "sampling.npz")))
    return g, [(i, Case(str(g[f"case{i}_name"])), [int(v) for v in g[f"case{i}_evidence"]])
               for i in range(int(g["num_cases"]))]


def oracle_samples(case, evidence, n, seed):
    """Philox-restated samples of the oracle (conditional when evidence)."""
    p = case.params("init")
    if not evidence:
        return O.sample_philox(case.circuit, p, case.fam_doc, n, seed=seed)
    mask = np.array([i not in evidence for i in range(case.circuit.d_vars)])
    tr = O.forward(case.circuit, p, case.fam_doc, case.x[:1], mask)
    return O.sample_philox(case.circuit, p, case.fam_doc, n, seed=seed, x_e=case.x[0],
                           evidence=evidence, trace=tr)


def moment_z(s, g, key):
    """Largest |z| of the sample moments of s against the fixture's reference
    moments (two-sample standard errors from s; constant columns such as
    evidence must match to 1e-9)."""
    n = s.shape[0]

    def z(mine, ref, var):
        se = np.sqrt(2.0 * var / n) + 1e-9 * (1.0 + np.abs(ref))
        return np.abs(mine - ref) / se

    prod = s[:, :, None] * s[:, None, :]
    zs = [z(s.mean(axis=0), g[f"{key}_mean"], s.var(axis=0)),
          z(prod.mean(axis=0), g[f"{key}_m2"], prod.var(axis=0))]
    if f"{key}_freq" in g:
        f = g[f"{key}_freq"]
        mine = np.stack([(s == v).mean(axis=0) for v in range(f.shape[1])], axis=1)
        zs.append(z(mine, f, np.maximum(mine * (1 - mine), 1.0 / n)))
    return max(float(np.max(v)) for v in zs)


# ---------------------------------------------------------------------------
# host-side packing in the device statistics layout (distributed tests)
# ---------------------------------------------------------------------------

def pack_stats(circuit, family, einsum, mixing, acc_pt, acc_p, ll_sum, n_samples, failed=0.0):
    """Reference-layout statistics -> flat fp64 vector in the device layout
    (acc_p compressed to one value per (leaf region, k))."""
    from paper_2004_06231_b200.distributed import stats_layout
    L = stats_layout(circuit, family)
    lay = L["layout"]
    out = np.zeros(L["total"])
    for i, (off, shape) in lay.einsum.items():
        out[off:off + int(np.prod(shape))] = np.asarray(einsum[i]).ravel()
    for i, (off, shape, _) in lay.mixing.items():
        out[off:off + int(np.prod(shape))] = np.asarray(mixing[i]).ravel()
    n_phi = int(np.prod(lay.phi_shape))
    out[L["acc_pt"]:L["acc_pt"] + n_phi] = np.asarray(acc_pt).ravel()
    leaf = circuit.layers[0]
    acc_p = np.asarray(acc_p)
    for li, (scope, rep) in enumerate(zip(leaf.scopes, leaf.replica)):
        out[L["p"] + li * circuit.k:L["p"] + (li + 1) * circuit.k] = acc_p[scope[0], :, int(rep)]
    out[L["ll"]:L["ll"] + 3] = (ll_sum, n_samples, failed)
    return out


def unpack_stats(circuit, family, flat):
    """Flat fp64 vector -> (einsum, mixing, acc_pt, acc_p, ll_sum, n_samples)."""
    from paper_2004_06231_b200.distributed import stats_layout
    L = stats_layout(circuit, family)
    lay = L["layout"]
    flat = np.asarray(flat, dtype=np.float64)
    einsum = {i: flat[o:o + int(np.prod(s))].reshape(s) for i, (o, s) in lay.einsum.items()}
    mixing = {i: flat[o:o + int(np.prod(s))].reshape(s) for i, (o, s, _) in lay.mixing.items()}
    n_phi = int(np.prod(lay.phi_shape))
    acc_pt = flat[L["acc_pt"]:L["acc_pt"] + n_phi].reshape(lay.phi_shape)
    acc_p = np.zeros(lay.phi_shape[:3])
    leaf = circuit.layers[0]
    for li, (scope, rep) in enumerate(zip(leaf.scopes, leaf.replica)):
        acc_p[np.asarray(scope), :, int(rep)] = flat[L["p"] + li * circuit.k:
                                                     L["p"] + (li + 1) * circuit.k]
    return einsum, mixing, acc_pt, acc_p, float(flat[L["ll"]]), float(flat[L["ll"] + 1])


def device_values(x32, active=None):
    """The float64 values the device evaluates for an fp32 batch.

    Gaussian leaves read image data on the 1/255 grid (every active value
    equal to float32(u / 255) for an integer u in [0, 255]) at u / 255
    exactly -- the value the reference's own u8 dataset loader produces
    (modelio.py:137-168) -- and any other batch at its fp32 values
    (csrc/leaf_i8.cu). Feeding the oracle these values makes both sides see
    the same inputs.
    """
    x32 = np.asarray(x32, dtype=np.float32)
    u = np.rint(x32.astype(np.float64) * 255.0)
    on = (u >= 0) & (u <= 255) & (np.float32(u / 255.0) == x32)
    if active is not None:
        on = on | ~np.asarray(active, bool)[None, :]
    if on.all():
        out = x32.astype(np.float64)
        fix = np.isfinite(x32)
        if active is not None:
            fix = fix & np.asarray(active, bool)[None, :]
        out[fix] = u[fix] / 255.0
        return out
    return x32.astype(np.float64)
