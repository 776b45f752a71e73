"""CPU oracle for the Einsum-Network EM hot path -- TEST INFRASTRUCTURE ONLY.

A float64 NumPy restatement of the reference algorithm, used by ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` as the *checker*. The product path
(``paper_2004_06231_b200``) never imports this module.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the reference package itself
(``tests/golden/gen_golden.py`` imports ``/root/reference/pkg/src``).

Each function cites the reference ``file:line`` it restates
(paths relative to ``/root/reference/pkg/src/einet``).

Inputs: a ``LayeredCircuit`` (from either compiler -- the plans are
identical), parameters as ``OracleParams`` in the reference layouts
(``einsum[i]: (L, K_out, K, K)``, ``mixing[i]: (M, Dmax)``,
``phi: (D, K, R, T)``) and the family as its ``to_dict()`` document.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

LOG_2PI = math.log(2.0 * math.pi)
EPS_W = 1e-12        # engine.py:20
EPS_COUNT = 1e-12    # trainer.py:23


class OracleSupportError(ValueError):
    """Mirrors ``UnsupportedValueError`` (expfam.py:19-20)."""


@dataclass
class OracleParams:
    einsum: dict
    mixing: dict
    phi: np.ndarray

    def copy(self):
        return OracleParams({i: w.copy() for i, w in self.einsum.items()},
                            {i: w.copy() for i, w in self.mixing.items()},
                            self.phi.copy())


@dataclass
class OracleTrace:
    buffer: np.ndarray
    outputs: list
    root: np.ndarray
    x: np.ndarray
    marg_mask: object = None

    @property
    def log_likelihood(self):
        return self.root[:, 0]


@dataclass
class OracleStats:
    einsum: dict
    mixing: dict
    acc_p: np.ndarray
    acc_pt: np.ndarray
    n_samples: int = 0
    ll_sum: float = 0.0

    def merge(self, other):
        """engine.py:228-236: elementwise sums."""
        for i in other.einsum:
            self.einsum[i] = self.einsum[i] + other.einsum[i]
        for i in other.mixing:
            self.mixing[i] = self.mixing[i] + other.mixing[i]
        self.acc_p = self.acc_p + other.acc_p
        self.acc_pt = self.acc_pt + other.acc_pt
        self.n_samples += other.n_samples
        self.ll_sum += other.ll_sum
        return self


def _kind(layer):
    name = type(layer).__name__
    if name == "LeafLayer":
        return "leaf"
    return "einsum" if name == "EinsumLayer" else "mixing"


# ----------------------------------------------------------------------------
# families (expfam.py:82-275)
# ----------------------------------------------------------------------------

def suff_dim(fam) -> int:
    if fam["family"] == "gaussian":
        return 2
    if fam["family"] == "categorical":
        return int(fam["num_states"])
    return 1


def check_support(fam, column, var):
    """expfam.py:104-106 / 174-178 / 239-243."""
    v = np.asarray(column, dtype=np.float64)
    kind = fam["family"]
    if kind == "gaussian":
        if not np.isfinite(v).all():
            raise OracleSupportError(f"variable {var}: non-finite value")
        return
    top = int(fam["num_states"]) - 1 if kind == "categorical" else int(fam["n_trials"])
    ok = (v >= 0) & (v <= top) & (v == np.floor(v))
    if not ok.all():
        raise OracleSupportError(f"variable {var}: value outside {{0..{top}}}")


def log_density(fam, phi_d, xcol):
    """Per-variable log density, phi_d (K, R, T), xcol (B,) -> (B, K, R).

    gaussian expfam.py:100-102 (phi = mean, second moment);
    categorical expfam.py:166-172; binomial expfam.py:231-237.
    """
    kind = fam["family"]
    xb = xcol[:, None, None]
    if kind == "gaussian":
        mean = phi_d[..., 0]
        var = phi_d[..., 1] - mean * mean
        return -0.5 * (LOG_2PI + np.log(var))[None] - (xb - mean[None]) ** 2 / (2.0 * var[None])
    if kind == "categorical":
        logp = np.log(phi_d)                               # (K, R, S)
        idx = xcol.astype(np.int64)
        return np.moveaxis(logp[..., idx], -1, 0)           # (B, K, R)
    from math import lgamma
    n = int(fam["n_trials"])
    p = phi_d[..., 0] / n
    log_h = np.array([lgamma(n + 1) - lgamma(v + 1) - lgamma(n - v + 1) for v in xcol])
    return (log_h[:, None, None] + xb * np.log(p)[None]
            + (n - xb) * np.log1p(-p)[None])


def sufficient_stats(fam, x):
    """expfam.py:92-93 / 163-164 / 228-229: (B, D) -> (B, D, T)."""
    kind = fam["family"]
    if kind == "gaussian":
        return np.stack([x, x * x], axis=-1)
    if kind == "categorical":
        s = int(fam["num_states"])
        return (x[..., None].astype(np.int64) == np.arange(s)).astype(np.float64)
    return x[..., None].astype(np.float64)


def project_phi(fam, phi):
    """expfam.py:112-115 / 184-186 / 249-251."""
    kind = fam["family"]
    if kind == "gaussian":
        mean = phi[..., 0]
        var = np.clip(phi[..., 1] - mean * mean, fam["var_min"], fam["var_max"])
        return np.stack([mean, var + mean * mean], axis=-1)
    if kind == "categorical":
        q = np.maximum(phi, fam["p_min"])
        return q / q.sum(axis=-1, keepdims=True)
    n = float(fam["n_trials"])
    p = np.clip(phi[..., 0] / n, fam["p_min"], 1.0 - fam["p_min"])
    return (p * n)[..., None]


# ----------------------------------------------------------------------------
# forward (engine.py:91-195, expfam.py:278-309)
# ----------------------------------------------------------------------------

def leaf_rows(circuit, fam, phi, x, marg_mask=None, leaf_log_offset=None):
    """Leaf-region log densities (B, n_leaf, K) -- expfam.py:278-309.

    Accumulated per leaf row directly instead of materialising E.
    """
    leaf = circuit.layers[0]
    b = x.shape[0]
    k = circuit.k
    masked = np.zeros(circuit.d_vars, dtype=bool) if marg_mask is None \
        else np.asarray(marg_mask, dtype=bool)
    out = np.zeros((b, len(leaf.region_ids), k))
    for d in range(circuit.d_vars):           # support check order: ascending d
        if not masked[d]:
            check_support(fam, x[:, d], d)
    for li, (scope, rep) in enumerate(zip(leaf.scopes, leaf.replica)):
        acc = np.zeros((b, k))
        for d in scope:
            if masked[d]:
                continue
            acc += log_density(fam, phi[d], x[:, d])[:, :, int(rep)]
            if leaf_log_offset is not None:
                acc += np.asarray(leaf_log_offset)[d, :, int(rep)][None]
        out[:, li, :] = acc
    return out


def log_einsum_exp(left, right, w):
    """engine.py:91-109: log sum_ij w[l,k,i,j] e^left[..,l,i] e^right[..,l,j]."""
    left = np.asarray(left, dtype=np.float64)
    right = np.asarray(right, dtype=np.float64)
    a = left.max(axis=-1, keepdims=True)
    c = right.max(axis=-1, keepdims=True)
    fa, fc = np.isfinite(a), np.isfinite(c)
    ea = np.where(fa, np.exp(left - np.where(fa, a, 0.0)), 0.0)
    ec = np.where(fc, np.exp(right - np.where(fc, c, 0.0)), 0.0)
    r = np.einsum("...li,lkij,...lj->...lk", ea, w, ec)
    good = fa & fc & (r > 0)
    with np.errstate(divide="ignore"):
        return np.where(good, a + c + np.log(np.where(good, r, 1.0)), -np.inf)


def mixing_forward(vals, w, mask):
    """engine.py:112-122: masked log-sum-exp over Dmax children."""
    v = np.where(mask[None, :, :, None], vals, -np.inf)
    top = v.max(axis=2)
    fin = np.isfinite(top)
    e = np.where(fin[:, :, None, :], np.exp(v - np.where(fin, top, 0.0)[:, :, None, :]), 0.0)
    s = np.einsum("mc,bmck->bmk", w, e)
    with np.errstate(divide="ignore"):
        return np.where(fin & (s > 0), top + np.log(np.where(s > 0, s, 1.0)), -np.inf)


def forward(circuit, params, fam, x, marg_mask=None, leaf_log_offset=None):
    """engine.py:143-195."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    if x.shape[1] != circuit.d_vars:
        raise ValueError("batch width does not match the circuit")
    b = x.shape[0]
    buf = np.zeros((b, circuit.num_buffer_rows, circuit.k))
    lr = leaf_rows(circuit, fam, params.phi, x, marg_mask, leaf_log_offset)
    buf[:, circuit.layers[0].out_rows, :] = lr
    outs = [lr]
    for i, layer in enumerate(circuit.layers[1:], start=1):
        if _kind(layer) == "einsum":
            ln, rn = buf[:, layer.left_src, :], buf[:, layer.right_src, :]
            if np.isnan(ln).any() or np.isnan(rn).any():
                raise RuntimeError(f"NaN entering einsum layer {i}")
            o = log_einsum_exp(ln, rn, params.einsum[i])
        else:
            o = mixing_forward(outs[i - 1][:, layer.src, :], params.mixing[i], layer.mask)
        if not layer.is_root:
            buf[:, layer.out_rows, :] = o
        outs.append(o)
    last = circuit.layers[-1]
    if _kind(last) == "mixing":
        root = outs[-1][:, last.region_ids.index(circuit.rg.root), :]
    else:
        root = outs[-1][:, 0, :]
    return OracleTrace(buffer=buf, outputs=outs, root=root, x=x,
                       marg_mask=None if marg_mask is None else np.asarray(marg_mask, bool))


# ----------------------------------------------------------------------------
# backward (engine.py:218-328)
# ----------------------------------------------------------------------------

def zero_stats(circuit, params, fam):
    """engine.py:239-244."""
    shape = params.phi.shape[:3]
    return OracleStats(einsum={i: np.zeros_like(w) for i, w in params.einsum.items()},
                       mixing={i: np.zeros_like(w) for i, w in params.mixing.items()},
                       acc_p=np.zeros(shape), acc_pt=np.zeros(shape + (suff_dim(fam),)))


def backward(circuit, params, fam, trace):
    """Explicit responsibility back-pass, engine.py:247-328."""
    stats = zero_stats(circuit, params, fam)
    b = trace.x.shape[0]
    stats.n_samples = b
    stats.ll_sum = float(trace.root[:, 0].sum()) if trace.root.shape[1] == 1 else 0.0
    buf = trace.buffer
    resp = np.zeros((b, circuit.num_buffer_rows, circuit.k))
    pending_root = {}
    layers = circuit.layers
    for i in range(len(layers) - 1, 0, -1):
        layer = layers[i]
        out = trace.outputs[i]
        if _kind(layer) == "mixing":                         # engine.py:268-293
            if layer.is_root:
                rho = np.zeros_like(out)
                rho[:, layer.region_ids.index(circuit.rg.root), :] = 1.0
            else:
                rho = resp[:, layer.out_rows, :]
            w = params.mixing[i]
            prev = trace.outputs[i - 1]
            delta = prev[:, layer.src, :] - out[:, :, None, :]
            keep = np.isfinite(delta) & layer.mask[None, :, :, None]
            ratio = np.where(keep, np.exp(np.where(keep, delta, 0.0)), 0.0)
            share = rho[:, :, None, :] * w[None, :, :, None] * ratio
            stats.mixing[i] = stats.mixing[i] + share.sum(axis=(0, 3))
            prev_rho = np.zeros_like(prev)
            ms, cs = np.nonzero(layer.mask)
            for m, c in zip(ms, cs):
                prev_rho[:, layer.src[m, c], :] += share[:, m, c, :]
            if layers[i - 1].is_root:
                pending_root[i - 1] = prev_rho
            else:
                resp[:, layers[i - 1].out_rows, :] += prev_rho
            continue
        # einsum branch, engine.py:294-316
        if layer.is_root:
            rho = pending_root.get(i, np.ones_like(out))
        else:
            rho = resp[:, layer.out_rows, :]
        w = params.einsum[i]
        ln, rn = buf[:, layer.left_src, :], buf[:, layer.right_src, :]
        a = ln.max(axis=-1, keepdims=True)
        c = rn.max(axis=-1, keepdims=True)
        fa, fc = np.isfinite(a), np.isfinite(c)
        ea = np.where(fa, np.exp(ln - np.where(fa, a, 0.0)), 0.0)
        ec = np.where(fc, np.exp(rn - np.where(fc, c, 0.0)), 0.0)
        r = np.where(np.isfinite(out), np.exp(out - a - c), 0.0)
        rho_t = np.where(r > 0, rho / np.where(r > 0, r, 1.0), 0.0)
        stats.einsum[i] = stats.einsum[i] + np.einsum("blk,bli,blj->lkij", rho_t, ea, ec) * w
        u = np.einsum("blk,lkij->blij", rho_t, w)
        left_c = ea * np.einsum("blij,blj->bli", u, ec)
        right_c = ec * np.einsum("blij,bli->blj", u, ea)
        np.add.at(resp, (slice(None), layer.left_src), left_c)
        np.add.at(resp, (slice(None), layer.right_src), right_c)
    # leaf statistics, engine.py:318-327
    leaf = layers[0]
    rho_leaf = resp[:, leaf.out_rows, :]
    t = sufficient_stats(fam, trace.x)
    masked = trace.marg_mask
    for li, (scope, rep) in enumerate(zip(leaf.scopes, leaf.replica)):
        rho = rho_leaf[:, li, :]
        mass = rho.sum(axis=0)
        sel = np.asarray(scope, dtype=np.int64)
        stats.acc_p[sel, :, int(rep)] += mass[None, :]
        if masked is not None:
            sel = sel[~masked[sel]]
        if len(sel):
            stats.acc_pt[sel, :, int(rep), :] += np.einsum("bk,bdt->dkt", rho, t[:, sel, :])
    return stats


# ----------------------------------------------------------------------------
# M-step (trainer.py:69-124, engine.py:46-54)
# ----------------------------------------------------------------------------

def project_einsum(w, eps_w=EPS_W):
    """engine.py:46-49."""
    w = np.maximum(w, eps_w)
    return w / w.sum(axis=(2, 3), keepdims=True)


def project_mixing(w, mask, eps_w=EPS_W):
    """engine.py:52-54."""
    w = np.where(mask, np.maximum(w, eps_w), 0.0)
    return w / w.sum(axis=1, keepdims=True)


def mstep_targets(params, stats):
    """trainer.py:69-86."""
    wt = {}
    for i, n in stats.einsum.items():
        den = n.sum(axis=(2, 3), keepdims=True)
        wt[i] = np.where(den > 0, n / np.where(den > 0, den, 1.0), params.einsum[i])
    mt = {}
    for i, n in stats.mixing.items():
        den = n.sum(axis=1, keepdims=True)
        mt[i] = np.where(den > 0, n / np.where(den > 0, den, 1.0), params.mixing[i])
    keep = stats.acc_p <= EPS_COUNT
    den = np.where(keep, 1.0, stats.acc_p)
    pt = np.where(keep[..., None], params.phi, stats.acc_pt / den[..., None])
    return wt, mt, pt


def apply_update(circuit, params, fam, stats, lam, eps_w=EPS_W):
    """Gliding average + projection, trainer.py:107-116 and 89-96."""
    if lam == 0.0:
        return params.copy()
    wt, mt, pt = mstep_targets(params, stats)
    new = params.copy()
    for i in new.einsum:
        new.einsum[i] = project_einsum((1.0 - lam) * params.einsum[i] + lam * wt[i], eps_w)
    for i in new.mixing:
        new.mixing[i] = project_mixing((1.0 - lam) * params.mixing[i] + lam * mt[i],
                                       circuit.layers[i].mask, eps_w)
    new.phi = project_phi(fam, (1.0 - lam) * params.phi + lam * pt)
    return new


def em_step(circuit, params, fam, batch, lam, eps_w=EPS_W, chunk=4096):
    """trainer.py:57-66 + 99-117: returns (pre-update mean LL, new params)."""
    batch = np.atleast_2d(np.asarray(batch, dtype=np.float64))
    stats = None
    for lo in range(0, len(batch), chunk):
        tr = forward(circuit, params, fam, batch[lo:lo + chunk])
        part = backward(circuit, params, fam, tr)
        stats = part if stats is None else stats.merge(part)
    mean_ll = stats.ll_sum / len(batch)
    return mean_ll, apply_update(circuit, params, fam, stats, lam, eps_w)


# ----------------------------------------------------------------------------
# parameter init (engine.py:57-73, expfam.py:135-145, 206-208, 267-269)
# ----------------------------------------------------------------------------

def init_params(circuit, fam, seed=0, data=None, eps_w=EPS_W):
    """Seeded init in the reference's RNG call order (used by fixtures)."""
    rng = np.random.default_rng(seed)
    ein, mix = {}, {}
    for i, layer in enumerate(circuit.layers):
        kind = _kind(layer)
        if kind == "einsum":
            w = rng.random((len(layer.left_src), layer.k_out, circuit.k, circuit.k))
            ein[i] = project_einsum(w, eps_w)
        elif kind == "mixing":
            mix[i] = project_mixing(rng.random(layer.src.shape), layer.mask, eps_w)
    shape = (circuit.d_vars, circuit.k, circuit.num_replicas)
    kind = fam["family"]
    if kind == "gaussian":
        if data is not None and len(data):
            lo = np.min(data, axis=0)[:, None, None]
            hi = np.max(data, axis=0)[:, None, None]
        else:
            lo, hi = 0.0, 1.0
        mean = lo + (hi - lo) * rng.random(shape)
        phi = project_phi(fam, np.stack([mean, 1.0 + mean * mean], axis=-1))
    elif kind == "categorical":
        phi = project_phi(fam, rng.dirichlet(np.ones(int(fam["num_states"])), size=shape))
    else:
        p = 0.25 + 0.5 * rng.random(shape)
        phi = project_phi(fam, (p * float(fam["n_trials"]))[..., None])
    return OracleParams(einsum=ein, mixing=mix, phi=phi)


# ----------------------------------------------------------------------------
# sampling (engine.py:331-423) with the device's Philox4x32-10 uniforms
# ----------------------------------------------------------------------------
# The reference draws from per-sample numpy generators; the device kernels
# (paper_2004_06231_b200/csrc/sample.cu) use a counter-based Philox4x32-10
# stream keyed by (seed, sample b, decision site). This restatement performs
# the reference descent (_descend: mixing draw, einsum (i, j) draw over the
# flattened K x K weights, leaf draws) with those uniforms, so device samples
# can be checked draw for draw; the reference's own sampler is matched
# statistically (tests/golden/sampling.npz).

_PHILOX_M0, _PHILOX_M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_PHILOX_W0, _PHILOX_W1 = 0x9E3779B9, 0xBB67AE85


def philox4x32_10(ctr, key):
    """ctr (N, 4) uint32, key (k0, k1) -> (N, 4) uint32 (Random123 Philox4x32-10)."""
    c = [np.asarray(ctr[:, i], dtype=np.uint64) for i in range(4)]
    k0, k1 = int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF
    mask = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = _PHILOX_M0 * c[0]
        p1 = _PHILOX_M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & mask
        hi1, lo1 = p1 >> np.uint64(32), p1 & mask
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
        k0 = (k0 + _PHILOX_W0) & 0xFFFFFFFF
        k1 = (k1 + _PHILOX_W1) & 0xFFFFFFFF
    return np.stack(c, axis=1).astype(np.uint64)


def philox_uniforms(seed, b, site):
    """(u0, u1) in [0, 1) with 53 bits each for samples b (array) at one site."""
    b = np.asarray(b, dtype=np.uint64)
    ctr = np.stack([b & np.uint64(0xFFFFFFFF), b >> np.uint64(32),
                    np.full_like(b, np.uint64(site)), np.zeros_like(b)], axis=1)
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    r = philox4x32_10(ctr, (seed & 0xFFFFFFFF, seed >> 32))
    u0 = ((r[:, 0] >> np.uint64(5)).astype(np.float64) * 67108864.0 +
          (r[:, 1] >> np.uint64(6)).astype(np.float64)) / 9007199254740992.0
    u1 = ((r[:, 2] >> np.uint64(5)).astype(np.float64) * 67108864.0 +
          (r[:, 3] >> np.uint64(6)).astype(np.float64)) / 9007199254740992.0
    return u0, u1


def slab_ids(circuit):
    """Slab of every (layer, row) output, numbered like the device plan
    (csrc/abi.cu build_plan): buffer rows first, then the unbuffered outputs
    (out_rows == -1) in layer order."""
    nxt = circuit.num_buffer_rows
    out = {}
    for i, layer in enumerate(circuit.layers[1:], start=1):
        ids = []
        for o in np.asarray(layer.out_rows):
            if o >= 0:
                ids.append(int(o))
            else:
                ids.append(nxt)
                nxt += 1
        out[i] = ids
    return out, nxt


def sample_philox(circuit, params, fam, n, seed=0, x_e=None, evidence=None, trace=None):
    """Ancestral / conditional samples (engine.py:339-423) drawn with the
    device uniforms; ``trace`` = ``forward`` of x_e with the evidence-
    marginalised mask for conditional sampling."""
    slabs, num_slabs = slab_ids(circuit)
    layers = circuit.layers
    k_sel = np.full((num_slabs, n), -1, dtype=np.int64)
    last = len(layers) - 1
    if _kind(layers[last]) == "mixing":
        root_slab = slabs[last][list(layers[last].region_ids).index(circuit.rg.root)]
    else:
        root_slab = slabs[last][0]
    k_sel[root_slab, :] = 0
    bidx = np.arange(n)
    for i in range(last, 0, -1):
        layer = layers[i]
        for row, os in enumerate(slabs[i]):
            active = np.nonzero(k_sel[os] >= 0)[0]
            if active.size == 0:
                continue
            u0, _ = philox_uniforms(seed, bidx[active], os)
            for t, b in enumerate(active):
                k = int(k_sel[os, b])
                if _kind(layer) == "einsum":
                    w = params.einsum[i][row, k]
                    if trace is not None:
                        log_n = trace.buffer[0, layer.left_src[row], :]
                        log_np = trace.buffer[0, layer.right_src[row], :]
                        log_s = trace.outputs[i][0, row, k]
                        w = w * np.exp(log_n[:, None] + log_np[None, :] - log_s)
                    c = np.cumsum(w.ravel())
                    if c[-1] <= 0.0:
                        raise RuntimeError("cannot sample from an all-zero weight vector")
                    idx = int(np.searchsorted(c, u0[t] * c[-1], side="right"))
                    idx = min(idx, c.size - 1)
                    ii, jj = divmod(idx, circuit.k)
                    k_sel[layer.left_src[row], b] = ii
                    k_sel[layer.right_src[row], b] = jj
                else:
                    w = np.where(layer.mask[row], params.mixing[i][row], 0.0)
                    if trace is not None:
                        prev = trace.outputs[i - 1]
                        diff = prev[0, layer.src[row], k] - trace.outputs[i][0, row, k]
                        ok = layer.mask[row] & np.isfinite(diff)
                        w = w * np.where(ok, np.exp(np.where(ok, diff, 0.0)), 0.0)
                    c = np.cumsum(w)
                    if c[-1] <= 0.0:
                        raise RuntimeError("cannot sample from an all-zero weight vector")
                    ci = min(int(np.searchsorted(c, u0[t] * c[-1], side="right")), c.size - 1)
                    src_slab = slabs[i - 1][int(layer.src[row, ci])]
                    k_sel[src_slab, b] = k
    leaf = layers[0]
    d_vars = circuit.d_vars
    out = np.full((n, d_vars), np.nan)
    ev = set() if evidence is None else set(evidence)
    for li, scope in enumerate(leaf.scopes):
        slab = int(leaf.out_rows[li])
        rep = int(leaf.replica[li])
        active = np.nonzero(k_sel[slab] >= 0)[0]
        for dv in scope:
            if dv in ev:
                out[active, dv] = x_e[dv]
                continue
            u0, u1 = philox_uniforms(seed, bidx[active], num_slabs + dv)
            for t, b in enumerate(active):
                phi = params.phi[dv, int(k_sel[slab, b]), rep]
                if fam["family"] == "gaussian":
                    mu, var = phi[0], phi[1] - phi[0] * phi[0]
                    z = math.sqrt(-2.0 * math.log(1.0 - u0[t])) * math.cos(
                        6.283185307179586 * u1[t])
                    out[b, dv] = mu + math.sqrt(var) * z
                elif fam["family"] == "categorical":
                    c = np.cumsum(phi)
                    out[b, dv] = min(int(np.searchsorted(c, u0[t] * c[-1], side="right")),
                                     c.size - 1)
                else:
                    nt = int(fam["n_trials"])
                    pr = phi[0] / nt
                    acc, pick = 0.0, nt
                    for xv in range(nt + 1):
                        acc += math.exp(math.lgamma(nt + 1.0) - math.lgamma(xv + 1.0) -
                                        math.lgamma(nt - xv + 1.0) + xv * math.log(pr) +
                                        (nt - xv) * math.log1p(-pr))
                        if acc > u0[t]:
                            pick = xv
                            break
                    out[b, dv] = pick
    return out
