"""Device-resident Einsum-Network engine: the drop-in for the reference
``engine.py`` (forward, backward, log_einsum_exp, parameters, statistics).

Every batch-level computation runs in ``libeinet_b200.so`` (hand-written
sm_100a CUDA behind the C ABI of ``include/einet_b200.h``); this module only
marshals plans, buffers and error words. There is no CPU fallback.

Layouts at this boundary are the reference's: einsum weights ``(L, K_out, K,
K)``, mixing weights ``(M, Dmax)``, leaf ``phi (D, K, R, T)`` and the matching
``BackwardStats``. Internally the master parameters and the statistics are
single fp64 device buffers (the statistics buffer is the unit of the
multi-GPU all-reduce); the kernels read fp32 compute copies derived from
them.
"""

from __future__ import annotations

import ctypes
from ctypes import byref, c_void_p
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .expfam import UnsupportedValueError

EPS_W = 1e-12


class EngineError(RuntimeError):
    pass


class EvidenceError(ValueError):
    """The supplied evidence has probability zero under the model."""


def _kind(layer) -> str:
    name = type(layer).__name__
    if name == "LeafLayer":
        return "leaf"
    if name == "EinsumLayer":
        return "einsum"
    if name == "MixingLayer":
        return "mixing"
    raise TypeError(f"unknown layer type {name}")


def _stream():
    return c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor):
    return c_void_p(t.data_ptr()) if t is not None else None


# ---------------------------------------------------------------------------
# parameter layout (same element order as the C++ plan)
# ---------------------------------------------------------------------------

@dataclass
class _Layout:
    einsum: dict            # layer index -> (offset, shape)
    mixing: dict            # layer index -> (offset, shape, mask)
    phi_offset: int
    phi_shape: tuple
    total: int
    n_w: int
    n_mix: int
    n_leaf: int
    k: int

    @staticmethod
    def of(circuit, family) -> "_Layout":
        k = circuit.k
        off = 0
        ein, mix = {}, {}
        for i, layer in enumerate(circuit.layers):
            if _kind(layer) == "einsum":
                shape = (len(layer.left_src), layer.k_out, k, k)
                ein[i] = (off, shape)
                off += int(np.prod(shape))
        n_w = off
        for i, layer in enumerate(circuit.layers):
            if _kind(layer) == "mixing":
                shape = tuple(layer.src.shape)
                mix[i] = (off, shape, np.asarray(layer.mask, dtype=bool))
                off += int(np.prod(shape))
        n_mix = off - n_w
        phi_shape = (circuit.d_vars, k, circuit.num_replicas, family.suff_dim)
        phi_off = off
        off += int(np.prod(phi_shape))
        return _Layout(ein, mix, phi_off, phi_shape, off, n_w, n_mix,
                       len(circuit.layers[0].region_ids), k)


# ---------------------------------------------------------------------------
# native plan
# ---------------------------------------------------------------------------

def _family_fields(family):
    doc = family.to_dict()
    fid = _native.FAMILY_IDS[doc["family"]]
    return (fid, int(doc.get("num_states", 0)), int(doc.get("n_trials", 0)),
            float(doc.get("var_min", 0.0)), float(getattr(family, "var_max", 0.0)),
            float(doc.get("p_min", 0.0)))


class _Engine:
    """One ``einet_plan`` for (circuit, family, max_chunk)."""

    def __init__(self, circuit, family, max_chunk: int):
        lib = _native.require_cuda()
        torch.cuda.init()
        self.circuit = circuit
        self.family = family
        self.max_chunk = int(max_chunk)
        keep = []

        def arr(values, dtype=np.int32):
            a = np.ascontiguousarray(np.asarray(values), dtype=dtype)
            if a.size == 0:
                a = np.zeros(1, dtype=dtype)
            keep.append(a)
            ctype = ctypes.c_uint8 if dtype == np.uint8 else ctypes.c_int32
            return a.ctypes.data_as(ctypes.POINTER(ctype))

        leaf = circuit.layers[0]
        offsets = np.zeros(len(leaf.scopes) + 1, dtype=np.int64)
        offsets[1:] = np.cumsum([len(s) for s in leaf.scopes])
        flat_vars = [v for s in leaf.scopes for v in s]
        layers = circuit.layers[1:]
        descs = (_native.LayerDesc * len(layers))()
        root_mix_row = -1
        for n, layer in enumerate(layers):
            d = descs[n]
            if _kind(layer) == "einsum":
                d.kind = _native.LAYER_EINSUM
                d.rows = len(layer.left_src)
                d.left = arr(layer.left_src)
                d.right = arr(layer.right_src)
                d.dmax = 0
                d.src = arr([0])
                d.mask = arr([0], np.uint8)
            else:
                d.kind = _native.LAYER_MIXING
                d.rows = int(layer.src.shape[0])
                d.dmax = int(layer.src.shape[1])
                d.src = arr(np.asarray(layer.src).ravel())
                d.mask = arr(np.asarray(layer.mask).ravel(), np.uint8)
                d.left = arr([0])
                d.right = arr([0])
                if layer.is_root:
                    root_mix_row = list(layer.region_ids).index(circuit.rg.root)
            d.k_out = int(layer.k_out)
            d.is_root = int(bool(layer.is_root))
            d.out_rows = arr(layer.out_rows)
        fid, ns, nt, vmin, vmax, pmin = _family_fields(family)
        desc = _native.PlanDesc(
            d_vars=circuit.d_vars, k=circuit.k, k_root=circuit.k_root,
            num_replicas=circuit.num_replicas, num_buffer_rows=circuit.num_buffer_rows,
            family=fid, num_states=ns, n_trials=nt, var_min=vmin,
            var_max=min(vmax, 1e308), p_min=pmin, n_leaf=len(leaf.region_ids),
            leaf_scope_offsets=arr(offsets), leaf_scope_vars=arr(flat_vars),
            leaf_replica=arr(leaf.replica), leaf_out_rows=arr(leaf.out_rows),
            n_layers=len(layers), layers=descs, root_mix_row=root_mix_row)
        handle = c_void_p()
        _native.check(lib.einet_plan_create(byref(desc), self.max_chunk, byref(handle)),
                      "einet_plan_create")
        self.handle = handle
        self._lib = lib
        sizes = _native.Sizes()
        _native.check(lib.einet_plan_sizes(handle, byref(sizes)), "einet_plan_sizes")
        self.sizes = sizes
        self.layout = _Layout.of(circuit, family)
        if self.layout.total != sizes.params_f64:
            raise RuntimeError("parameter layout mismatch between host and native plan")
        self.device = torch.device("cuda", torch.cuda.current_device())

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                if torch.cuda.is_current_stream_capturing():
                    # the garbage collector may run inside a CUDA graph capture;
                    # cudaFree there would invalidate the capture
                    _DEFERRED_PLANS.append((self._lib, h))
                else:
                    self._lib.einet_plan_destroy(h)
            except Exception:
                pass

    def set_tensor_cores(self, enabled: bool):
        """Route eligible EinsumLayers to the tcgen05 kernels (default) or not."""
        _native.check(self._lib.einet_plan_set_tensor_cores(self.handle, 1 if enabled else 0),
                      "einet_plan_set_tensor_cores")

    # -- buffers ---------------------------------------------------------
    def new_workspace(self):
        return torch.empty(int(self.sizes.workspace_bytes), dtype=torch.uint8,
                           device=self.device)

    def new_stats(self):
        return torch.zeros(int(self.sizes.stats_f64), dtype=torch.float64, device=self.device)

    def new_status(self):
        st = torch.empty(_native.STATUS_WORDS, dtype=torch.int32, device=self.device)
        self.status_reset(st)
        return st

    # -- thin wrappers -----------------------------------------------------
    def log_step(self, stats, status, log_ll, log_st, cursor):
        """Row ``cursor`` of the step logs <- (LL sum, count) and the status
        words; the device cursor advances (``einet_log_step``)."""
        off = int(self.sizes.stats_ll_offset)
        _native.check(self._lib.einet_log_step(c_void_p(stats.data_ptr() + 8 * off), _ptr(status),
                                               _ptr(log_ll),
                                               _ptr(log_st), _ptr(cursor), log_ll.shape[0],
                                               _stream()), "einet_log_step")

    def status_reset(self, status):
        _native.check(self._lib.einet_status_reset(_ptr(status), _stream()),
                      "einet_status_reset")

    def status_to_stats(self, status, stats):
        """stats[ll+2] = this rank's failure flag (enqueue after the last backward)."""
        _native.check(self._lib.einet_status_to_stats(self.handle, _ptr(status), _ptr(stats),
                                                      _stream()), "einet_status_to_stats")

    def status_from_stats(self, stats, status):
        """After the all-reduce: status word 3 = 0 when any rank failed."""
        _native.check(self._lib.einet_status_from_stats(self.handle, _ptr(stats), _ptr(status),
                                                        _stream()), "einet_status_from_stats")

    def prepare(self, flat, compute, mask=None, offset=None):
        _native.check(self._lib.einet_prepare(self.handle, _ptr(flat), _ptr(compute),
                                              _ptr(mask), _ptr(offset), _stream()),
                      "einet_prepare")

    def forward(self, compute, x, batch, ws, root, status):
        _native.check(self._lib.einet_forward(self.handle, _ptr(compute), _ptr(x), int(batch),
                                              _ptr(ws), _ptr(root), _ptr(status), _stream()),
                      "einet_forward")

    def backward(self, flat, compute, x, batch, ws, stats, status):
        _native.check(self._lib.einet_backward(self.handle, _ptr(flat), _ptr(compute), _ptr(x),
                                               int(batch), _ptr(ws), _ptr(stats),
                                               _ptr(status), _stream()),
                      "einet_backward")

    def mstep(self, flat, compute, stats, lam, eps_w, status):
        _native.check(self._lib.einet_mstep(self.handle, _ptr(flat), _ptr(compute), _ptr(stats),
                                            float(lam), float(eps_w), _ptr(status), _stream()),
                      "einet_mstep")


def _bucket(batch: int) -> int:
    b = 256
    while b < batch:
        b *= 2
    return b


_DEFERRED_PLANS = []


def _release_deferred_plans():
    """Destroy plans whose owners were collected during a graph capture."""
    if _DEFERRED_PLANS and not torch.cuda.is_current_stream_capturing():
        while _DEFERRED_PLANS:
            lib, h = _DEFERRED_PLANS.pop()
            lib.einet_plan_destroy(h)


def get_engine(circuit, family, batch: int = 256) -> _Engine:
    """Cached native plan whose max_chunk covers ``batch``."""
    _release_deferred_plans()
    cache = circuit.__dict__.setdefault("_einet_b200_engines", {})
    key = (family.key(), _bucket(max(int(batch), 1)))
    eng = cache.get(key)
    if eng is None:
        eng = _Engine(circuit, family, key[1])
        cache[key] = eng
    return eng


def raise_status(status: torch.Tensor, family):
    """Map the device status words to the reference exceptions (syncs)."""
    words = status.cpu().tolist()
    _raise_words(words, family)


def _raise_words(words, family):
    if words[0] != _native.STATUS_NONE:
        var = int(words[0])
        if family.name == "gaussian":
            raise UnsupportedValueError(f"variable {var}: non-finite value")
        top = family.num_states - 1 if family.name == "categorical" else family.n_trials
        raise UnsupportedValueError(f"variable {var}: value outside {{0..{top}}}")
    if words[1] != _native.STATUS_NONE:
        raise EngineError(f"NaN entering einsum layer {int(words[1])}")


# ---------------------------------------------------------------------------
# parameters
# ---------------------------------------------------------------------------

class _ParamDict:
    """dict-like view of the einsum or mixing weights; item reads return host
    copies, item assignment uploads (reference code rebinds entries)."""

    def __init__(self, params, which):
        self._p = params
        self._which = which

    def _table(self):
        return self._p._layout.einsum if self._which == "einsum" else self._p._layout.mixing

    def __getitem__(self, i):
        off, shape = self._table()[i][:2]
        n = int(np.prod(shape))
        return self._p.flat[off:off + n].view(shape).cpu().numpy()

    def __setitem__(self, i, value):
        off, shape = self._table()[i][:2]
        v = np.asarray(value, dtype=np.float64)
        if v.shape != tuple(shape):
            raise ValueError(f"{self._which}[{i}] expects shape {shape}, got {v.shape}")
        n = int(np.prod(shape))
        self._p.flat[off:off + n].copy_(torch.from_numpy(np.ascontiguousarray(v).ravel()))
        self._p.touch()

    def keys(self):
        return list(self._table().keys())

    def __iter__(self):
        return iter(self.keys())

    def __len__(self):
        return len(self._table())

    def __contains__(self, i):
        return i in self._table()

    def items(self):
        return [(i, self[i]) for i in self.keys()]

    def values(self):
        return [self[i] for i in self.keys()]


class Parameters:
    """All trainable tensors of one circuit (reference ``engine.py:31-43``),
    held as one fp64 device buffer in the reference layouts."""

    def __init__(self, layout: _Layout, flat: torch.Tensor):
        self._layout = layout
        self.flat = flat
        self.version = 0
        self._compute = None
        self._compute_version = -1
        self._compute_owner = None

    # reference-compatible views
    @property
    def einsum(self):
        return _ParamDict(self, "einsum")

    @property
    def mixing(self):
        return _ParamDict(self, "mixing")

    @property
    def phi(self):
        n = int(np.prod(self._layout.phi_shape))
        o = self._layout.phi_offset
        return self.flat[o:o + n].view(self._layout.phi_shape).cpu().numpy()

    @phi.setter
    def phi(self, value):
        v = np.asarray(value, dtype=np.float64)
        if v.shape != tuple(self._layout.phi_shape):
            raise EngineError("leaf parameter tensor does not match the circuit")
        n = v.size
        o = self._layout.phi_offset
        self.flat[o:o + n].copy_(torch.from_numpy(np.ascontiguousarray(v).ravel()))
        self.touch()

    def touch(self):
        """Mark the device compute copies stale after a parameter change."""
        self.version += 1

    def copy(self):
        p = Parameters(self._layout, self.flat.clone())
        return p

    def to_numpy(self):
        return ({i: self.einsum[i] for i in self.einsum},
                {i: self.mixing[i] for i in self.mixing}, self.phi)

    @staticmethod
    def from_numpy(circuit, family, einsum, mixing, phi, device=None) -> "Parameters":
        layout = _Layout.of(circuit, family)
        host = np.empty(layout.total, dtype=np.float64)
        for i, (off, shape) in layout.einsum.items():
            host[off:off + int(np.prod(shape))] = np.asarray(einsum[i], np.float64).ravel()
        for i, (off, shape, _) in layout.mixing.items():
            host[off:off + int(np.prod(shape))] = np.asarray(mixing[i], np.float64).ravel()
        phi = np.asarray(phi, dtype=np.float64)
        if phi.shape != tuple(layout.phi_shape):
            raise EngineError("leaf parameter tensor does not match the circuit")
        host[layout.phi_offset:] = phi.ravel()
        _native.require_cuda()
        dev = device or torch.device("cuda", torch.cuda.current_device())
        return Parameters(layout, torch.from_numpy(host).to(dev))

    def compute_for(self, engine: _Engine, marg_mask=None, leaf_log_offset=None):
        """Device compute tensors for a forward pass (cached when unmasked)."""
        if marg_mask is None and leaf_log_offset is None:
            if (self._compute is None or self._compute_version != self.version
                    or self._compute_owner != engine.sizes.compute_bytes):
                if self._compute is None or self._compute.numel() != engine.sizes.compute_bytes:
                    self._compute = torch.empty(int(engine.sizes.compute_bytes),
                                                dtype=torch.uint8, device=self.flat.device)
                engine.prepare(self.flat, self._compute)
                self._compute_version = self.version
                self._compute_owner = engine.sizes.compute_bytes
            return self._compute
        comp = torch.empty(int(engine.sizes.compute_bytes), dtype=torch.uint8,
                           device=self.flat.device)
        mask_t = None
        if marg_mask is not None:
            mask_t = torch.from_numpy(np.ascontiguousarray(
                np.asarray(marg_mask, dtype=bool).astype(np.uint8))).to(self.flat.device)
        off_t = None
        if leaf_log_offset is not None:
            off = np.asarray(leaf_log_offset, dtype=np.float64)
            off_t = torch.from_numpy(np.ascontiguousarray(off).ravel()).to(self.flat.device)
        engine.prepare(self.flat, comp, mask_t, off_t)
        return comp

    def mark_compute_current(self, engine):
        """The fused M-step rewrote both the master and the compute copies."""
        self.version += 1
        self._compute_version = self.version
        self._compute_owner = engine.sizes.compute_bytes


def project_einsum_weights(w, eps_w=EPS_W):
    """Floor then renormalise each (l, k) slice (``engine.py:46-49``)."""
    w = np.maximum(np.asarray(w, dtype=np.float64), eps_w)
    return w / w.sum(axis=(2, 3), keepdims=True)


def project_mixing_weights(w, mask, eps_w=EPS_W):
    """Masked floor + renormalise (``engine.py:52-54``)."""
    w = np.where(mask, np.maximum(np.asarray(w, dtype=np.float64), eps_w), 0.0)
    return w / w.sum(axis=1, keepdims=True)


def init_parameters_host(circuit, family, seed=0, data=None, eps_w=EPS_W):
    """Seeded init in the reference's RNG call order (``engine.py:57-73``):
    host-side setup returning (einsum, mixing, phi) in reference layouts."""
    rng = np.random.default_rng(seed)
    einsum, mixing = {}, {}
    for i, layer in enumerate(circuit.layers):
        kind = _kind(layer)
        if kind == "einsum":
            w = rng.random((len(layer.left_src), layer.k_out, circuit.k, circuit.k))
            einsum[i] = project_einsum_weights(w, eps_w)
        elif kind == "mixing":
            mixing[i] = project_mixing_weights(rng.random(layer.src.shape), layer.mask, eps_w)
    phi = family.init_phi((circuit.d_vars, circuit.k, circuit.num_replicas), rng, data=data)
    return einsum, mixing, phi


def init_parameters(circuit, family, seed=0, data=None, eps_w=EPS_W) -> Parameters:
    """Seeded init, uploaded once to the device."""
    einsum, mixing, phi = init_parameters_host(circuit, family, seed, data, eps_w)
    return Parameters.from_numpy(circuit, family, einsum, mixing, phi)


class AllocationTracker:
    """High-water mark of engine buffer bytes (reference ``engine.py:76-88``)."""

    def __init__(self):
        self.current = 0
        self.peak = 0

    def add(self, arr):
        n = arr.numel() * arr.element_size() if isinstance(arr, torch.Tensor) else arr.nbytes
        self.current += int(n)
        self.peak = max(self.peak, self.current)

    def reset(self):
        self.current = 0


# ---------------------------------------------------------------------------
# forward / backward
# ---------------------------------------------------------------------------

def _is_u8(x) -> bool:
    return (x.dtype == torch.uint8) if isinstance(x, torch.Tensor) else \
        (np.asarray(x).dtype == np.uint8)


def _divisor(normalize) -> float:
    """u8 payloads divide by 255 unless ``normalize`` is False (reference
    ``modelio.py:150-166``: normalisation defaults on for u8 data)."""
    return 1.0 if normalize is False else 255.0


def decode_u8(src: torch.Tensor, normalize=None, out: torch.Tensor = None) -> torch.Tensor:
    """fp32 values of a device u8 batch, decoded by the engine's kernel
    (``einet_decode_u8``): ``float(float64(v) / 255)`` with the reference's
    default normalisation, raw counts with ``normalize=False``."""
    if not (src.is_cuda and src.dtype == torch.uint8):
        raise TypeError("decode_u8 needs a CUDA uint8 tensor")
    src = src.contiguous()
    if out is None:
        out = torch.empty(src.shape, dtype=torch.float32, device=src.device)
    _native.check(_native.lib().einet_decode_u8(_ptr(src), src.numel(), _divisor(normalize),
                                                _ptr(out), _stream()), "einet_decode_u8")
    return out


_PINNED_MIN_BYTES = 1 << 22


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy. Large results come back through a pinned block
    of torch's caching host allocator (the array keeps it alive; freed blocks
    are reused), ~20x faster than a pageable copy."""
    if t.numel() * t.element_size() < _PINNED_MIN_BYTES:
        return t.cpu().numpy()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h.numpy()


def _upload(t: torch.Tensor, device) -> torch.Tensor:
    """Host tensor -> device; large pageable tensors go through a pinned
    staging block (asynchronous copy, stream ordered)."""
    if t.is_pinned() or t.numel() * t.element_size() < _PINNED_MIN_BYTES:
        return t.to(device, non_blocking=t.is_pinned())
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.to(device, non_blocking=True)


def as_device_batch(x, device=None, normalize=None) -> torch.Tensor:
    """(B, D) fp32 contiguous CUDA tensor (zero-copy for such tensors). u8
    batches (EIND1 payloads) travel as bytes and are decoded on the device."""
    if _is_u8(x):
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
        if t.dim() == 1:
            t = t[None, :]
        if not t.is_cuda:
            t = _upload(t.contiguous(), device or "cuda")
        return decode_u8(t, normalize)
    if isinstance(x, torch.Tensor):
        t = x
        if t.dim() == 1:
            t = t[None, :]
        if t.is_cuda and t.dtype == torch.float32 and t.is_contiguous():
            return t
        if not t.is_cuda:
            return _upload(t.to(torch.float32).contiguous(), device or "cuda")
        return t.to(device=device or "cuda", dtype=torch.float32).contiguous()
    a = np.asarray(x)
    if a.dtype != np.float32:
        a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a[None, :]
    if a.nbytes >= _PINNED_MIN_BYTES:
        # large batches: ATen converts fp64 -> fp32 (round to nearest, like
        # numpy's astype) on all host threads straight into a pinned block
        h = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
        h.copy_(torch.from_numpy(np.ascontiguousarray(a)))
        return h.to(device or "cuda", non_blocking=True)
    return _upload(torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)),
                   device or "cuda")


class ForwardTrace:
    """Everything one forward pass produced, resident on the device
    (reference ``engine.py:125-140``)."""

    def __init__(self, engine, workspace, root, x, batch, compute, marg_mask, status):
        self.engine = engine
        self.workspace = workspace
        self.root_device = root
        self.x_device = x
        self.batch = batch
        self.compute = compute
        self.marg_mask = None if marg_mask is None else np.asarray(marg_mask, dtype=bool)
        self.status = status

    @property
    def root(self):
        return self.root_device.cpu().numpy()

    @property
    def log_likelihood(self):
        if self.root_device.shape[1] != 1:
            raise EngineError("root vector length != 1 has no scalar density")
        return self.root_device[:, 0].cpu().numpy()

    @property
    def x(self):
        return self.x_device.double().cpu().numpy()

    @property
    def buffer(self):
        """(B, num_buffer_rows, K) log values (debug / parity export)."""
        c = self.engine.circuit
        out = torch.empty((self.batch, c.num_buffer_rows, c.k), dtype=torch.float64,
                          device=self.x_device.device)
        if self.batch and c.num_buffer_rows:
            _native.check(self.engine._lib.einet_export_buffer(
                self.engine.handle, _ptr(self.workspace), self.batch, _ptr(out), _stream()),
                "einet_export_buffer")
        return out.cpu().numpy()

    @property
    def leaf_rows(self):
        c = self.engine.circuit
        n_leaf = len(c.layers[0].region_ids)
        out = torch.empty((self.batch, n_leaf, c.k), dtype=torch.float64,
                          device=self.x_device.device)
        _native.check(self.engine._lib.einet_export_leaf_rows(
            self.engine.handle, _ptr(self.workspace), self.batch, _ptr(out), _stream()),
            "einet_export_leaf_rows")
        return out.cpu().numpy()


def _check_shapes(circuit, params, x):
    if x.shape[1] != circuit.d_vars:
        raise EngineError(
            f"batch has {x.shape[1]} variables, circuit expects {circuit.d_vars}")
    if tuple(params._layout.phi_shape[:3]) != (circuit.d_vars, circuit.k,
                                               circuit.num_replicas):
        raise EngineError("leaf parameter tensor does not match the circuit")


def forward(circuit, params: Parameters, family, x, marg_mask=None, leaf_log_offset=None,
            tracker=None, check=True) -> ForwardTrace:
    """Batched log-densities on the GPU (reference ``engine.py:143-195``)."""
    xd = as_device_batch(x)
    _check_shapes(circuit, params, xd)
    batch = xd.shape[0]
    eng = get_engine(circuit, family, batch)
    root = torch.empty((batch, circuit.k_root), dtype=torch.float64, device=xd.device)
    status = eng.new_status()
    if batch == 0:
        return ForwardTrace(eng, None, root, xd, 0, None, marg_mask, status)
    compute = params.compute_for(eng, marg_mask, leaf_log_offset)
    ws = eng.new_workspace()
    if tracker:
        tracker.add(ws)
    eng.forward(compute, xd, batch, ws, root, status)
    if check:
        raise_status(status, family)
    return ForwardTrace(eng, ws, root, xd, batch, compute, marg_mask, status)


class BackwardStats:
    """Expected statistics (reference ``engine.py:218-236``) in one fp64
    device buffer: [n_W | n_mix | acc_pt | P(n_leaf, K) | ll_sum, n]."""

    def __init__(self, engine, flat, n_samples=0):
        self.engine = engine
        self.flat = flat
        self.n_samples = int(n_samples)

    @property
    def _layout(self):
        return self.engine.layout

    @property
    def einsum(self):
        out = {}
        for i, (off, shape) in self._layout.einsum.items():
            out[i] = self.flat[off:off + int(np.prod(shape))].view(shape).cpu().numpy()
        return out

    @property
    def mixing(self):
        out = {}
        for i, (off, shape, _) in self._layout.mixing.items():
            out[i] = self.flat[off:off + int(np.prod(shape))].view(shape).cpu().numpy()
        return out

    @property
    def acc_pt(self):
        s = self.engine.sizes
        n = int(np.prod(self._layout.phi_shape))
        o = int(s.stats_acc_pt_offset)
        return self.flat[o:o + n].view(self._layout.phi_shape).cpu().numpy()

    @property
    def acc_p(self):
        shape = self._layout.phi_shape[:3]
        out = torch.empty(shape, dtype=torch.float64, device=self.flat.device)
        _native.check(self.engine._lib.einet_stats_expand_acc_p(
            self.engine.handle, _ptr(self.flat), _ptr(out), _stream()),
            "einet_stats_expand_acc_p")
        return out.cpu().numpy()

    @property
    def ll_sum(self) -> float:
        return float(self.flat[int(self.engine.sizes.stats_ll_offset)].item())

    def merge(self, other: "BackwardStats"):
        self.flat.add_(other.flat)
        self.n_samples += other.n_samples
        return self


def backward(circuit, params: Parameters, family, trace: ForwardTrace,
             tracker=None) -> BackwardStats:
    """Responsibility back-pass on the GPU (reference ``engine.py:247-328``)."""
    eng = trace.engine
    stats = eng.new_stats()
    if tracker:
        tracker.add(stats)
    if trace.batch == 0:
        return BackwardStats(eng, stats, 0)
    eng.backward(params.flat, trace.compute, trace.x_device, trace.batch, trace.workspace,
                 stats, trace.status)
    return BackwardStats(eng, stats, trace.batch)


def log_einsum_exp(log_left, log_right, w):
    """Stable contraction ``out[..., l, k] = log sum_ij w[l,k,i,j]
    exp(left[..., l, i]) exp(right[..., l, j])`` on the GPU in fp64
    (reference ``engine.py:91-109``)."""
    lib = _native.require_cuda()
    left = np.asarray(log_left, dtype=np.float64)
    right = np.asarray(log_right, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    lead = left.shape[:-2]
    L, K = left.shape[-2], left.shape[-1]
    Ko = w.shape[1]
    B = int(np.prod(lead)) if lead else 1
    dev = torch.device("cuda", torch.cuda.current_device())
    tl = torch.from_numpy(np.ascontiguousarray(left.reshape(B, L, K))).to(dev)
    tr = torch.from_numpy(np.ascontiguousarray(right.reshape(B, L, K))).to(dev)
    tw = torch.from_numpy(np.ascontiguousarray(w)).to(dev)
    out = torch.empty((B, L, Ko), dtype=torch.float64, device=dev)
    _native.check(lib.einet_log_einsum_exp(_ptr(tl), _ptr(tr), _ptr(tw), B, L, K, Ko,
                                           _ptr(out), _stream()), "einet_log_einsum_exp")
    return out.cpu().numpy().reshape(lead + (L, Ko))


def conditional_log_density(circuit, params, family, x, query, evidence):
    """log p(x_q | x_e), other variables marginalised (``engine.py:198-215``)."""
    query, evidence = set(query), set(evidence)
    if query & evidence:
        raise ValueError("query and evidence sets overlap")
    d = circuit.d_vars
    mask_num = np.array([i not in query and i not in evidence for i in range(d)])
    mask_den = np.array([i not in evidence for i in range(d)])
    xd = as_device_batch(x)  # one upload for both passes
    num = forward(circuit, params, family, xd, mask_num).log_likelihood
    den = forward(circuit, params, family, xd, mask_den).log_likelihood
    if np.any(np.isneginf(den)):
        raise EvidenceError("evidence has probability zero under the model")
    return num - den


def ef_log_prob_device(family, phi, x, marg_mask=None):
    """E (B, D, K, R) fp64 from phi (numpy or Parameters) on the GPU."""
    lib = _native.require_cuda()
    xd = as_device_batch(x)
    if isinstance(phi, Parameters):
        flat, shape = phi.flat, phi._layout.phi_shape
        base = phi._layout.phi_offset
        phi_t = flat[base:base + int(np.prod(shape))]
    else:
        arr = np.asarray(phi, dtype=np.float64)
        shape = arr.shape
        phi_t = torch.from_numpy(np.ascontiguousarray(arr).ravel()).to(xd.device)
    D, K, R = shape[:3]
    from .compiler import EinsumLayer, LayeredCircuit, LeafLayer, ReplicaAssignment
    from .structures import Partition, Region, RegionGraph
    # a one-partition scratch circuit gives the kernel its plan constants
    rg = RegionGraph(d_vars=D)
    rg.regions[0] = Region(0, frozenset(range(D)))
    circ = LayeredCircuit(rg=rg, k=K, k_root=1, layers=[
        LeafLayer([1], [list(range(D))], np.zeros(1, np.int64), np.zeros(1, np.int64)),
        EinsumLayer(np.zeros(1, np.int64), np.zeros(1, np.int64), np.array([-1]), [(0, 0)],
                    1, True)], num_buffer_rows=1, region_row={},
        replicas=ReplicaAssignment({}, R))
    eng = get_engine(circ, family, 1)
    params = torch.zeros(int(eng.sizes.params_f64), dtype=torch.float64, device=xd.device)
    params[int(eng.sizes.phi_offset):] = phi_t
    out = torch.empty((xd.shape[0], D, K, R), dtype=torch.float64, device=xd.device)
    mask_t = None
    if marg_mask is not None:
        mask_t = torch.from_numpy(np.asarray(marg_mask, dtype=np.uint8)).to(xd.device)
    status = eng.new_status()
    if xd.shape[0]:
        _native.check(lib.einet_ef_log_prob(eng.handle, _ptr(params), _ptr(xd), xd.shape[0],
                                            _ptr(mask_t), _ptr(out), _ptr(status), _stream()),
                      "einet_ef_log_prob")
    raise_status(status, family)
    return out.cpu().numpy()


def leaf_forward_device(circuit, family, phi, x, marg_mask=None, leaf_log_offset=None):
    """(leaf rows (B, n_leaf, K), E) with the production leaf kernels."""
    if isinstance(phi, Parameters):
        params = phi
    else:
        layout = _Layout.of(circuit, family)
        zeros_e = {i: np.full(s, 1.0 / (circuit.k * circuit.k)) for i, (_, s) in
                   layout.einsum.items()}
        zeros_m = {i: np.where(m, 1.0, 0.0) / np.maximum(m.sum(1, keepdims=True), 1)
                   for i, (_, s, m) in layout.mixing.items()}
        params = Parameters.from_numpy(circuit, family, zeros_e, zeros_m, phi)
    tr = forward(circuit, params, family, x, marg_mask, leaf_log_offset)
    e = ef_log_prob_device(family, params, x, marg_mask)
    if leaf_log_offset is not None:
        off = np.asarray(leaf_log_offset, dtype=np.float64)
        if marg_mask is not None:
            off = np.where(np.asarray(marg_mask)[:, None, None], 0.0, off)
        e = e + off[None]
    return tr.leaf_rows, e
