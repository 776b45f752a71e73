"""EM training on the GPU (reference ``trainer.py``).

One EM step = for each chunk: forward + responsibility back-pass (statistics
accumulate in one fp64 device buffer) -> optional all-reduce of that buffer
across ranks -> one fused M-step kernel sequence. The host synchronises once
per step, to read the log-likelihood sum and the error words.

On a single device the whole step (statistics reset, every chunk's forward and
back-pass, M-step) is captured once into a CUDA graph per (batch buffer,
shape, lambda, chunk) and replayed, removing the per-kernel launch gaps
(EINET_CUDA_GRAPHS=0 disables it).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native, engine
from .model import EinetModel

EPS_COUNT = 1e-12


class TrainingDiverged(RuntimeError):
    pass


@dataclass
class TrainerConfig:
    """Reference ``trainer.py:30-46``."""

    mode: str = "stochastic"
    step_size: float = 0.5
    batch_size: int = 500
    epochs: int = 10
    seed: int = 0
    eps_w: float = engine.EPS_W
    chunk: int = 4096

    def __post_init__(self):
        if self.mode not in ("full", "stochastic"):
            raise ValueError(f"unknown mode {self.mode!r}")
        if not 0.0 <= self.step_size <= 1.0:
            raise ValueError("step size must lie in [0, 1]")
        if self.batch_size < 1:
            raise ValueError("batch size must be >= 1")


@dataclass
class EpochMetrics:
    epoch: int
    train_ll: float
    valid_ll: float
    wall_seconds: float


def accumulate(model: EinetModel, batch: torch.Tensor, chunk: int, reset_status=True):
    """E-step over a device batch into the model's stats buffer
    (reference ``trainer.py:57-66``). Returns (engine, stats, status).
    ``reset_status=False`` keeps earlier error words (a pipelined sequence of
    steps: once a step fails, every later M-step is skipped)."""
    n = batch.shape[0]
    eng, ws, stats, status, root = model.step_buffers(min(chunk, max(n, 1)))
    compute = model.params.compute_for(eng)
    stats.zero_()  # an empty local shard contributes zero statistics
    if reset_status:
        eng.status_reset(status)
    step = eng.max_chunk if chunk >= eng.max_chunk else chunk
    for lo in range(0, n, step):
        xb = batch[lo:lo + step]
        b = xb.shape[0]
        eng.forward(compute, xb, b, ws, root, status)
        eng.backward(model.params.flat, compute, xb, b, ws, stats, status)
    return eng, stats, status, compute


_GRAPH_CACHE_SIZE = 8


def _graphs_enabled() -> bool:
    return os.environ.get("EINET_CUDA_GRAPHS", "1") != "0" and not _native.PROFILING


def _f64_batch(batch):
    """A float64 NumPy batch (the reference caller's type, trainer.py:104) as a
    C-contiguous 2-D array, else None."""
    if isinstance(batch, np.ndarray) and batch.dtype == np.float64 and batch.ndim in (1, 2):
        return np.ascontiguousarray(batch if batch.ndim == 2 else batch[None, :])
    return None


def _pack_f64(model: EinetModel, a: np.ndarray, slot: int):
    """Pack a float64 batch into the model's pinned host half ``slot`` with
    ``einet_pack_f64`` (all host threads): one byte per value when the batch
    is on the v/255 (or raw count) grid, else fp32 (the fp32 half is pinned
    on first need). Returns (pinned tensor, ``decode_u8`` normalize flag:
    None = /255, False = raw counts, or "f32" for an fp32 tensor). A half is
    repacked only after its previous copy has ended (``ent["ev"]``)."""
    import ctypes
    pool = model.__dict__.setdefault("_pin_f64", {})
    ent = pool.get(slot)
    if ent is None or ent["shape"] != a.shape:
        ent = pool[slot] = {"shape": a.shape, "f32": None, "ev": None,
                            "u8": torch.empty(a.shape, dtype=torch.uint8, pin_memory=True)}
    if ent["ev"] is not None:
        ent["ev"].synchronize()
    lib = _native.lib()
    kind = ctypes.c_int32(-1)
    for _ in range(2):
        f32 = ent["f32"]
        _native.check(lib.einet_pack_f64(a.ctypes.data, a.size, ent["u8"].data_ptr(),
                                         f32.data_ptr() if f32 is not None else None, 0,
                                         ctypes.byref(kind)), "einet_pack_f64")
        if kind.value >= 0:
            break
        ent["f32"] = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
    k = kind.value
    if k == 0:
        return ent, ent["f32"], "f32"
    return ent, ent["u8"], (None if k == 255 else False)


def _staging(model, shape, dev):
    st = model.__dict__.get("_staging")
    if st is None or st.shape != shape:
        st = torch.empty(shape, dtype=torch.float32, device=dev)
        model.__dict__["_staging"] = st
    return st


def _stage_batch(model: EinetModel, batch, normalize=None) -> torch.Tensor:
    """Device batch for the graph path. Device fp32 tensors are used in place;
    host data is copied (asynchronously when pinned) into a persistent
    per-model staging buffer, so the captured graph's input address is stable
    across steps. u8 batches travel as bytes and are decoded on the device
    into the fp32 staging buffer (``engine.decode_u8``)."""
    if isinstance(batch, torch.Tensor) and batch.is_cuda and batch.dtype != torch.uint8:
        return engine.as_device_batch(batch)
    dev = model.params.flat.device
    a = _f64_batch(batch)
    if a is not None:
        # float64 (the reference caller's type): packed on the host threads
        # into pinned memory, copied as bytes when on the u8 grid
        ent, t, norm = _pack_f64(model, a, 0)
        st = _staging(model, t.shape, dev)
        if norm == "f32":
            st.copy_(t, non_blocking=True)
        else:
            engine.decode_u8(t.to(dev, non_blocking=True), norm, out=st)
        ent["ev"] = torch.cuda.Event()
        ent["ev"].record()
        return st
    t = _host_batch(batch)
    st = _staging(model, t.shape, dev)
    if t.dtype == torch.uint8:
        if not t.is_cuda:
            t = t.to(dev, non_blocking=t.is_pinned())
        engine.decode_u8(t, normalize, out=st)
    else:
        st.copy_(t, non_blocking=t.is_pinned())
    return st


def _e_step_tail(eng, stats, status, process_group):
    """End of a data-parallel E-step: this rank's failure flag into the
    statistics buffer, so the single all-reduce also counts failing ranks."""
    if process_group is not None:
        eng.status_to_stats(status, stats)


def _reduce(eng, stats, status, process_group):
    """The one collective of a data-parallel EM update: all-reduce(sum) of the
    packed statistics buffer (reference ``BackwardStats.merge``,
    engine.py:228-236), then status word 3 from the failing-rank count."""
    if process_group is not None:
        import torch.distributed as dist
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=process_group)
        eng.status_from_stats(stats, status)


def _step_log(model: EinetModel, n: int, dev):
    """Persistent per-model step logs (LL sum and count, status words) for a
    pipelined sequence of n steps, and their device cursor reset to row 0; the
    buffers only grow, so the graphs that write them stay valid."""
    ent = model.__dict__.get("_steplog")
    if ent is None or ent[0].shape[0] < n:
        cap = max(n, 64, 2 * (ent[0].shape[0] if ent is not None else 0))
        ent = (torch.empty((cap, 2), dtype=torch.float64, device=dev),
               torch.empty((cap, _native.STATUS_WORDS), dtype=torch.int32, device=dev),
               torch.zeros(1, dtype=torch.int64, device=dev))
        model.__dict__["_steplog"] = ent
    ent[2].zero_()
    return ent


def _graph_step(model: EinetModel, xd: torch.Tensor, lam, eps_w, chunk, process_group=None,
                sticky=False, log=None):
    """Replay (capturing on first use) the CUDA graph of one EM step on the
    device batch ``xd``; returns (engine, stats, status). With a process group
    the step is two graphs (E-step, M-step) around the one all-reduce of the
    statistics buffer (outside the graphs; NCCL or gloo).
    ``sticky``: the graph does not reset the status words."""
    n = xd.shape[0]
    eng, ws, stats, status, root = model.step_buffers(min(chunk, max(n, 1)))
    compute = model.params.compute_for(eng)  # prepares outside the graph if stale
    # every buffer the graph reads or writes is part of the key
    key = (xd.data_ptr(), tuple(xd.shape), float(lam), float(eps_w), int(chunk),
           model.params.flat.data_ptr(), ws.data_ptr(), compute.data_ptr(), stats.data_ptr(),
           status.data_ptr(), root.data_ptr(), process_group is not None, bool(sticky),
           None if log is None else tuple(t.data_ptr() for t in log))
    cache = model.__dict__.setdefault("_graphs", {})
    gs = cache.get(key)
    if gs is None:
        if len(cache) >= _GRAPH_CACHE_SIZE:
            cache.pop(next(iter(cache)))
        torch.cuda.current_stream().synchronize()
        if process_group is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                accumulate(model, xd, chunk, reset_status=not sticky)
                eng.mstep(model.params.flat, compute, stats, lam, eps_w, status)
                if log is not None:
                    eng.log_step(stats, status, *log)
            gs = (g,)
        else:
            ge, gm = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(ge):
                accumulate(model, xd, chunk, reset_status=not sticky)
                _e_step_tail(eng, stats, status, process_group)
            with torch.cuda.graph(gm):
                eng.status_from_stats(stats, status)
                eng.mstep(model.params.flat, compute, stats, lam, eps_w, status)
                if log is not None:
                    eng.log_step(stats, status, *log)
            gs = (ge, gm)
        cache[key] = gs
    if process_group is None:
        gs[0].replay()
    else:
        import torch.distributed as dist
        gs[0].replay()
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=process_group)
        gs[1].replay()
    return eng, stats, status


def em_stochastic_step(model: EinetModel, batch, lam, eps_w=engine.EPS_W, chunk=4096,
                       process_group=None, normalize=None) -> float:
    """One gliding-average EM update; returns the pre-update mean LL of the
    batch (reference ``trainer.py:99-117``). ``lam == 0`` leaves every
    parameter bitwise unchanged.

    With ``process_group`` this rank's ``batch`` is its shard of the global
    batch (it may be empty): the statistics are summed across ranks by ONE
    all-reduce of the packed buffer (which also counts failing ranks), every
    rank applies the identical M-step, and the returned mean LL is the global
    one. The error words cross ranks (a MIN all-reduce) only when some rank
    failed.

    A uint8 batch (an EIND1 payload, reference ``modelio.py:145-166``) is
    copied as bytes and decoded on the device: divided by 255 unless
    ``normalize`` is False, like the reference's ``load_dataset``.
    """
    use_graph = lam != 0.0 and _graphs_enabled()
    xd = (_stage_batch(model, batch, normalize) if use_graph
          else engine.as_device_batch(batch, normalize=normalize))
    if xd.shape[0] == 0 and process_group is None:
        raise ValueError("empty batch")
    if use_graph:
        eng, stats, status = _graph_step(model, xd, lam, eps_w, chunk, process_group)
    else:
        eng, stats, status, compute = accumulate(model, xd, chunk)
        _e_step_tail(eng, stats, status, process_group)
        _reduce(eng, stats, status, process_group)
        if lam != 0.0:
            eng.mstep(model.params.flat, compute, stats, lam, eps_w, status)
    return _finish_step(model, eng, stats, status, lam, process_group)


def _cross_rank_words(words, process_group, status):
    """Exact error words of a step some rank failed (word 3 set): one MIN
    all-reduce of the status words, issued by every rank of the group (they
    all see the same failing-rank count)."""
    if process_group is None or words[3] == _native.STATUS_NONE:
        return words
    import torch.distributed as dist
    dist.all_reduce(status, op=dist.ReduceOp.MIN, group=process_group)
    return status.cpu().tolist()


def _raise_step_words(words, family):
    engine._raise_words(words, family)
    if words[3] != _native.STATUS_NONE:
        raise engine.EngineError("EM step failed on another rank")


def _finish_step(model, eng, stats, status, lam, process_group=None) -> float:
    """Read the LL sum and the error words (one device->host copy, syncs),
    raise the reference exceptions, return the mean LL."""
    ll_off = int(eng.sizes.stats_ll_offset)
    info = torch.cat([stats[ll_off:ll_off + 2], status.to(torch.float64)]).cpu().tolist()
    words = _cross_rank_words([int(v) for v in info[2:]], process_group, status)
    _raise_step_words(words, model.family)
    if info[1] == 0:
        raise ValueError("empty batch")
    if lam != 0.0:
        model.params.mark_compute_current(eng)
    return info[0] / info[1]


def _host_batch(batch) -> torch.Tensor:
    """(B, D) contiguous tensor: uint8 stays bytes, everything else fp32."""
    if isinstance(batch, torch.Tensor):
        t = batch
    elif engine._is_u8(batch):
        t = torch.from_numpy(np.ascontiguousarray(batch))
    else:
        a = np.asarray(batch)
        if a.dtype == np.float32:
            t = torch.from_numpy(np.ascontiguousarray(a))
        else:  # ATen converts on all host threads (round to nearest, as numpy)
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(torch.float32)
    if t.dim() == 1:
        t = t[None, :]
    if t.dtype not in (torch.float32, torch.uint8):
        t = t.to(torch.float32)
    return t.contiguous()


def em_stochastic_steps(model: EinetModel, batches, lam, eps_w=engine.EPS_W,
                        chunk=4096, normalize=None, process_group=None) -> list:
    """Consecutive gliding-average EM steps over a sequence of host batches of
    one shape (equivalent to calling ``em_stochastic_step`` on each): the
    host->device copy of batch i+1 runs on a copy stream into the other half
    of a double-buffered staging area while step i runs on the device, and
    the host does not wait between steps: each step's LL sum and error words
    are logged on the device and read once at the end. The error words stay
    set across the sequence, so after a failing step every later M-step is a
    no-op: the first failing step raises its reference exception with the
    parameters left as after the steps before it, as a loop of
    ``em_stochastic_step`` would. Returns the list of mean LLs. uint8 batches
    are copied as bytes and decoded on the device (see
    ``em_stochastic_step``). With an NCCL ``process_group`` each step is the
    E-step graph, the all-reduces of the statistics and error words, and the
    M-step graph, still without a host wait; the error words cross ranks
    (a MIN all-reduce of the logs) only when some rank failed."""
    batches = list(batches)
    f64 = [_f64_batch(b) for b in batches]
    # float64 NumPy batches (the reference caller's type) are packed lazily on
    # the host threads (einet_pack_f64) into two pinned halves: batch i+1 is
    # packed while step i runs, and crosses PCIe as bytes when on the grid
    f64_mode = bool(batches) and all(a is not None for a in f64) and lam != 0.0 \
        and _graphs_enabled()
    hosts = f64 if f64_mode else [_host_batch(b) for b in batches]
    if not hosts:
        return []
    if lam == 0.0 or not _graphs_enabled():
        return [em_stochastic_step(model, b, lam, eps_w, chunk, process_group=process_group,
                                   normalize=normalize) for b in hosts]
    if not f64_mode and hosts[0].is_cuda:
        return _device_steps(model, hosts, lam, eps_w, chunk, normalize, process_group)
    shape = tuple(hosts[0].shape)
    dtype = "f64" if f64_mode else hosts[0].dtype
    if shape[0] == 0 and process_group is None:
        raise ValueError("empty batch")
    dev = model.params.flat.device
    copy = model.__dict__.get("_copy_stream")
    if copy is None:
        copy = torch.cuda.Stream(device=dev)
        model.__dict__["_copy_stream"] = copy
    u8 = dtype == torch.uint8
    key = "_stage2_u8" if u8 or f64_mode else "_stage2_f32"
    bufs = model.__dict__.get(key)
    if bufs is None or tuple(bufs[0].shape) != shape:
        bufs = [torch.empty(shape, dtype=torch.uint8 if u8 or f64_mode else dtype, device=dev)
                for _ in range(2)]
        model.__dict__[key] = bufs
    dec = u8 or f64_mode
    if dec:  # u8 batches are decoded on the copy stream into their own fp32 halves
        xfs = model.__dict__.get("_stage2_dec")
        if xfs is None or tuple(xfs[0].shape) != shape:
            xfs = [torch.empty(shape, dtype=torch.float32, device=dev) for _ in range(2)]
            model.__dict__["_stage2_dec"] = xfs
    cur = torch.cuda.current_stream(dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]  # half ready for its step
    used = [torch.cuda.Event(), torch.cuda.Event()]    # step done with the half
    raw = [torch.cuda.Event(), torch.cuda.Event()]     # bytes landed (decode may start)
    dstream = model.__dict__.get("_decode_stream")
    if dec and dstream is None:
        dstream = torch.cuda.Stream(device=dev)
        model.__dict__["_decode_stream"] = dstream

    def issue_copy(i):
        # batch i into half i % 2. Byte batches: the copy stream only moves
        # bytes (the u8 half is free once batch i-2's decode has read it) and
        # the decode runs on its own stream once step i-2 is done with the fp32
        # half, so consecutive copies keep the PCIe link busy back to back.
        s = i & 1
        norm = normalize
        if f64_mode:  # host packing (waits only for this pinned half's last copy)
            ent, t, norm = _pack_f64(model, hosts[i], s)
        direct = not dec or norm == "f32"  # the copy lands where the step reads
        if i < 2:
            copy.wait_stream(cur)
        else:
            copy.wait_event(used[s] if direct else copied[s])
        with torch.cuda.stream(copy):
            if f64_mode:
                (xfs[s] if norm == "f32" else bufs[s]).copy_(t, non_blocking=True)
                ent["ev"] = torch.cuda.Event()
                ent["ev"].record(copy)
            else:
                bufs[s].copy_(hosts[i], non_blocking=hosts[i].is_pinned())
            (copied if direct else raw)[s].record(copy)
        if not direct:
            dstream.wait_event(raw[s])
            dstream.wait_stream(cur) if i < 2 else dstream.wait_event(used[s])
            with torch.cuda.stream(dstream):
                engine.decode_u8(bufs[s], norm, out=xfs[s])
                copied[s].record(dstream)

    for h in hosts:
        if tuple(h.shape) != shape or (not f64_mode and h.dtype != dtype):
            raise ValueError("em_stochastic_steps needs batches of one shape and dtype")
    # No host sync between steps: the status words stay sticky over the
    # sequence (a failed step makes every later M-step a no-op, so the
    # parameters end where the reference's exception would leave them); each
    # step's LL sum and error words go to a device log read once at the end.
    eng, ws, stats, status, root = model.step_buffers(min(chunk, shape[0]))
    log = _step_log(model, len(hosts), dev)
    eng.status_reset(status)
    issue_copy(0)
    for i in range(len(hosts)):
        s = i & 1
        cur.wait_event(copied[s])
        eng, stats, status = _graph_step(model, xfs[s] if dec else bufs[s], lam, eps_w, chunk,
                                         process_group, sticky=True, log=log)
        used[s].record(cur)
        if i + 1 < len(hosts):
            issue_copy(i + 1)
        model.params.mark_compute_current(eng)
    n = len(hosts)
    return _finish_steps(model, log[0][:n], log[1][:n], process_group)


def _finish_steps(model, log_ll, log_st, process_group):
    """Raise the first failing step's reference exception (after the steps'
    logs are read once), else return the mean LLs."""
    lls = log_ll.cpu().tolist()
    rows = log_st.cpu().tolist()
    if process_group is not None and any(r[3] != _native.STATUS_NONE for r in rows):
        import torch.distributed as dist
        dist.all_reduce(log_st, op=dist.ReduceOp.MIN, group=process_group)
        rows = log_st.cpu().tolist()
    for words in rows:
        _raise_step_words(words, model.family)
    for a, b in lls:
        if b == 0:
            raise ValueError("empty batch")
    return [a / b for a, b in lls]


def _device_steps(model, batches, lam, eps_w, chunk, normalize, process_group):
    """em_stochastic_steps over device-resident batches: fp32 batches are used
    in place (one CUDA graph per distinct buffer), u8 batches are decoded into
    the two fp32 staging halves; sticky error words and device logs as in the
    host pipeline, one host sync at the end."""
    dev = model.params.flat.device
    if not all(b.is_cuda for b in batches):
        raise ValueError("em_stochastic_steps needs all batches on the host or all on the device")
    shape = tuple(batches[0].shape)
    if shape[0] == 0 and process_group is None:
        raise ValueError("empty batch")
    if any(tuple(b.shape) != shape or b.dtype != batches[0].dtype for b in batches):
        raise ValueError("em_stochastic_steps needs batches of one shape and dtype")
    u8 = batches[0].dtype == torch.uint8
    if u8:
        xfs = model.__dict__.get("_stage2_dec")
        if xfs is None or tuple(xfs[0].shape) != shape:
            xfs = [torch.empty(shape, dtype=torch.float32, device=dev) for _ in range(2)]
            model.__dict__["_stage2_dec"] = xfs
    eng, ws, stats, status, root = model.step_buffers(min(chunk, shape[0]))
    log = _step_log(model, len(batches), dev)
    eng.status_reset(status)
    for i, b in enumerate(batches):
        if u8:
            xd = engine.decode_u8(b, normalize, out=xfs[i & 1])
        else:
            xd = engine.as_device_batch(b)
        eng, stats, status = _graph_step(model, xd, lam, eps_w, chunk, process_group,
                                         sticky=True, log=log)
        model.params.mark_compute_current(eng)
    n = len(batches)
    return _finish_steps(model, log[0][:n], log[1][:n], process_group)


def em_full_step(model: EinetModel, data, eps_w=engine.EPS_W, chunk=4096,
                 process_group=None) -> float:
    """Full-batch EM update == a lam = 1 stochastic step on all data."""
    return em_stochastic_step(model, data, lam=1.0, eps_w=eps_w, chunk=chunk,
                              process_group=process_group)


def _check_finite(model, epoch, batch_idx):
    if not bool(torch.isfinite(model.params.flat).all()):
        raise TrainingDiverged(
            f"non-finite parameters after epoch {epoch}, batch {batch_idx}")


def _enqueue_step(model: EinetModel, xd: torch.Tensor, lam, eps_w, chunk):
    """One EM step on a device batch, enqueued on the current stream without
    a host sync (the caller reads the status words later). Returns the
    device status words."""
    if lam != 0.0 and _graphs_enabled():
        eng, stats, status = _graph_step(model, xd, lam, eps_w, chunk)
    else:
        eng, stats, status, compute = accumulate(model, xd, chunk)
        if lam != 0.0:
            eng.mstep(model.params.flat, compute, stats, lam, eps_w, status)
    if lam != 0.0:
        model.params.mark_compute_current(eng)
    return status


def _ll_pass(model, eng, ws, root, status, compute, xd, out):
    eng.status_reset(status)
    step = eng.max_chunk
    for lo in range(0, xd.shape[0], step):
        b = min(step, xd.shape[0] - lo)
        eng.forward(compute, xd[lo:lo + b], b, ws, root, status)
        out[lo:lo + b].copy_(root[:b, 0])


def _enqueue_ll(model: EinetModel, xd: torch.Tensor, chunk):
    """Per-sample log-likelihoods of the device dataset on the current stream,
    in chunks of the EM step's engine (``chunk`` = the step's chunk) with its
    workspace; the chunk loop is one CUDA graph per (model, dataset).
    Returns (device LLs, device status words), both owned by the model."""
    n = xd.shape[0]
    eng, ws, stats, status, root = model.step_buffers(chunk)
    if root.shape[1] != 1:
        raise engine.EngineError("root vector length != 1 has no scalar density")
    compute = model.params.compute_for(eng)
    key = (xd.data_ptr(), tuple(xd.shape), ws.data_ptr(), compute.data_ptr(),
           model.params.flat.data_ptr())
    cache = model.__dict__.setdefault("_ll_graphs", {})
    ent = cache.get(key)
    if ent is None:
        out = torch.empty(n, dtype=torch.float64, device=xd.device)
        if not _graphs_enabled():
            _ll_pass(model, eng, ws, root, status, compute, xd, out)
            return out, status
        if len(cache) >= 4:
            cache.pop(next(iter(cache)))
        torch.cuda.current_stream().synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            _ll_pass(model, eng, ws, root, status, compute, xd, out)
        ent = cache[key] = (g, out)
    ent[0].replay()
    return ent[1], status


def _pinned(shape, dtype):
    t = torch.empty(shape, dtype=dtype)
    return t.pin_memory() if torch.cuda.is_available() else t


class _EpochPlan:
    """One model's training epoch on one device dataset as a single enqueue
    (a CUDA graph when graphs are enabled and lam != 0): for every batch the
    gather ``x[order[lo:hi]]`` from the persistent permutation buffer, the EM
    step (statistics reset, chunked forward + back-pass, M-step), a copy of
    the step's error words and the sum of the parameters (the finiteness
    check of ``_check_finite``); then the epoch log-likelihood pass. The
    host sends the epoch's permutation and reads the logs back once."""

    def __init__(self, model, xd, cfg):
        dev = xd.device
        self.full = cfg.mode == "full"
        self.n = xd.shape[0]
        self.xd = xd
        self.lam = 1.0 if self.full else cfg.step_size
        self.eps_w, self.chunk = cfg.eps_w, cfg.chunk
        self.bs = self.n if self.full else cfg.batch_size
        self.nb = -(-self.n // self.bs)
        # epoch log-likelihoods in chunks of up to cfg.chunk (the reference's
        # log_likelihood chunking), on their own engine bucket
        self.ll_chunk = min(cfg.chunk, self.n)
        self.order = None if self.full else torch.empty(self.n, dtype=torch.int64, device=dev)
        self.logs = torch.empty((self.nb, _native.STATUS_WORDS), dtype=torch.int32, device=dev)
        self.sums = torch.empty(self.nb, dtype=torch.float64, device=dev)
        self.lstat = torch.empty(_native.STATUS_WORDS, dtype=torch.int32, device=dev)
        self.stage = {}
        if not self.full:
            for b in {min(self.bs, self.n - lo) for lo in range(0, self.n, self.bs)}:
                self.stage[b] = torch.empty((b, xd.shape[1]), dtype=torch.float32, device=dev)
        self.h_perm = _pinned((self.n,), torch.int64)
        self.h_logs = _pinned(tuple(self.logs.shape), torch.int32)
        self.h_sums = _pinned((self.nb,), torch.float64)
        self.h_lstat = _pinned((_native.STATUS_WORDS,), torch.int32)
        self.h_ll = _pinned((self.n,), torch.float64)
        self.graph = None
        self.ll = None
        self.engines = []
        self.valid_host = None

    @staticmethod
    def get(model, xd, cfg):
        key = (xd.data_ptr(), tuple(xd.shape), cfg.mode, cfg.batch_size, cfg.step_size,
               cfg.eps_w, cfg.chunk, model.params.flat.data_ptr())
        cache = model.__dict__.setdefault("_epoch_plans", {})
        ep = cache.get(key)
        if ep is None:
            if len(cache) >= 2:
                cache.pop(next(iter(cache)))
            ep = cache[key] = _EpochPlan(model, xd, cfg)
        return ep

    def _body(self, model):
        for bi in range(self.nb):
            lo = bi * self.bs
            if self.full:
                xb = self.xd
            else:
                idx = self.order[lo:lo + self.bs]
                xb = self.stage[idx.shape[0]]
                torch.index_select(self.xd, 0, idx, out=xb)
            # error words are reset once per epoch (the model's one status
            # buffer): after a failing batch every later M-step is a no-op, so
            # the parameters stay as after the last good batch, where the
            # reference's exception leaves them
            eng, stats, status, compute = accumulate(model, xb, self.chunk,
                                                     reset_status=bi == 0)
            if self.lam != 0.0:
                eng.mstep(model.params.flat, compute, stats, self.lam, self.eps_w, status)
            self.logs[bi].copy_(status)
            self.sums[bi].copy_(model.params.flat.sum())
        eng, ws, stats, status, root = model.step_buffers(self.ll_chunk)
        if root.shape[1] != 1:
            raise engine.EngineError("root vector length != 1 has no scalar density")
        if self.ll is None:
            self.ll = torch.empty(self.n, dtype=torch.float64, device=self.xd.device)
        _ll_pass(model, eng, ws, root, status, model.params.compute_for(eng), self.xd, self.ll)
        self.lstat.copy_(status)
        return eng

    def run(self, model, perm):
        """Enqueue one epoch on the current stream (no host sync)."""
        if perm is not None:
            self.h_perm.copy_(torch.from_numpy(perm))
            self.order.copy_(self.h_perm, non_blocking=True)
        use_graph = self.lam != 0.0 and _graphs_enabled()
        if use_graph:
            # parameters may have changed since the capture (setters, another
            # trainer): stale compute copies are re-derived in place first, and
            # buffers must exist before a capture (nothing is allocated inside)
            for s in self._sizes():
                model.params.compute_for(model.step_buffers(s)[0])
            if self.graph is not None and self.graph[1] != self._buffer_key(model):
                self.graph = None  # buffers moved (e.g. evicted workspace): capture again
            if self.graph is None:
                torch.cuda.current_stream().synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    eng = self._body(model)
                self.graph = (g, self._buffer_key(model), eng)
            self.graph[0].replay()
            eng = self.graph[2]
        else:
            eng = self._body(model)
        if self.lam != 0.0:
            model.params.mark_compute_current(eng)
        self.h_logs.copy_(self.logs, non_blocking=True)
        self.h_sums.copy_(self.sums, non_blocking=True)
        self.h_lstat.copy_(self.lstat, non_blocking=True)
        self.h_ll.copy_(self.ll, non_blocking=True)

    def _sizes(self):
        return {min(self.chunk, b) for b in
                ([self.n] if self.full else list(self.stage))} | {self.ll_chunk}

    def _buffer_key(self, model):
        return tuple(sorted((k, b[1].data_ptr(), b[2].data_ptr(), b[3].data_ptr(),
                             b[4].data_ptr()) for k, b in model._buffers.items())) + (
            model.params._compute.data_ptr() if model.params._compute is not None else 0,)


def train(model: EinetModel, data, cfg: TrainerConfig, valid=None) -> list:
    """Seeded epoch loop (reference ``trainer.py:137-162``); the dataset is
    uploaded once and batches are gathered on the device."""
    return train_many([model], [data], cfg, None if valid is None else [valid])[0]


def train_many(models, datasets, cfg: TrainerConfig, valids=None, streams=16) -> list:
    """Train each model on its own dataset exactly like ``train`` (reference
    ``trainer.py:137-162``: seeded permutation per epoch, one
    ``em_stochastic_step`` per batch, or ``em_full_step``; epoch metrics),
    all models at once: model c's steps are CUDA-graph replays on stream
    c mod ``streams``, its batches are gathered on the device, and the host
    synchronises once per epoch to read every step's error words, the
    parameter-finiteness checks and the epoch log-likelihoods. Every model
    ends bitwise where a sequential ``train`` would leave it; errors raise
    the reference exceptions for the first failing (model, batch) in
    sequential order. Returns one metrics list per model; ``wall_seconds``
    is the epoch time of the whole group."""
    models = list(models)
    datasets = list(datasets)
    if len(datasets) != len(models):
        raise ValueError("one dataset per model")
    for d in datasets:
        if (d.shape[0] if isinstance(d, torch.Tensor) else len(np.atleast_2d(d))) == 0:
            raise ValueError("training dataset is empty")
    valids = list(valids) if valids is not None else [None] * len(models)
    if not models:
        return []
    dev = models[0].params.flat.device
    cur = torch.cuda.current_stream(dev)
    # datasets stay resident on the device (device fp32 tensors are used in place)
    xds = [engine.as_device_batch(d, device=dev) for d in datasets]
    vds = [None if v is None else engine.as_device_batch(v, device=dev) for v in valids]
    if len(models) == 1:
        pool = [cur]
    else:
        pool = [torch.cuda.Stream(device=dev) for _ in range(min(len(models), max(1, streams)))]
        for s in pool:
            s.wait_stream(cur)
    rngs = [np.random.default_rng(cfg.seed) for _ in models]
    plans = [_EpochPlan.get(m, xd, cfg) for m, xd in zip(models, xds)]
    metrics = [[] for _ in models]
    for epoch in range(cfg.epochs):
        t0 = time.perf_counter()
        for c, (m, ep) in enumerate(zip(models, plans)):
            perm = None if ep.full else rngs[c].permutation(ep.n)
            with torch.cuda.stream(pool[c % len(pool)]):
                ep.run(m, perm)
                if vds[c] is not None:
                    vo, st = _enqueue_ll(m, vds[c], ep.ll_chunk)
                    ep.valid_host = (_pinned(vo.shape, torch.float64), st.clone())
                    ep.valid_host[0].copy_(vo, non_blocking=True)
        for s in pool:
            s.synchronize()
        for c, (m, ep) in enumerate(zip(models, plans)):
            words = ep.h_logs.tolist()
            fin = np.isfinite(ep.h_sums.numpy())
            for bi in range(ep.nb):
                engine._raise_words(words[bi], m.family)
                if not fin[bi]:
                    raise TrainingDiverged(
                        f"non-finite parameters after epoch {epoch}, batch {bi}")
            engine._raise_words(ep.h_lstat.tolist(), m.family)
            if vds[c] is not None:
                engine._raise_words(ep.valid_host[1].cpu().tolist(), m.family)
        wall = time.perf_counter() - t0
        for c, ep in enumerate(plans):
            valid_ll = (float(np.mean(ep.valid_host[0].numpy())) if vds[c] is not None
                        else float("nan"))
            metrics[c].append(EpochMetrics(epoch=epoch, train_ll=float(np.mean(ep.h_ll.numpy())),
                                           valid_ll=valid_ll, wall_seconds=wall))
    for s in pool:
        cur.wait_stream(s)
    return metrics


# ---------------------------------------------------------------------------
# cluster-then-mix pipeline (reference trainer.py:165-228, paper section 4.2)
# ---------------------------------------------------------------------------

def _sq_dists(data, centers, rows=None):
    """Squared distances data x centers with the reference's arithmetic
    (elementwise difference, square, sum over the variable axis), computed in
    row blocks so SVHN-sized data never materialises an (n, k, d) array."""
    n, k = len(data), len(centers)
    d2 = np.empty((n, k))
    step = rows or max(1, int(2 ** 25 // max(1, k * data.shape[1])))
    for lo in range(0, n, step):
        blk = data[lo:lo + step]
        d2[lo:lo + step] = ((blk[:, None, :] - centers[None, :, :]) ** 2).sum(axis=2)
    return d2


def kmeans(data, k, seed=0, max_iter=50, block_rows=None):
    """Lloyd's algorithm; an empty cluster is re-seeded to the point farthest
    from its nearest centre (reference ``trainer.py:165-190``, identical
    labels and centres). Returns (labels, centers)."""
    data = np.asarray(data)
    if k < 1:
        raise ValueError("need at least one cluster")
    if k > len(data):
        raise ValueError("more clusters than samples")
    rng = np.random.default_rng(seed)
    centers = data[rng.choice(len(data), size=k, replace=False)].astype(float)
    labels = np.zeros(len(data), dtype=np.int64)
    for _ in range(max_iter):
        d2 = _sq_dists(data, centers, rows=block_rows)
        assign = d2.argmin(axis=1)
        nearest = None
        for c in range(k):
            members = assign == c
            if members.any():
                centers[c] = data[members].mean(axis=0)
                continue
            if nearest is None:
                nearest = d2.min(axis=1)
            far = nearest.argmax()
            centers[c] = data[far]
            assign[far] = c
        if np.array_equal(assign, labels):
            break
        labels = assign
    return labels, centers


@dataclass
class MixtureModel:
    """Convex mixture of trained models (reference ``trainer.py:193-209``)."""

    components: list
    log_pi: np.ndarray

    @property
    def weights(self):
        return np.exp(self.log_pi)

    def log_likelihood(self, x) -> np.ndarray:
        from scipy.special import logsumexp
        xd = engine.as_device_batch(x)
        parts = np.stack([m.log_likelihood(xd) for m in self.components])
        return logsumexp(parts + self.log_pi[:, None], axis=0)

    def mean_log_likelihood(self, x) -> float:
        return float(np.mean(self.log_likelihood(x)))


def train_mixture(data, n_clusters, model_factory, cfg: TrainerConfig, seed=0,
                  streams=16) -> MixtureModel:
    """Cluster the data (``kmeans``), train one model per cluster, mix by
    cluster proportion (reference ``trainer.py:212-228``).
    ``model_factory(cluster_index, cluster_data)`` returns a fresh untrained
    EinetModel. The component trainings run concurrently on the device
    (``train_many``), each bitwise equal to training it alone."""
    data = np.atleast_2d(np.asarray(data, dtype=np.float64))
    labels, _ = kmeans(data, n_clusters, seed=seed)
    subsets = [data[labels == c] for c in range(n_clusters)]
    components = [model_factory(c, s) for c, s in enumerate(subsets)]
    train_many(components, subsets, cfg, streams=streams)
    pi = np.asarray([len(s) for s in subsets], dtype=np.float64)
    pi /= pi.sum()
    return MixtureModel(components=components, log_pi=np.log(pi))
