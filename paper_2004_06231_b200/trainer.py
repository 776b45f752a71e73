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


def accumulate(model: EinetModel, batch: torch.Tensor, chunk: int):
    """E-step over a device batch into the model's stats buffer
    (reference ``trainer.py:57-66``). Returns (engine, stats, status)."""
    n = batch.shape[0]
    eng, ws, stats, status, root = model.step_buffers(min(chunk, max(n, 1)))
    compute = model.params.compute_for(eng)
    stats.zero_()
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


def _nccl_group(group) -> bool:
    try:
        import torch.distributed as dist
        return dist.get_backend(group) == "nccl"
    except Exception:
        return False


def _stage_batch(model: EinetModel, batch, normalize=None) -> torch.Tensor:
    """Device batch for the graph path. Device fp32 tensors are used in place;
    host data is copied (asynchronously when pinned) into a persistent
    per-model staging buffer, so the captured graph's input address is stable
    across steps. u8 batches travel as bytes and are decoded on the device
    into the fp32 staging buffer (``engine.decode_u8``)."""
    if isinstance(batch, torch.Tensor) and batch.is_cuda and batch.dtype != torch.uint8:
        return engine.as_device_batch(batch)
    t = _host_batch(batch)
    dev = model.params.flat.device
    st = model.__dict__.get("_staging")
    if st is None or st.shape != t.shape:
        st = torch.empty(t.shape, dtype=torch.float32, device=dev)
        model.__dict__["_staging"] = st
    if t.dtype == torch.uint8:
        if not t.is_cuda:
            t = t.to(dev, non_blocking=t.is_pinned())
        engine.decode_u8(t, normalize, out=st)
    else:
        st.copy_(t, non_blocking=t.is_pinned())
    return st


def _graph_step(model: EinetModel, xd: torch.Tensor, lam, eps_w, chunk, process_group=None):
    """Replay (capturing on first use) the CUDA graph of one EM step on the
    device batch ``xd``; returns (engine, stats, status). With a process group
    the step is two graphs (E-step, M-step) around the all-reduce of the
    statistics and of the status words (NCCL, outside the graphs)."""
    n = xd.shape[0]
    eng, ws, stats, status, root = model.step_buffers(min(chunk, max(n, 1)))
    compute = model.params.compute_for(eng)  # prepares outside the graph if stale
    key = (xd.data_ptr(), tuple(xd.shape), float(lam), float(eps_w), int(chunk),
           model.params.flat.data_ptr(), ws.data_ptr(), compute.data_ptr(),
           process_group is not None)
    cache = model.__dict__.setdefault("_graphs", {})
    gs = cache.get(key)
    if gs is None:
        if len(cache) >= _GRAPH_CACHE_SIZE:
            cache.pop(next(iter(cache)))
        torch.cuda.current_stream().synchronize()
        if process_group is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                accumulate(model, xd, chunk)
                eng.mstep(model.params.flat, compute, stats, lam, eps_w, status)
            gs = (g,)
        else:
            ge, gm = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(ge):
                accumulate(model, xd, chunk)
            with torch.cuda.graph(gm):
                eng.mstep(model.params.flat, compute, stats, lam, eps_w, status)
            gs = (ge, gm)
        cache[key] = gs
    if process_group is None:
        gs[0].replay()
    else:
        import torch.distributed as dist
        gs[0].replay()
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=process_group)
        dist.all_reduce(status, op=dist.ReduceOp.MIN, group=process_group)
        gs[1].replay()
    return eng, stats, status


def em_stochastic_step(model: EinetModel, batch, lam, eps_w=engine.EPS_W, chunk=4096,
                       process_group=None, normalize=None) -> float:
    """One gliding-average EM update; returns the pre-update mean LL of the
    batch (reference ``trainer.py:99-117``). ``lam == 0`` leaves every
    parameter bitwise unchanged.

    With ``process_group`` the statistics are summed across ranks (one NCCL
    all-reduce of the packed buffer) and every rank applies the identical
    M-step; the returned mean LL is then the global one.

    A uint8 batch (an EIND1 payload, reference ``modelio.py:145-166``) is
    copied as bytes and decoded on the device: divided by 255 unless
    ``normalize`` is False, like the reference's ``load_dataset``.
    """
    use_graph = (lam != 0.0 and _graphs_enabled() and
                 (process_group is None or _nccl_group(process_group)))
    xd = (_stage_batch(model, batch, normalize) if use_graph
          else engine.as_device_batch(batch, normalize=normalize))
    if xd.shape[0] == 0:
        raise ValueError("empty batch")
    if use_graph:
        eng, stats, status = _graph_step(model, xd, lam, eps_w, chunk, process_group)
    else:
        eng, stats, status, compute = accumulate(model, xd, chunk)
        if process_group is not None:
            import torch.distributed as dist
            dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=process_group)
            dist.all_reduce(status, op=dist.ReduceOp.MIN, group=process_group)
        if lam != 0.0:
            eng.mstep(model.params.flat, compute, stats, lam, eps_w, status)
    return _finish_step(model, eng, stats, status, lam)


def _finish_step(model, eng, stats, status, lam) -> float:
    """Read the LL sum and the error words (one device->host copy, syncs),
    raise the reference exceptions, return the mean LL."""
    ll_off = int(eng.sizes.stats_ll_offset)
    info = torch.cat([stats[ll_off:ll_off + 2], status.to(torch.float64)]).cpu().tolist()
    engine._raise_words([int(v) for v in info[2:]], model.family)
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
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(batch, dtype=np.float64),
                                                  dtype=np.float32))
    if t.dim() == 1:
        t = t[None, :]
    if t.dtype not in (torch.float32, torch.uint8):
        t = t.to(torch.float32)
    return t.contiguous()


def em_stochastic_steps(model: EinetModel, batches, lam, eps_w=engine.EPS_W,
                        chunk=4096, normalize=None) -> list:
    """Consecutive gliding-average EM steps over a sequence of host batches of
    one shape (equivalent to calling ``em_stochastic_step`` on each): the
    host->device copy of batch i+1 runs on a copy stream into the other half
    of a double-buffered staging area while step i runs on the device. Every
    step's LL (and error words) is read back after the step, as in
    ``em_stochastic_step``; returns the list of mean LLs. uint8 batches are
    copied as bytes and decoded on the device (see ``em_stochastic_step``)."""
    hosts = [_host_batch(b) for b in batches]
    if not hosts:
        return []
    if lam == 0.0 or not _graphs_enabled() or hosts[0].is_cuda:
        return [em_stochastic_step(model, b, lam, eps_w, chunk, normalize=normalize)
                for b in hosts]
    shape = tuple(hosts[0].shape)
    dtype = hosts[0].dtype
    if shape[0] == 0:
        raise ValueError("empty batch")
    dev = model.params.flat.device
    copy = model.__dict__.get("_copy_stream")
    if copy is None:
        copy = torch.cuda.Stream(device=dev)
        model.__dict__["_copy_stream"] = copy
    key = "_stage2_u8" if dtype == torch.uint8 else "_stage2_f32"
    bufs = model.__dict__.get(key)
    if bufs is None or tuple(bufs[0].shape) != shape:
        bufs = [torch.empty(shape, dtype=dtype, device=dev) for _ in range(2)]
        model.__dict__[key] = bufs
    u8 = dtype == torch.uint8
    if u8:
        xf = model.__dict__.get("_staging")
        if xf is None or tuple(xf.shape) != shape:
            xf = torch.empty(shape, dtype=torch.float32, device=dev)
            model.__dict__["_staging"] = xf
    cur = torch.cuda.current_stream(dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    used = [torch.cuda.Event(), torch.cuda.Event()]

    def issue_copy(i):
        s = i & 1
        copy.wait_stream(cur) if i < 2 else copy.wait_event(used[s])
        with torch.cuda.stream(copy):
            bufs[s].copy_(hosts[i], non_blocking=hosts[i].is_pinned())
            copied[s].record(copy)

    issue_copy(0)
    out = []
    for i, h in enumerate(hosts):
        if tuple(h.shape) != shape or h.dtype != dtype:
            raise ValueError("em_stochastic_steps needs batches of one shape and dtype")
        s = i & 1
        cur.wait_event(copied[s])
        if u8:
            engine.decode_u8(bufs[s], normalize, out=xf)  # frees bufs[s] for batch i + 2
            used[s].record(cur)
            eng, stats, status = _graph_step(model, xf, lam, eps_w, chunk)
        else:
            eng, stats, status = _graph_step(model, bufs[s], lam, eps_w, chunk)
            used[s].record(cur)
        if i + 1 < len(hosts):
            issue_copy(i + 1)
        out.append(_finish_step(model, eng, stats, status, lam))
    return out


def em_full_step(model: EinetModel, data, eps_w=engine.EPS_W, chunk=4096,
                 process_group=None) -> float:
    """Full-batch EM update == a lam = 1 stochastic step on all data."""
    return em_stochastic_step(model, data, lam=1.0, eps_w=eps_w, chunk=chunk,
                              process_group=process_group)


def _check_finite(model, epoch, batch_idx):
    if not bool(torch.isfinite(model.params.flat).all()):
        raise TrainingDiverged(
            f"non-finite parameters after epoch {epoch}, batch {batch_idx}")


def train(model: EinetModel, data, cfg: TrainerConfig, valid=None) -> list:
    """Seeded epoch loop (reference ``trainer.py:137-162``); the dataset is
    uploaded once and batches are gathered on the device."""
    host = np.atleast_2d(np.asarray(data, dtype=np.float64))
    if len(host) == 0:
        raise ValueError("training dataset is empty")
    xd = engine.as_device_batch(host)
    vd = None if valid is None else engine.as_device_batch(valid)
    rng = np.random.default_rng(cfg.seed)
    metrics = []
    for epoch in range(cfg.epochs):
        t0 = time.perf_counter()
        if cfg.mode == "full":
            em_full_step(model, xd, eps_w=cfg.eps_w, chunk=cfg.chunk)
            _check_finite(model, epoch, 0)
        else:
            order = torch.from_numpy(rng.permutation(len(host))).to(xd.device)
            for bi, lo in enumerate(range(0, len(host), cfg.batch_size)):
                em_stochastic_step(model, xd.index_select(0, order[lo:lo + cfg.batch_size]),
                                   cfg.step_size, eps_w=cfg.eps_w, chunk=cfg.chunk)
                _check_finite(model, epoch, bi)
        train_ll = model.mean_log_likelihood(xd)
        valid_ll = model.mean_log_likelihood(vd) if vd is not None else float("nan")
        metrics.append(EpochMetrics(epoch=epoch, train_ll=train_ll, valid_ll=valid_ll,
                                    wall_seconds=time.perf_counter() - t0))
    return metrics
