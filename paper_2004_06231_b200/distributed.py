"""Data-parallel EM across GPUs.

Every sample's forward/backward is independent, so the global batch is
sharded contiguously across ranks (``shard_range``); the only exchange per EM
update is ONE all-reduce(sum) of the packed fp64 statistics buffer -- the
associative merge of the reference (``BackwardStats.merge``,
engine.py:228-236), which also carries each rank's failure flag -- after which
every rank applies the identical, deterministic M-step, so the parameters stay
bitwise equal across ranks. One process per GPU (``torchrun``), NCCL over
NVLink/NVSwitch; a gloo group works too (the tests run two ranks on one GPU).

The per-step work itself is ``trainer.em_stochastic_step(s)(...,
process_group=)``; this module maps a global batch onto a rank's shard.
"""

from __future__ import annotations

import numpy as np
import torch

from . import trainer
from .engine import EPS_W


def shard_range(n: int, rank: int, world: int):
    """Contiguous shard [lo, hi) of n samples for ``rank`` (sizes differ by <= 1;
    a rank gets an empty shard when n < world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must lie in [0, world)")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _rank_world(group):
    import torch.distributed as dist
    if group is None:
        group = dist.group.WORLD
    return dist.get_rank(group), dist.get_world_size(group), group


def local_shard(batch, rank: int, world: int):
    """This rank's rows of a global (B, D) batch (numpy array or tensor; a
    view, no copy)."""
    n = batch.shape[0] if hasattr(batch, "shape") else len(batch)
    lo, hi = shard_range(n, rank, world)
    return batch[lo:hi]


def em_stochastic_step(model, global_batch, lam, group=None, eps_w=EPS_W, chunk=4096,
                       normalize=None) -> float:
    """One data-parallel EM step on the global batch (reference
    ``trainer.py:99-117`` over the whole batch): this rank's contiguous shard
    through the E-step, one all-reduce of the statistics, the replicated
    M-step. Returns the global pre-update mean log-likelihood on every rank."""
    rank, world, group = _rank_world(group)
    return trainer.em_stochastic_step(model, local_shard(global_batch, rank, world), lam,
                                      eps_w=eps_w, chunk=chunk, process_group=group,
                                      normalize=normalize)


def em_stochastic_steps(model, global_batches, lam, group=None, eps_w=EPS_W, chunk=4096,
                        normalize=None) -> list:
    """``em_stochastic_step`` over a sequence of global batches of one shape,
    pipelined (no host wait between steps; ``trainer.em_stochastic_steps``)."""
    rank, world, group = _rank_world(group)
    shards = [local_shard(b, rank, world) for b in global_batches]
    return trainer.em_stochastic_steps(model, shards, lam, eps_w=eps_w, chunk=chunk,
                                       normalize=normalize, process_group=group)


def em_full_step(model, global_data, group=None, eps_w=EPS_W, chunk=4096) -> float:
    """Full-batch EM over the sharded data set (a lam = 1 step)."""
    return em_stochastic_step(model, global_data, 1.0, group=group, eps_w=eps_w, chunk=chunk)


def stats_layout(circuit, family):
    """Offsets of the packed statistics buffer (the all-reduce unit):
    [n_W | n_mix | acc_pt | P(n_leaf, K) | ll_sum, n, failed ranks]."""
    from .engine import _Layout
    lay = _Layout.of(circuit, family)
    n_phi = int(np.prod(lay.phi_shape))
    acc_pt = lay.n_w + lay.n_mix
    p_off = acc_pt + n_phi
    ll = p_off + lay.n_leaf * circuit.k
    return {"layout": lay, "acc_pt": acc_pt, "p": p_off, "ll": ll, "total": ll + 3,
            "bytes": 8 * (ll + 3)}
