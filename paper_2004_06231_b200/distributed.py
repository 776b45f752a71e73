"""Data-parallel EM across GPUs.

Every sample's forward/backward is independent, so the batch is sharded
contiguously across ranks; the only exchange per EM update is one all-reduce
(sum) of the packed fp64 statistics buffer -- the associative merge of the
reference (``BackwardStats.merge``, engine.py:228-236) -- after which every rank
applies the identical, deterministic M-step. One process per GPU, NCCL over
NVLink/NVSwitch for the collective (gloo works for the host-side tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import trainer
from .engine import _Layout


def shard_range(n: int, rank: int, world: int):
    """Contiguous shard [lo, hi) of n samples for ``rank`` (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def allreduce_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the packed statistics buffer over the ranks of ``group`` in place."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def em_step(model, local_batch, lam, group=None, eps_w=1e-12, chunk=4096) -> float:
    """One data-parallel EM step: local E-step, one all-reduce, replicated M-step.
    Returns the global pre-update mean log-likelihood."""
    return trainer.em_stochastic_step(model, local_batch, lam, eps_w=eps_w, chunk=chunk,
                                      process_group=group)


# ---------------------------------------------------------------------------
# host-side packing in the device buffer layout (tests, checkpoint tools)
# ---------------------------------------------------------------------------

def stats_layout(circuit, family):
    """Offsets of the packed statistics: [n_W | n_mix | acc_pt | P | ll_sum, n]."""
    lay = _Layout.of(circuit, family)
    n_phi = int(np.prod(lay.phi_shape))
    acc_pt = lay.n_w + lay.n_mix
    p_off = acc_pt + n_phi
    ll = p_off + lay.n_leaf * circuit.k
    return {"layout": lay, "acc_pt": acc_pt, "p": p_off, "ll": ll, "total": ll + 2}


def pack_stats(circuit, family, einsum, mixing, acc_pt, acc_p, ll_sum, n_samples):
    """Reference-layout statistics -> flat fp64 vector (acc_p compressed to one
    value per (leaf region, k), exactly as the device keeps it)."""
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
    out[L["ll"]] = ll_sum
    out[L["ll"] + 1] = n_samples
    return out


def unpack_stats(circuit, family, flat):
    """Flat fp64 vector -> (einsum, mixing, acc_pt, acc_p, ll_sum, n_samples)."""
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
