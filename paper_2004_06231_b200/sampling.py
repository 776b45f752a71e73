"""Ancestral / conditional sampling on the GPU (reference ``engine.py:331-423``).

The reference descends the region graph one sample at a time with a numpy
generator per sample (``SeedSequence(seed).spawn(n)``). Here all n samples
descend together on the device (``einet_sample``, csrc/sample.cu): the chosen
component of every node of a sample's induced tree is propagated layer by
layer from the root, each sum decision inverts a cumulative weight vector --
the einsum weights W[l,k] (times the evidence posterior for conditional
sampling) or the mixing weights -- exactly like the reference's ``_draw``
(``np.searchsorted(cumsum, u * total, side="right")``), and the leaves draw
from their exponential family. The uniforms come from a counter-based
Philox4x32-10 stream keyed by (seed, sample, decision site), so results are
deterministic in ``seed`` and independent of n, but they are not the numpy
streams of the reference: parity is exact against the oracle restatement fed
the same uniforms (``oracle.einet_oracle.sample_philox``) and statistical
against the reference's own sampler (tests/golden/sampling.npz).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native, engine


def _raise_sampling(words, family):
    engine._raise_words(words, family)
    if words[3] != _native.STATUS_NONE:
        raise engine.EngineError("cannot sample from an all-zero weight vector")


def _run(circuit, params, family, n, seed, trace=None, x_e=None, evidence_mask=None):
    if circuit.k_root != 1:
        raise engine.EngineError("sampling requires a scalar root (k_root = 1)")
    n = int(n)
    if n < 0:
        raise ValueError("n must be >= 0")
    eng = trace.engine if trace is not None else engine.get_engine(circuit, family, 1)
    lib = eng._lib
    dev = params.flat.device
    out = torch.empty((n, circuit.d_vars), dtype=torch.float64, device=dev)
    if n == 0:
        return out.cpu().numpy()
    scratch = torch.empty(int(lib.einet_sample_scratch_bytes(eng.handle, n)), dtype=torch.uint8,
                          device=dev)
    status = eng.new_status()
    cond = trace is not None
    ws = trace.workspace if cond else None
    xe = torch.from_numpy(np.asarray(x_e, dtype=np.float64)).to(dev) if cond else None
    ev = torch.from_numpy(np.asarray(evidence_mask, dtype=np.uint8)).to(dev) if cond else None
    p = engine._ptr
    _native.check(lib.einet_sample(eng.handle, p(params.flat), p(ws), 1 if cond else 0, p(xe),
                                   p(ev), n, int(seed) & 0xFFFFFFFFFFFFFFFF, p(scratch), p(out),
                                   p(status), engine._stream()), "einet_sample")
    _raise_sampling([int(v) for v in status.cpu().tolist()], family)
    return engine.to_host(out)


def sample(circuit, params, family, n, seed=0):
    """Ancestral sampling: n complete assignments, deterministic in seed
    (reference ``engine.py:398-404``)."""
    return _run(circuit, params, family, n, seed)


def conditional_sample(circuit, params, family, x_e, evidence, n, seed=0):
    """Samples from the conditional given evidence values (reference
    ``engine.py:407-423``): observed variables are copied from ``x_e``, branch
    choices follow the posterior of an evidence-marginalised forward pass."""
    evidence = set(int(v) for v in evidence)
    if not evidence:
        return sample(circuit, params, family, n, seed)
    if circuit.k_root != 1:
        raise engine.EngineError("sampling requires a scalar root (k_root = 1)")
    d = circuit.d_vars
    mask = np.array([i not in evidence for i in range(d)])
    x_e = np.asarray(x_e, dtype=np.float64)
    trace = engine.forward(circuit, params, family, x_e[None, :], mask)
    if not np.isfinite(trace.log_likelihood[0]):
        raise engine.EvidenceError("evidence has probability zero under the model")
    return _run(circuit, params, family, n, seed, trace=trace, x_e=x_e,
                evidence_mask=~mask)
