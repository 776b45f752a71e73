"""Ancestral / conditional sampling (reference ``engine.py:331-423``).

Out of the EM hot path ("next" rank 1); not yet built
as device kernels in this round.
"""

from __future__ import annotations


def sample(circuit, params, family, n, seed=0):
    raise NotImplementedError("ancestral sampling is a SURVEY.md 8f 'next' item")


def conditional_sample(circuit, params, family, x_e, evidence, n, seed=0):
    raise NotImplementedError("conditional sampling is a SURVEY.md 8f 'next' item")
