"""Synthetic inputs of the benchmark configurations.

Image data: per-variable N(0.5, 0.2) plus a per-image N(0, 0.15) brightness
offset, clipped to [0, 1] and quantised to k/255; variables are
channel-interleaved (var = 3 * pixel + channel).
"""

from __future__ import annotations

import numpy as np

from .builders import make_family
from .structures import StructureConfig, lift_channels, poon_domingos, random_binary_tree


def image_batch(n, d_vars, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.normal(0.5, 0.2, size=(n, d_vars)) + rng.normal(0.0, 0.15, size=(n, 1))
    return np.round(np.clip(x, 0.0, 1.0) * 255.0) / 255.0


def binary_batch(n, d_vars, seed=0):
    return np.random.default_rng(seed).integers(0, 2, size=(n, d_vars)).astype(np.float64)


CONFIGS = {
    # name: (graph factory, family factory, k, data factory)
    "C1": (lambda: random_binary_tree(16, StructureConfig(depth=3, replicas=2, seed=0)),
           lambda: make_family("categorical", num_states=2), 10, binary_batch),
    "C2": (lambda: poon_domingos(28, 28, StructureConfig(deltas=(7,), axes="vertical")),
           lambda: make_family("gaussian", image_mode=True), 10, image_batch),
    "C3": (lambda: lift_channels(poon_domingos(32, 32, StructureConfig(deltas=(8,),
                                                                     axes="vertical"))),
           lambda: make_family("gaussian", image_mode=True), 40, image_batch),
    "C3b": (lambda: lift_channels(poon_domingos(32, 32, StructureConfig(deltas=(8,),
                                                                      axes="both"))),
            lambda: make_family("gaussian", image_mode=True), 40, image_batch),
    "C4": (lambda: lift_channels(poon_domingos(128, 128, StructureConfig(deltas=(32,),
                                                                       axes="vertical"))),
           lambda: make_family("gaussian", image_mode=True), 40, image_batch),
}


def config(name):
    graph, fam, k, data = CONFIGS[name]
    rg = graph()
    return rg, fam(), k, (lambda n, seed=0: data(n, rg.d_vars, seed))
