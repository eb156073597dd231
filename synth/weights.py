"""Seeded random weights for the dense density estimator (inputs, not arithmetic).

Layer list format shared by the oracle and the C-ABI: a list of (W, b) with
W float32 of shape [in][out] (row-major) and b float32 of shape [out].
Initialisation is He-uniform with zero biases, because the
paper ships no weights.
"""

from __future__ import annotations

import numpy as np


def he_uniform_layers(dims, seed: int = 0, bias_scale: float = 0.0):
    rng = np.random.default_rng(seed)
    layers = []
    for i in range(len(dims) - 1):
        fan_in, fan_out = dims[i], dims[i + 1]
        lim = np.sqrt(6.0 / fan_in)
        w = rng.uniform(-lim, lim, size=(fan_in, fan_out)).astype(np.float32)
        b = (rng.uniform(-1, 1, size=fan_out) * bias_scale).astype(np.float32)
        layers.append((np.ascontiguousarray(w), np.ascontiguousarray(b)))
    return layers


def zero_layers(dims):
    return [(np.zeros((dims[i], dims[i + 1]), np.float32), np.zeros(dims[i + 1], np.float32))
            for i in range(len(dims) - 1)]


def he_uniform_pooled(n_in: int, widths, pool, seed: int = 0, bias_scale: float = 0.0):
    """Layers for a network with optional pooling: layer i has widths[i]
    outputs; its successor's input is widths[i] / pool[i] (pool 0 = none)."""
    rng = np.random.default_rng(seed)
    layers = []
    fan_in = n_in
    for i, fan_out in enumerate(widths):
        lim = np.sqrt(6.0 / fan_in)
        w = rng.uniform(-lim, lim, size=(fan_in, fan_out)).astype(np.float32)
        b = (rng.uniform(-1, 1, size=fan_out) * bias_scale).astype(np.float32)
        layers.append((np.ascontiguousarray(w), np.ascontiguousarray(b)))
        fan_in = fan_out // (pool[i] or 1)
    return layers
