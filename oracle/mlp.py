"""Dense density estimator (oracle; test infrastructure only).

P:96 — "Our proposed model is a dense network consisting of six dense layers
... The output layer consists of 256 neurons ... uses the softmax function as
activation function. The number of neurons in the hidden layers varies between
128 neurons to 4096 neurons per layer".  Eq. (1): the network maps
the neighbourhood x_j..x_k to P(x_i | ...).

Readings: hidden activation ReLU (R4); optional pooling omitted
(Q6); presets P100K = 78->128x5->256 (109,184 params) and P350K = 78->256x5->256
(349,184) matching Table I's ~100K / ~350K rows.

Layers are (W [in][out] float32, b [out] float32).  This module returns the
LOGITS (pre-softmax); softmax lives in quant.py.

Optional pooling ("two optional pooling layers between the first and
second and the third and fourth layer"; semantics for flat vectors unstated,
reading R11 = SPEC S:249): pool[i] = g > 0 averages contiguous groups of g
units of layer i's activation (after ReLU) before layer i+1.  In the bf16
definition the average is taken exactly over the bf16-rounded activations
(no re-rounding of the average: it enters the next layer's exact products).

Precision variants:
  forward_fp64   exact reference (fp64 throughout);
  forward_fp32   numpy float32 matmul (checks fp32 is within 1e-6 of fp64);
  forward_bf16   the bf16 path's plain definition: every matmul operand
                 (inputs, activations, weights) rounded to bf16 (RN-even),
                 products summed exactly (fp64) and rounded once to fp32,
                 bias added in fp32 (RN), ReLU, and the hidden activation
                 rounded to bf16 (RN-even) before it enters the next layer;
  logits_path    the value the codec uses: fp64 (precision 0) or bf16-emulated
                 (precision 1) forward, rounded once to float32.
"""

from __future__ import annotations

import numpy as np

P100K = (78, 128, 128, 128, 128, 128, 256)
P350K = (78, 256, 256, 256, 256, 256, 256)
# 12-bit alphabet (P:207-208, 4096 outputs; reading R16): P350K's hidden
# stack with a 4096-neuron softmax layer, 1,336,064 parameters (Table III
# "~1,350,000")
P12 = (78, 256, 256, 256, 256, 256, 4096)


def n_params(dims) -> int:
    return sum(dims[i] * dims[i + 1] + dims[i + 1] for i in range(len(dims) - 1))


def flops_per_pixel(dims) -> int:
    """2 * sum K*N multiply-adds."""
    return 2 * sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))


def avg_pool(h: np.ndarray, g: int) -> np.ndarray:
    """Average over contiguous groups of g units (last axis), exact in fp64."""
    if not g:
        return h
    h = np.asarray(h, dtype=np.float64)
    return h.reshape(h.shape[:-1] + (h.shape[-1] // g, g)).sum(-1) / g


def forward_fp64(layers, x: np.ndarray, pool=None) -> np.ndarray:
    h = np.asarray(x, dtype=np.float64)
    n = len(layers)
    for i, (w, b) in enumerate(layers):
        h = h @ np.asarray(w, np.float64) + np.asarray(b, np.float64)
        if i < n - 1:
            h = np.maximum(h, 0.0)
            if pool is not None:
                h = avg_pool(h, pool[i])
    return h


def forward_fp32(layers, x: np.ndarray, pool=None) -> np.ndarray:
    h = np.asarray(x, dtype=np.float32)
    n = len(layers)
    for i, (w, b) in enumerate(layers):
        h = h @ np.asarray(w, np.float32) + np.asarray(b, np.float32)
        if i < n - 1:
            h = np.maximum(h, np.float32(0))
            if pool is not None and pool[i]:
                h = avg_pool(h, pool[i]).astype(np.float32)
    return h


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float values to the nearest bfloat16 (ties to even), returned as
    float64.  Plain definition on the float32 bit pattern: keep the top 16
    bits after adding 0x7FFF + lsb (finite inputs only)."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = ((u + 0x7FFF + lsb) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def forward_bf16(layers, x: np.ndarray, pool=None) -> np.ndarray:
    """bf16 operands, exact (fp64) accumulation; activations re-rounded to
    bf16 after bias+ReLU computed in fp32 (the GPU epilogue's precision);
    pooling (if any) averages the bf16 activations exactly."""
    h = bf16_round(np.asarray(x, dtype=np.float64))
    n = len(layers)
    for i, (w, b) in enumerate(layers):
        acc = h @ bf16_round(w)
        z = (acc.astype(np.float32) + np.asarray(b, np.float32)).astype(np.float64)
        if i < n - 1:
            h = bf16_round(np.maximum(z, 0.0))
            if pool is not None:
                h = avg_pool(h, pool[i])
        else:
            h = z
    return h


def logits_path(layers, x: np.ndarray, precision: int, pool=None) -> np.ndarray:
    """Logits used by the oracle codec: fp64 (0) or bf16 emulation (1), as fp32."""
    if precision == 0:
        return forward_fp64(layers, x, pool).astype(np.float32)
    if precision == 1:
        return forward_bf16(layers, x, pool).astype(np.float32)
    raise ValueError("precision")
