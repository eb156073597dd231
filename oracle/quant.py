"""Softmax and PDF -> integer frequency table (oracle; test infrastructure only).

P:96 — "The output layer consists of 256 neurons, each representing the
probability of a 8-bit grayscale value. The output layer uses the softmax
function as activation function."

The paper is silent on turning the PDF into the integer table rANS needs
(SPEC S:224 calls it "invented — artifact plumbing").  Reading R5 ("Q1"):
with precision k (2^k total) and n symbols,
    f_i = 1 + floor(fl32(p_i * (2^k - n)))            (fp32 multiply, RN)
    R   = 2^k - sum_i f_i ;  a = first index of max_i f_i ;  f_a += R
    c_i = sum_{j<i} f_j                                (exclusive prefix sum)
For k = 16, n = 256 the scale is 65280.
"""

from __future__ import annotations

import numpy as np


def softmax_fp64(logits: np.ndarray) -> np.ndarray:
    """Numerically stable softmax (subtract the row max), fp64."""
    z = np.asarray(logits, dtype=np.float64)
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def q1(p: np.ndarray, k: int = 16) -> np.ndarray:
    """Reading R5 on float32 probabilities; works on (..., n). Returns int64 f."""
    p = np.asarray(p, dtype=np.float32)
    n = p.shape[-1]
    scale = np.float32((1 << k) - n)
    f = 1 + np.floor(p * scale).astype(np.int64)        # fp32 product, then floor
    tot = f.sum(axis=-1, keepdims=True)
    r = (1 << k) - tot
    a = np.argmax(f, axis=-1)                             # first index of the max
    np.put_along_axis(f, a[..., None], np.take_along_axis(f, a[..., None], -1) + r, -1)
    assert np.all(f.sum(axis=-1) == (1 << k)) and np.all(f >= 1)
    return f


def cdf(f: np.ndarray) -> np.ndarray:
    """Exclusive prefix sums c_i = sum_{j<i} f_j."""
    f = np.asarray(f, dtype=np.int64)
    c = np.cumsum(f, axis=-1) - f
    return c


def tables_from_logits(logits_f32: np.ndarray, k: int = 16):
    """logits (fp32) -> (p fp32, f, c) with the oracle's softmax."""
    p = softmax_fp64(np.asarray(logits_f32, dtype=np.float32)).astype(np.float32)
    f = q1(p, k)
    return p, f, cdf(f)
