"""Softmax and PDF -> integer frequency table (oracle; test infrastructure only).

P:96 — "The output layer consists of 256 neurons, each representing the
probability of a 8-bit grayscale value. The output layer uses the softmax
function as activation function."

The paper is silent on turning the PDF into the integer table rANS needs
(SPEC S:224 calls it "invented — artifact plumbing").  Reading R5 (DESIGN.md,
"Q1'"): with precision k (total 2^k) and n symbols,
    f_i = 1 + floor(fl32(p_i * (2^k - n - 1)))         (fp32 multiply, RN)
    R   = 2^k - sum_i f_i   (>= 0, see below) ;  f_{n-1} += R
    c_i = sum_{j<i} f_j                                (exclusive prefix sum)
For k = 16, n = 256 the scale is 65279.  Because sum_i p_i <= 1 + 258*2^-24
for an fp32 softmax, sum_i fl(p_i * 65279) < 65281, so sum_i f_i <= 2^16 and
R >= 0: every f_i >= 1 without a guard.  Putting the residual on the LAST
symbol leaves c_i unchanged for i < n-1, so a decoder can search the slot in
the same pass that builds the table.

12-bit alphabet ("our final model has 4096 output layer neurons";
reading R17): the same rule with n = 4096, k = 16 (SPEC S:95 keeps k = 16 for
both alphabets) and a guard of 64 instead of 1: scale = 2^16 - 4096 - 64 =
61376.  With 4096 terms an fp32 softmax may sum to 1 + ~4096 ulp, so the
guard must absorb 61376 * 4096 * 2^-23 ~ 30 units; 64 does.  (For n = 256 the
guard stays 1: the 8-bit definition is unchanged.)
"""

from __future__ import annotations

import numpy as np


def softmax_fp64(logits: np.ndarray) -> np.ndarray:
    """Numerically stable softmax (subtract the row max), fp64."""
    z = np.asarray(logits, dtype=np.float64)
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def guard(n: int) -> int:
    """Mass held back from the scale: 1 for the 8-bit alphabet (R5), 64 for
    4096 symbols (R17)."""
    return 1 if n <= 256 else 64


def q1(p: np.ndarray, k: int = 16) -> np.ndarray:
    """Reading R5 (Q1') on float32 probabilities; works on (..., n). Returns int64 f."""
    p = np.asarray(p, dtype=np.float32)
    n = p.shape[-1]
    scale = np.float32((1 << k) - n - guard(n))
    f = 1 + np.floor(p * scale).astype(np.int64)        # fp32 product, then floor
    r = (1 << k) - f.sum(axis=-1)
    assert np.all(r >= 0), "sum of probabilities exceeds the guard"
    f[..., n - 1] += r
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
