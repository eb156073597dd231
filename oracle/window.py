"""Causal neighbourhood window (oracle; test infrastructure only).

PAPER.md:63 — the neighbourhood window "is masked to only contain the already
decoded pixels"; P:290 (Fig. 6 caption) — "A 9-by-9 window was used; the target
pixel is located in the last row, third to last column".  P:59 (Fig. 1 right)
— pixels outside the image "are substituted with dummy values".

Readings (R1/R2):
  * the 9x9 box spans dr in [-8, 0], dc in [-6, +2] around the target;
  * cells at or after the target in raster order ((0,0), (0,1), (0,2)) are
    masked out and dropped, leaving 78 inputs in row-major order;
  * the dummy value is pixel value 0; features are v / 256.
  * 12-bit alphabet ("one 12-bit channel, leading to 4096 possible
    shades of gray"; reading R15): features are v / 4096, the same 78 taps.
"""

from __future__ import annotations

import numpy as np

BOX_ROWS = 9
BOX_COLS = 9
TARGET_ROW = BOX_ROWS - 1          # last row
TARGET_COL = BOX_COLS - 3          # third-to-last column
FILL = 0                           # dummy value (reading R2)


def _offsets():
    offs = []
    for br in range(BOX_ROWS):
        for bc in range(BOX_COLS):
            dr, dc = br - TARGET_ROW, bc - TARGET_COL
            # raster-order causality mask
            if dr < 0 or (dr == 0 and dc < 0):
                offs.append((dr, dc))
    return tuple(offs)


OFFSETS = _offsets()               # 78 (dr, dc) pairs, row-major over the box
N_INPUTS = len(OFFSETS)


def gather(img: np.ndarray, r: int, c: int, fill: int = FILL) -> np.ndarray:
    """Window values x_j = img[r+dr_j, c+dc_j] (or `fill` outside)."""
    h, w = img.shape
    out = np.empty(N_INPUTS, dtype=np.int64)
    for j, (dr, dc) in enumerate(OFFSETS):
        rr, cc = r + dr, c + dc
        out[j] = img[rr, cc] if (0 <= rr < h and 0 <= cc < w) else fill
    return out


def gather_many(img: np.ndarray, rows: np.ndarray, cols: np.ndarray, fill: int = FILL) -> np.ndarray:
    """Vectorised `gather` for many targets: returns (n, 78) int64.

    Same definition as `gather`: pads the image by the box extent with `fill`
    and indexes; pinned against `gather` in tests.
    """
    h, w = img.shape
    pad = np.full((h + 8, w + 8), fill, dtype=np.int64)   # 8 above, 6 left, 2 right
    pad[8:8 + h, 6:6 + w] = img
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    dr = np.array([o[0] for o in OFFSETS], dtype=np.int64)
    dc = np.array([o[1] for o in OFFSETS], dtype=np.int64)
    return pad[(rows[:, None] + dr[None, :] + 8), (cols[:, None] + dc[None, :] + 6)]


def features(x: np.ndarray, bits: int = 8) -> np.ndarray:
    """Network inputs v / 2^bits (reading R2: v / 256, exact in fp32 and bf16;
    R15: v / 4096 for 12-bit pixels, exact in fp32, rounded to bf16 by the bf16
    definition's input rounding)."""
    return np.asarray(x, dtype=np.float64) / float(1 << bits)


def meta_features(meta, meta_range) -> np.ndarray:
    """Metadata features ("including metadata as a feature"; reading R12 =
    SPEC S:252): raw per-image reals m_k min-max normalised with the model's
    constants, (m_k - min_k) / (max_k - min_k), in IEEE binary32 (each step
    rounded once), appended after the 78 pixel features.  Returns float64
    holding the binary32 values."""
    m = np.asarray(meta if meta is not None else [], dtype=np.float32).reshape(-1)
    if len(m) != len(meta_range):
        raise ValueError("metadata count %d != model's %d" % (len(m), len(meta_range)))
    lo = np.array([r[0] for r in meta_range], dtype=np.float32)
    hi = np.array([r[1] for r in meta_range], dtype=np.float32)
    return ((m - lo) / (hi - lo)).astype(np.float32).astype(np.float64)


def net_inputs(img: np.ndarray, rows, cols, meta_norm=None, bits: int = 8) -> np.ndarray:
    """Network input rows: 78 window features, then the metadata features
    (identical for every pixel of the image)."""
    x = features(gather_many(img, rows, cols), bits)
    if meta_norm is None or len(meta_norm) == 0:
        return x
    return np.concatenate([x, np.broadcast_to(np.asarray(meta_norm, np.float64), (x.shape[0], len(meta_norm)))], 1)


# ---- 3D window ("we choose a 2-layered window"; Fig. 6 right: the
# window in the layer below is shifted down by WS).  Reading R13: the 78-tap
# causal window in slice z (the top layer, holding the pixel of interest) plus
# a 3x3 box in slice z-1 centred on the target (dr, dc in {-1, 0, 1}, row-major,
# i.e. WS = 1: one row below the target), 87 inputs; fill 0 outside the slice
# and below slice 0.
OFFSETS_3D = tuple((dr, dc) for dr in (-1, 0, 1) for dc in (-1, 0, 1))
N_INPUTS_3D = N_INPUTS + len(OFFSETS_3D)


def gather_many_3d(prev: np.ndarray | None, rows, cols, shape, fill: int = FILL) -> np.ndarray:
    """(n, 9) lower-layer taps of the targets (rows, cols) from slice z-1
    (`prev`, or None for slice 0: all fill)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if prev is None:
        return np.full((len(rows), len(OFFSETS_3D)), fill, dtype=np.int64)
    h, w = shape
    pad = np.full((h + 2, w + 2), fill, dtype=np.int64)
    pad[1:1 + h, 1:1 + w] = prev
    dr = np.array([o[0] for o in OFFSETS_3D], dtype=np.int64)
    dc = np.array([o[1] for o in OFFSETS_3D], dtype=np.int64)
    return pad[rows[:, None] + dr[None, :] + 1, cols[:, None] + dc[None, :] + 1]


def net_inputs_3d(img: np.ndarray, prev, rows, cols, meta_norm=None) -> np.ndarray:
    """87 (+ metadata) network inputs: the 2D window, the lower-layer box, then
    the metadata features."""
    x = features(gather_many(img, rows, cols))
    x3 = features(gather_many_3d(prev, rows, cols, img.shape))
    out = np.concatenate([x, x3], 1)
    if meta_norm is None or len(meta_norm) == 0:
        return out
    return np.concatenate([out, np.broadcast_to(np.asarray(meta_norm, np.float64), (out.shape[0], len(meta_norm)))], 1)
