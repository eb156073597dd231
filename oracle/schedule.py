"""Wavefront schedule (oracle; test infrastructure only).

PAPER.md:87 — "We use a principle similar to wavefront parallel processing
(WPP) as defined in the HEVC standard ... we instead determine in each coding
step which pixels we may code next. These pixels are then coded in parallel."
P:59 (Fig. 1 right) visualises the front.

Reading R3: step(r, c) = c + L*r with the minimal row lag L for the window:
L = 1 + max{dc : (dr, dc) in window, dr < 0} (SPEC S:135 lag algebra); for the
78-offset window L = 3.  Fronts t = 0 .. W + L(H-1) - 1; within a front, rows
ascending.
"""

from __future__ import annotations

from . import window


def row_lag(offsets=window.OFFSETS) -> int:
    """Minimal lag so every in-image neighbour has a strictly smaller step."""
    dcs = [dc for dr, dc in offsets if dr < 0]
    return 1 + max(0, max(dcs) if dcs else 0)


LAG = row_lag()


def step(r: int, c: int, lag: int = LAG) -> int:
    return c + lag * r


def n_fronts(width: int, height: int, lag: int = LAG) -> int:
    if width <= 0 or height <= 0:
        return 0
    return width + lag * (height - 1)


def front(t: int, width: int, height: int, lag: int = LAG):
    """Pixels (r, c) with step(r, c) == t, rows ascending."""
    out = []
    for r in range(height):
        c = t - lag * r
        if 0 <= c < width:
            out.append((r, c))
    return out


def front_rows(t: int, width: int, height: int, lag: int = LAG):
    """Closed form of the active row range [lo, hi] of front t (may be empty)."""
    lo = max(0, -(-(t - width + 1) // lag))
    hi = min(height - 1, t // lag)
    return lo, hi


# ---- 3D wavefront ("We overlap 2D wavefronts to decode all layers
# at once.  The wavefronts are shifted in each layer in such a way that the
# pixels used in the neighborhood window in the layer above are already
# decoded").  Reading R14: slice z runs the 2D schedule delayed by z * lag3d
# steps; the minimal lag3d makes every lower-layer tap (z-1, r+dr, c+dc) of a
# pixel precede it: 1 + max over the 3D box of (dc + L dr) (= 5 for the 3x3
# box and L = 3).  The decoder may use any larger lag (more slack); the
# bitstream does not depend on it (each slice's streams follow its own 2D
# order).
def slice_lag(offsets_3d=window.OFFSETS_3D, lag: int = LAG) -> int:
    return 1 + max(dc + lag * dr for dr, dc in offsets_3d)


LAG3D = slice_lag()


def step_3d(z: int, r: int, c: int, lag3d: int = LAG3D, lag: int = LAG) -> int:
    return z * lag3d + step(r, c, lag)


def n_fronts_3d(width: int, height: int, depth: int, lag3d: int = LAG3D) -> int:
    if depth <= 0:
        return 0
    return n_fronts(width, height) + lag3d * (depth - 1)
