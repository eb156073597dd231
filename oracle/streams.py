"""Row lanes interleaved into group streams (oracle; test infrastructure only).

P:103 — "the rANS implementation consists of multiple coder instances. These
coder instances code into/from multiple bitstreams, depending on the image
dimensions and at most one per pixel row."

Reading R7: one rANS state per pixel row (a "lane"); the G consecutive rows
[G*g, G*g+G) of a unit share stream g.  Stream layout (16-bit words):
    [x_r >> 16, x_r & 0xFFFF  for r in the group's rows ascending]   (flushed states)
    + renormalisation words in DECODER order: front t ascending, then row ascending.
The encoder walks the exact reverse, (t descending, row descending), appends
emitted words and reverses them at the end (LIFO).
"""

from __future__ import annotations

import numpy as np

from . import rans, schedule

K = 16


def n_groups(height: int, group_rows: int) -> int:
    return (height + group_rows - 1) // group_rows


def encode_unit(fs: np.ndarray, cs: np.ndarray, group_rows: int, lag: int = schedule.LAG):
    """fs, cs: (h, w) ints — frequency and cumulative of the TRUE symbol of
    every pixel.  Returns a list of streams (lists of 16-bit words)."""
    h, w = fs.shape
    T = schedule.n_fronts(w, h, lag)
    streams = []
    for g in range(n_groups(h, group_rows)):
        r0, r1 = g * group_rows, min(h, (g + 1) * group_rows)
        x = {r: rans.L for r in range(r0, r1)}
        emitted = []
        for t in range(T - 1, -1, -1):
            for r in range(r1 - 1, r0 - 1, -1):
                c = t - lag * r
                if 0 <= c < w:
                    x[r] = rans.encode_symbol(x[r], int(fs[r, c]), int(cs[r, c]), K, emitted.append)
        words = []
        for r in range(r0, r1):
            words += [x[r] >> 16, x[r] & 0xFFFF]
        words += emitted[::-1]
        streams.append(words)
    return streams


class CorruptStream(Exception):
    """End-of-lane invariant violated (CorruptContainer)."""


def decode_unit(streams, width: int, height: int, group_rows: int, front_tables,
                lag: int = schedule.LAG, dtype=np.uint8):
    """Wavefront decode of one unit.

    front_tables(t, rows, cols, img) -> (freqs, cums), arrays (n, A) for the
    pixels (rows[i], cols[i]) of front t, computed from the partially decoded
    image `img` (the window only holds already-decoded pixels).
    Returns the decoded (h, w) image (uint8; uint16 for the 12-bit alphabet).
    """
    h, w = height, width
    ng = n_groups(h, group_rows)
    if len(streams) != ng:
        raise CorruptStream("stream count")
    img = np.zeros((h, w), dtype=dtype)
    x = {}
    cursor = []
    for g in range(ng):
        r0, r1 = g * group_rows, min(h, (g + 1) * group_rows)
        s = streams[g]
        if len(s) < 2 * (r1 - r0):
            raise rans.Underflow("states")
        for r in range(r0, r1):
            i = 2 * (r - r0)
            x[r] = (s[i] << 16) | s[i + 1]
        cursor.append(2 * (r1 - r0))
    for t in range(schedule.n_fronts(w, h, lag)):
        pix = schedule.front(t, w, h, lag)
        if not pix:
            continue
        rows = np.array([p[0] for p in pix], dtype=np.int64)
        cols = np.array([p[1] for p in pix], dtype=np.int64)
        freqs, cums = front_tables(t, rows, cols, img)
        for i, (r, c) in enumerate(pix):
            g = r // group_rows

            def read(g=g):
                if cursor[g] >= len(streams[g]):
                    raise rans.Underflow("group %d" % g)
                wd = streams[g][cursor[g]]
                cursor[g] += 1
                return wd

            s, x[r] = rans.decode_symbol(x[r], freqs[i], cums[i], K, read)
            img[r, c] = s
    for r in range(h):
        if x[r] != rans.L:
            raise CorruptStream("row %d final state %d" % (r, x[r]))
    for g in range(ng):
        if cursor[g] != len(streams[g]):
            raise CorruptStream("group %d cursor %d of %d" % (g, cursor[g], len(streams[g])))
    return img


def decode_unit_with_tables(streams, freq_tables: np.ndarray, group_rows: int):
    """Decode given every pixel's full frequency table (h, w, A) — the
    "oracle fed the same integer tables" leg of north_star."""
    h, w, _ = freq_tables.shape
    cum_tables = np.cumsum(freq_tables.astype(np.int64), axis=-1) - freq_tables

    def ft(t, rows, cols, img):
        return freq_tables[rows, cols].astype(np.int64), cum_tables[rows, cols]

    return decode_unit(streams, w, h, group_rows, ft, dtype=np.uint8 if freq_tables.shape[-1] <= 256 else np.uint16)
