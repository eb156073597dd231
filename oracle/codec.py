"""Encode / decode (oracle; test infrastructure only).

P:63 — in each coding substep the network estimates the PDF of the target
pixel from its window of already-decoded pixels; the PDF drives the entropy
coder (Fig. 2).  P:87 — pixels of one wavefront step are coded in
parallel.  P:90 — "it is paramount that the same matrices enter the neural
network in the encoding and decoding steps": this oracle's encoder therefore
walks the same fronts as its decoder and feeds the network the same per-front
matrices, so oracle encode/decode are bit-consistent by construction.

Units (Q16): the image, or fixed tiles coded as independent images with fill
0 at their borders.  Streams: streams.py (R7).  Container: container.py.
"""

from __future__ import annotations

import hashlib

import numpy as np

from . import container, mlp, model_io, quant, schedule, streams, window


def alphabet_bits(layers) -> int:
    """8 for a 256-output network, 12 for 4096 outputs."""
    lay = layers["layers"] if isinstance(layers, dict) else layers
    n = np.asarray(lay[-1][0]).shape[1]
    if n not in (256, 4096):
        raise ValueError("output layer must have 256 or 4096 neurons")
    return 8 if n == 256 else 12


def _net(layers):
    """`layers` is a list of (W, b), or the dict of model_io.load_net (+ the
    image's normalised metadata under "meta_norm")."""
    if isinstance(layers, dict):
        return layers["layers"], layers.get("pool"), layers.get("meta_norm")
    return layers, None, None


def unit_front_tables(layers, precision: int, img: np.ndarray, rows, cols):
    """Tables for the pixels (rows, cols) of one front of one unit image.

    P:90: one matrix per front, one row per pixel neighbourhood (window
    features, then the image's metadata features).  The alphabet (8 or 12
    bits) follows from the network's output width."""
    lay, pool, meta_norm = _net(layers)
    x = window.net_inputs(img, rows, cols, meta_norm, alphabet_bits(lay))
    logits = mlp.logits_path(lay, x, precision, pool)
    p, f, c = quant.tables_from_logits(logits)
    return logits, p, f, c


def unit_tables_by_front(layers, precision: int, img: np.ndarray):
    """(h, w) arrays of (f_s, c_s) of each pixel's true symbol, computed front by
    front (the paper's encoder)."""
    h, w = img.shape
    fs = np.zeros((h, w), np.int64)
    cs = np.zeros((h, w), np.int64)
    for t in range(schedule.n_fronts(w, h)):
        pix = schedule.front(t, w, h)
        if not pix:
            continue
        rows = np.array([p[0] for p in pix], dtype=np.int64)
        cols = np.array([p[1] for p in pix], dtype=np.int64)
        _, _, f, c = unit_front_tables(layers, precision, img, rows, cols)
        sym = img[rows, cols].astype(np.int64)
        fs[rows, cols] = f[np.arange(len(pix)), sym]
        cs[rows, cols] = c[np.arange(len(pix)), sym]
    return fs, cs


def all_pixel_tables(layers, precision: int, img: np.ndarray, chunk: int = 65536):
    """Every pixel at once (north_star's encode batch); returns logits, p, f, c
    as (h*w, A) arrays in raster order.  Used for bpp estimates and as the
    reference for GPU logits; NOT the oracle codec's coding path."""
    h, w = img.shape
    rr, cc = np.divmod(np.arange(h * w), w)
    out = [], [], [], []
    for s in range(0, h * w, chunk):
        lg, p, f, c = unit_front_tables(layers, precision, img, rr[s:s + chunk], cc[s:s + chunk])
        for lst, v in zip(out, (lg, p, f, c)):
            lst.append(v)
    return tuple(np.concatenate(v) for v in out)


def encode_with_tables(fs_img: np.ndarray, cs_img: np.ndarray, width: int, height: int,
                       precision: int, group_rows: int, tile_w: int, tile_h: int,
                       model_sha: bytes, numerics: int = container.ORACLE_NUMERICS, meta=None,
                       bits: int = 8) -> bytes:
    """Container from given per-pixel (f_s, c_s) of the true symbols — the
    "oracle fed the same integer tables" leg (north_star).  `numerics` is the
    header field naming the arithmetic that produced the tables (the caller's;
    0 = this oracle's own)."""
    out = []
    for (x0, y0, tw, th) in container.tiles(width, height, tile_w, tile_h):
        sts = streams.encode_unit(fs_img[y0:y0 + th, x0:x0 + tw], cs_img[y0:y0 + th, x0:x0 + tw], group_rows)
        out += [streams.rans.words_to_bytes(s) for s in sts]
    return container.write(width, height, precision, group_rows, tile_w, tile_h, model_sha, out, numerics, meta,
                           bits=bits)


def encode(img: np.ndarray, model_blob: bytes, precision: int = 0, group_rows: int = 32,
           tile_w: int = 0, tile_h: int = 0, meta=None) -> bytes:
    """meta: the image's raw metadata reals (the model's metadata inputs);
    stored uncompressed in the container."""
    net = model_io.load_net(model_blob)
    net["meta_norm"] = window.meta_features(meta, net["meta_range"])
    layers = net
    bits = alphabet_bits(net)
    if np.asarray(img).max(initial=0) >= (1 << bits):
        raise ValueError("pixel value outside the model's %d-bit alphabet" % bits)
    h, w = img.shape
    fs = np.zeros((h, w), np.int64)
    cs = np.zeros((h, w), np.int64)
    for (x0, y0, tw, th) in container.tiles(w, h, tile_w, tile_h):
        f_u, c_u = unit_tables_by_front(layers, precision, np.ascontiguousarray(img[y0:y0 + th, x0:x0 + tw]))
        fs[y0:y0 + th, x0:x0 + tw] = f_u
        cs[y0:y0 + th, x0:x0 + tw] = c_u
    return encode_with_tables(fs, cs, w, h, precision, group_rows, tile_w, tile_h, model_io.digest(model_blob),
                              meta=meta, bits=bits)


class ModelHashMismatch(Exception):
    pass


def _split_streams(hdr):
    """Per-unit lists of word streams, in container order (one slice)."""
    units = container.tiles(hdr["width"], hdr["height"], hdr["tile_w"], hdr["tile_h"])
    allw = [streams.rans.bytes_to_words(s) for s in hdr["streams"]]
    per = []
    k = 0
    for (x0, y0, tw, th) in units:
        ng = streams.n_groups(th, hdr["group_rows"])
        per.append(((x0, y0, tw, th), allw[k:k + ng]))
        k += ng
    if k != len(allw):
        raise container.CorruptContainer("stream count")
    return per


def decode(blob: bytes, model_blob: bytes) -> np.ndarray:
    hdr = container.parse(blob)
    if hdr["model_sha"] != model_io.digest(model_blob):      # before any pixel work
        raise ModelHashMismatch()
    if hdr["numerics"] != container.ORACLE_NUMERICS:         # tables of another arithmetic
        raise container.CorruptContainer("numerics revision %d is not the oracle's" % hdr["numerics"])
    layers = model_io.load_net(model_blob)
    layers["meta_norm"] = window.meta_features(hdr["meta"], layers["meta_range"])   # re-read from the container
    if alphabet_bits(layers) != hdr["bits"]:
        raise container.CorruptContainer("container alphabet does not match the model's output layer")
    prec = hdr["precision"]
    dt = np.uint8 if hdr["bits"] == 8 else np.uint16
    out = np.zeros((hdr["height"], hdr["width"]), dt)
    for (x0, y0, tw, th), sts in _split_streams(hdr):
        def ft(t, rows, cols, img):
            _, _, f, c = unit_front_tables(layers, prec, img, rows, cols)
            return f, c
        out[y0:y0 + th, x0:x0 + tw] = streams.decode_unit(sts, tw, th, hdr["group_rows"], ft, dtype=dt)
    return out


def decode_with_tables(blob: bytes, freq_tables: np.ndarray) -> np.ndarray:
    """Decode a container given every pixel's full table (H, W, 256)."""
    hdr = container.parse(blob)
    out = np.zeros((hdr["height"], hdr["width"]), np.uint8 if hdr["bits"] == 8 else np.uint16)
    for (x0, y0, tw, th), sts in _split_streams(hdr):
        out[y0:y0 + th, x0:x0 + tw] = streams.decode_unit_with_tables(
            sts, freq_tables[y0:y0 + th, x0:x0 + tw], hdr["group_rows"])
    return out


def raster_decode(blob: bytes, model_blob: bytes) -> np.ndarray:
    """Sequential reference decoder for G = 1: rows top to bottom,
    columns left to right, one pixel at a time.  With one lane per stream the
    within-lane order (column ascending) equals the wavefront's, so this must
    reproduce the wavefront decoder exactly.  Each pixel's table comes from a
    one-row matrix; the fp64 forward rounded once to fp32 makes a row's logits
    independent of the batch it sits in (barring fp64 ties at an fp32 rounding
    boundary, ~1e-9 per logit), so the tables equal the encoder's."""
    hdr = container.parse(blob)
    if hdr["group_rows"] != 1:
        raise ValueError("raster decoder needs G = 1")
    if hdr["numerics"] != container.ORACLE_NUMERICS:
        raise container.CorruptContainer("numerics revision %d is not the oracle's" % hdr["numerics"])
    layers = model_io.load_net(model_blob)
    layers["meta_norm"] = window.meta_features(hdr["meta"], layers["meta_range"])
    prec = hdr["precision"]
    dt = np.uint8 if hdr["bits"] == 8 else np.uint16
    out = np.zeros((hdr["height"], hdr["width"]), dt)
    for (x0, y0, tw, th), sts in _split_streams(hdr):
        img = np.zeros((th, tw), dt)
        x = {}
        cur = {}
        for r in range(th):
            s = sts[r]
            x[r] = (s[0] << 16) | s[1]
            cur[r] = 2
        # raster order is causal for the window: every neighbour of
        # (r, c) precedes it in raster order.
        for r in range(th):
            for c in range(tw):
                rows, cols = np.array([r]), np.array([c])
                _, _, f, cm = unit_front_tables(layers, prec, img, rows, cols)

                def read(r=r):
                    wd = sts[r][cur[r]]
                    cur[r] += 1
                    return wd

                sym, x[r] = streams.rans.decode_symbol(x[r], f[0], cm[0], streams.K, read)
                img[r, c] = sym
        for r in range(th):
            if x[r] != streams.rans.L or cur[r] != len(sts[r]):
                raise streams.CorruptStream("raster end state")
        out[y0:y0 + th, x0:x0 + tw] = img
    return out


def payload_bits_estimate(fs: np.ndarray) -> float:
    """Sum of -log2(f_s / 2^16) over pixels (information content, bits)."""
    return float(np.sum(16.0 - np.log2(np.asarray(fs, np.float64))))


def sha256(b: bytes) -> bytes:
    return hashlib.sha256(b).digest()


# ---- volumes (§8(f) f2): the 3D window R13, slices in order ------
def unit_tables_by_front_3d(net, precision: int, img: np.ndarray, prev):
    """(f_s, c_s) of one slice unit, front by front (2D order within the
    slice); the lower-layer taps come from `prev` (the same unit of the
    slice below, or None for slice 0).  The 3D wavefront (R14) only overlaps
    these per-slice fronts in time; the tables are the same."""
    lay, pool, meta_norm = _net(net)
    h, w = img.shape
    fs = np.zeros((h, w), np.int64)
    cs = np.zeros((h, w), np.int64)
    for t in range(schedule.n_fronts(w, h)):
        pix = schedule.front(t, w, h)
        if not pix:
            continue
        rows = np.array([q[0] for q in pix], dtype=np.int64)
        cols = np.array([q[1] for q in pix], dtype=np.int64)
        x = window.net_inputs_3d(img, prev, rows, cols, meta_norm)
        _, f, c = quant.tables_from_logits(mlp.logits_path(lay, x, precision, pool))
        sym = img[rows, cols].astype(np.int64)
        fs[rows, cols] = f[np.arange(len(pix)), sym]
        cs[rows, cols] = c[np.arange(len(pix)), sym]
    return fs, cs


def encode_volume_with_tables(fs_vol, cs_vol, width, height, precision, group_rows, tile_w, tile_h, model_sha,
                              numerics: int = container.ORACLE_NUMERICS, meta=None) -> bytes:
    """One container for the volume (window id 2): slice-major streams, each
    slice's units as in the 2D container."""
    out = []
    for z in range(fs_vol.shape[0]):
        for (x0, y0, tw, th) in container.tiles(width, height, tile_w, tile_h):
            sts = streams.encode_unit(fs_vol[z, y0:y0 + th, x0:x0 + tw], cs_vol[z, y0:y0 + th, x0:x0 + tw],
                                      group_rows)
            out += [streams.rans.words_to_bytes(s) for s in sts]
    return container.write(width, height, precision, group_rows, tile_w, tile_h, model_sha, out, numerics, meta,
                           container.WINDOW_3D)


def encode_volume(vol: np.ndarray, model_blob: bytes, precision: int = 0, group_rows: int = 32,
                  tile_w: int = 0, tile_h: int = 0, meta=None) -> bytes:
    """vol (D, H, W) u8.  The model's inputs: 87 (+ metadata)."""
    net = model_io.load_net(model_blob)
    net["meta_norm"] = window.meta_features(meta, net["meta_range"])
    d, h, w = vol.shape
    fs = np.zeros((d, h, w), np.int64)
    cs = np.zeros((d, h, w), np.int64)
    for z in range(d):
        for (x0, y0, tw, th) in container.tiles(w, h, tile_w, tile_h):
            prev = None if z == 0 else np.ascontiguousarray(vol[z - 1, y0:y0 + th, x0:x0 + tw])
            f_u, c_u = unit_tables_by_front_3d(net, precision, np.ascontiguousarray(vol[z, y0:y0 + th, x0:x0 + tw]),
                                               prev)
            fs[z, y0:y0 + th, x0:x0 + tw] = f_u
            cs[z, y0:y0 + th, x0:x0 + tw] = c_u
    return encode_volume_with_tables(fs, cs, w, h, precision, group_rows, tile_w, tile_h,
                                     model_io.digest(model_blob), meta=meta)


def _split_volume(hdr):
    """[slice][unit] -> ((x0, y0, tw, th), word streams)."""
    sps = container.streams_per_slice(hdr["width"], hdr["height"], hdr["tile_w"], hdr["tile_h"], hdr["group_rows"])
    out = []
    for z in range(hdr["depth"]):
        sub = dict(hdr, streams=hdr["streams"][z * sps:(z + 1) * sps])
        out.append(_split_streams(sub))
    return out


def decode_volume(blob: bytes, model_blob: bytes) -> np.ndarray:
    """Slice by slice (the dependency order of the 3D wavefront, R14)."""
    hdr = container.parse(blob)
    if hdr["window"] != container.WINDOW_3D:
        raise container.CorruptContainer("not a volume container")
    if hdr["model_sha"] != model_io.digest(model_blob):
        raise ModelHashMismatch()
    if hdr["numerics"] != container.ORACLE_NUMERICS:
        raise container.CorruptContainer("numerics revision %d is not the oracle's" % hdr["numerics"])
    net = model_io.load_net(model_blob)
    net["meta_norm"] = window.meta_features(hdr["meta"], net["meta_range"])
    lay, pool, meta_norm = _net(net)
    prec = hdr["precision"]
    out = np.zeros((hdr["depth"], hdr["height"], hdr["width"]), np.uint8)
    for z, units in enumerate(_split_volume(hdr)):
        for (x0, y0, tw, th), sts in units:
            prev = None if z == 0 else np.ascontiguousarray(out[z - 1, y0:y0 + th, x0:x0 + tw])

            def ft(t, rows, cols, img, prev=prev):
                x = window.net_inputs_3d(img, prev, rows, cols, meta_norm)
                _, f, c = quant.tables_from_logits(mlp.logits_path(lay, x, prec, pool))
                return f, c
            out[z, y0:y0 + th, x0:x0 + tw] = streams.decode_unit(sts, tw, th, hdr["group_rows"], ft)
    return out


def decode_volume_with_tables(blob: bytes, freq_tables: np.ndarray) -> np.ndarray:
    """freq_tables (D, H, W, 256)."""
    hdr = container.parse(blob)
    out = np.zeros((hdr["depth"], hdr["height"], hdr["width"]), np.uint8)
    for z, units in enumerate(_split_volume(hdr)):
        for (x0, y0, tw, th), sts in units:
            out[z, y0:y0 + th, x0:x0 + tw] = streams.decode_unit_with_tables(
                sts, freq_tables[z, y0:y0 + th, x0:x0 + tw], hdr["group_rows"])
    return out
