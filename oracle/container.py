"""Container bytes (oracle; test infrastructure only).

The paper states no framing.  Layout (SURVEY §8(c) O8 plus the numerics field
of DESIGN.md "Container", version 2), little-endian:
  off  0  4s  magic "DLIC"
  off  4  u8  version (2)
  off  5  u8  precision path (0 = fp32, 1 = bf16)
  off  6  u8  window id (1 = 9x9 causal, 78 inputs, R1; 2 = the 3D window of
              R13: 78 + a 3x3 box in the slice below, 87 inputs -- the
              container then holds a whole volume, streams slice-major)
  off  7  u8  alphabet: 0 = 8-bit pixels (256 symbols; the fill value 0 of
              R2 in earlier drafts, so 8-bit containers are unchanged), 12 =
              12-bit pixels (4096 symbols, reading R15)
  off  8  u32 width        off 12 u32 height
  off 16  u16 tile_w       off 18 u16 tile_h    (0, 0 = untiled)
  off 20  u16 group rows G
  off 22  u16 numerics: which arithmetic produced the integer tables (0 = this
              oracle's own network/softmax; the GPU build writes its revision).
              P:90: encoder and decoder agree only "as long as the precision
              of the floating point arithmetic is the same".
  off 24  32s SHA-256 of the model file
  off 56  u32 n_streams
  off 60  u32 sizes[n_streams]  (bytes per stream)
  then    u32 n_meta, f32 meta[n_meta]: the image's raw metadata reals, stored
          uncompressed ("We store the metadata uncompressed"; the
          decoder re-reads them as network inputs)
  then the streams, tile-major (tiles row-major), group-major within a tile.
"""

from __future__ import annotations

import struct

import numpy as np

MAGIC = b"DLIC"
VERSION = 2
WINDOW_ID = 1
WINDOW_3D = 2
HEADER_FIXED = 60
ORACLE_NUMERICS = 0


class CorruptContainer(Exception):
    pass


def tiles(width: int, height: int, tile_w: int, tile_h: int):
    """Independent units (Q16): row-major tiles (x0, y0, w, h); untiled -> one."""
    if tile_w == 0 or tile_h == 0:
        return [(0, 0, width, height)]
    out = []
    for y0 in range(0, height, tile_h):
        for x0 in range(0, width, tile_w):
            out.append((x0, y0, min(tile_w, width - x0), min(tile_h, height - y0)))
    return out


def streams_per_slice(width, height, tile_w, tile_h, group_rows) -> int:
    return sum(-(-th // group_rows) for (_, _, _, th) in tiles(width, height, tile_w, tile_h))


def write(width, height, precision, group_rows, tile_w, tile_h, model_sha, stream_bytes,
          numerics=ORACLE_NUMERICS, meta=None, window_id=WINDOW_ID, bits=8) -> bytes:
    assert len(model_sha) == 32 and bits in (8, 12)
    hdr = MAGIC + struct.pack("<BBBBIIHHHH", VERSION, precision, window_id, 0 if bits == 8 else 12, width, height,
                              tile_w, tile_h, group_rows, numerics)
    hdr += model_sha + struct.pack("<I", len(stream_bytes))
    hdr += b"".join(struct.pack("<I", len(s)) for s in stream_bytes)
    m = np.asarray(meta if meta is not None else [], dtype="<f4").reshape(-1)
    hdr += struct.pack("<I", len(m)) + m.tobytes()
    return hdr + b"".join(stream_bytes)


def parse(blob: bytes):
    if len(blob) < HEADER_FIXED or blob[:4] != MAGIC:
        raise CorruptContainer("magic")
    ver, prec, win, fill, w, h, tw, th, g, num = struct.unpack_from("<BBBBIIHHHH", blob, 4)
    if ver != VERSION or win not in (WINDOW_ID, WINDOW_3D) or fill not in (0, 12) or prec > 1 or g == 0:
        raise CorruptContainer("header fields")
    sha = blob[24:56]
    (n,) = struct.unpack_from("<I", blob, 56)
    if len(blob) < HEADER_FIXED + 4 * n:
        raise CorruptContainer("size table")
    sizes = struct.unpack_from("<%dI" % n, blob, HEADER_FIXED)
    off = HEADER_FIXED + 4 * n
    if len(blob) < off + 4:
        raise CorruptContainer("metadata block")
    (nm,) = struct.unpack_from("<I", blob, off)
    if nm > 255 or len(blob) < off + 4 + 4 * nm:
        raise CorruptContainer("metadata block")
    meta = np.frombuffer(blob, dtype="<f4", count=nm, offset=off + 4).astype(np.float32)
    off += 4 + 4 * nm
    hdr_bytes = off
    streams = []
    for s in sizes:
        if s % 2 or off + s > len(blob):
            raise CorruptContainer("stream bounds")
        streams.append(blob[off:off + s])
        off += s
    if off != len(blob):
        raise CorruptContainer("trailing bytes")
    sps = streams_per_slice(w, h, tw, th, g)
    if n % sps or (win == WINDOW_ID and n != sps):
        raise CorruptContainer("stream count")
    return dict(width=w, height=h, precision=prec, tile_w=tw, tile_h=th, group_rows=g, numerics=num,
                model_sha=sha, streams=streams, header_bytes=hdr_bytes, meta=meta, window=win, depth=n // sps,
                bits=8 if fill == 0 else 12)
