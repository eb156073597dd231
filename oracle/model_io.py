"""Model file "DLICMDL1" (oracle; test infrastructure only).

The paper ships no model format.  SPEC S:256 ("External Interfaces" of the
model module) fixes one; this oracle writes exactly that layout:
  magic "DLICMDL1"; u16 layer count; per layer: u32 in, u32 out,
  u8 activation (1 = ReLU, 0 = none), u8 pooling group g (0 = none: average
  over contiguous groups of g units after the activation, SPEC S:196/S:249 --
  the paper's "two optional pooling layers"), float32 W[in][out]
  row-major, float32 b[out]; u16 metadata feature count n and n x float32
  (min, max) (the network's last n inputs are metadata features min-max
  normalised with these constants; the paper's metadata inputs,
  P:210); trailing SHA-256 of all preceding bytes (the content hash the
  container records).
All integers little-endian.  With pooling, layer i+1's input dim is layer
i's output dim / g.
"""

from __future__ import annotations

import hashlib
import struct

import numpy as np

MAGIC = b"DLICMDL1"


class CorruptModel(Exception):
    pass


def save(layers, pool=None, meta_range=None) -> bytes:
    """pool[i]: pooling group after layer i (0 = none); meta_range: list of
    (min, max) of the metadata features (the last inputs of layer 0)."""
    pool = list(pool) if pool is not None else [0] * len(layers)
    meta_range = list(meta_range or [])
    body = bytearray(MAGIC)
    body += struct.pack("<H", len(layers))
    for i, (w, b) in enumerate(layers):
        w = np.ascontiguousarray(w, dtype="<f4")
        b = np.ascontiguousarray(b, dtype="<f4")
        act = 1 if i < len(layers) - 1 else 0
        body += struct.pack("<IIBB", w.shape[0], w.shape[1], act, pool[i])
        body += w.tobytes() + b.tobytes()
    body += struct.pack("<H", len(meta_range))
    for lo, hi in meta_range:
        body += struct.pack("<ff", lo, hi)
    return bytes(body) + hashlib.sha256(bytes(body)).digest()


def load(blob: bytes):
    """The (W, b) layers (pooling and metadata: load_net)."""
    return load_net(blob)["layers"]


def load_net(blob: bytes):
    """dict(layers=[(W, b)], pool=[g per layer], meta_range=[(min, max)])."""
    if len(blob) < 8 + 2 + 2 + 32 or blob[:8] != MAGIC:
        raise CorruptModel("magic")
    body, digest = blob[:-32], blob[-32:]
    if hashlib.sha256(body).digest() != digest:
        raise CorruptModel("hash")
    (n,) = struct.unpack_from("<H", body, 8)
    off = 10
    layers = []
    pool = []
    for _ in range(n):
        i, o, _act, g = struct.unpack_from("<IIBB", body, off)
        pool.append(g)
        off += 10
        w = np.frombuffer(body, dtype="<f4", count=i * o, offset=off).reshape(i, o).astype(np.float32)
        off += 4 * i * o
        b = np.frombuffer(body, dtype="<f4", count=o, offset=off).astype(np.float32)
        off += 4 * o
        layers.append((w, b))
    (nmeta,) = struct.unpack_from("<H", body, off)
    meta_range = [struct.unpack_from("<ff", body, off + 2 + 8 * k) for k in range(nmeta)]
    off += 2 + 8 * nmeta
    if off != len(body):
        raise CorruptModel("length")
    for k in range(len(layers) - 1):   # dims chain after pooling
        g = pool[k] or 1
        if layers[k][0].shape[1] % g or layers[k][0].shape[1] // g != layers[k + 1][0].shape[0]:
            raise CorruptModel("layer dims do not chain")
    return dict(layers=layers, pool=pool, meta_range=meta_range)


def digest(blob: bytes) -> bytes:
    return blob[-32:]
