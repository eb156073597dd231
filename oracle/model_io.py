"""Model file "DLICMDL1" (oracle; test infrastructure only).

The paper ships no model format.  SPEC S:256 ("External Interfaces" of the
model module) fixes one; this oracle writes exactly that layout:
  magic "DLICMDL1"; u16 layer count; per layer: u32 in, u32 out,
  u8 activation (1 = ReLU, 0 = none), u8 pooling group (0 = none),
  float32 W[in][out] row-major, float32 b[out]; u16 metadata feature count
  (0 here); trailing SHA-256 of all preceding bytes (the content hash the
  container records).
All integers little-endian.
"""

from __future__ import annotations

import hashlib
import struct

import numpy as np

MAGIC = b"DLICMDL1"


class CorruptModel(Exception):
    pass


def save(layers) -> bytes:
    body = bytearray(MAGIC)
    body += struct.pack("<H", len(layers))
    for i, (w, b) in enumerate(layers):
        w = np.ascontiguousarray(w, dtype="<f4")
        b = np.ascontiguousarray(b, dtype="<f4")
        act = 1 if i < len(layers) - 1 else 0
        body += struct.pack("<IIBB", w.shape[0], w.shape[1], act, 0)
        body += w.tobytes() + b.tobytes()
    body += struct.pack("<H", 0)
    return bytes(body) + hashlib.sha256(bytes(body)).digest()


def load(blob: bytes):
    if len(blob) < 8 + 2 + 2 + 32 or blob[:8] != MAGIC:
        raise CorruptModel("magic")
    body, digest = blob[:-32], blob[-32:]
    if hashlib.sha256(body).digest() != digest:
        raise CorruptModel("hash")
    (n,) = struct.unpack_from("<H", body, 8)
    off = 10
    layers = []
    for _ in range(n):
        i, o, _act, _pool = struct.unpack_from("<IIBB", body, off)
        off += 10
        w = np.frombuffer(body, dtype="<f4", count=i * o, offset=off).reshape(i, o).astype(np.float32)
        off += 4 * i * o
        b = np.frombuffer(body, dtype="<f4", count=o, offset=off).astype(np.float32)
        off += 4 * o
        layers.append((w, b))
    (nmeta,) = struct.unpack_from("<H", body, off)
    off += 2 + 8 * nmeta
    if off != len(body):
        raise CorruptModel("length")
    return layers


def digest(blob: bytes) -> bytes:
    return blob[-32:]
