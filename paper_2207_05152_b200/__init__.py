"""Thin Python binding of libdlic.so (include/dlic.h) — argument marshalling only.

Every function here has the name of the C entry point it wraps and does no
pixel-level work: the window gather, density estimator, softmax/quantiser,
rANS lanes, wavefront and stream compaction all run in the CUDA kernels of
csrc/.  NumPy carries host arrays; PyTorch is used only for device memory and
streams in the *_batch_device variants.  There is no CPU fallback: the
library is loaded on first use, and every call raises ImportError when
libdlic.so is not built (the pure-Python sharding helpers in dist.py import
without it).

Paper: arXiv 2207.05152 (DLIC) — encode(image, weights) -> bitstream,
decode(bitstream, weights) -> image (Fig. 2).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DLIC_LIB") or os.path.join(_HERE, "libdlic.so")
_lib = None

PREC_FP32 = 0
PREC_BF16 = 1

c_u8p = ctypes.POINTER(ctypes.c_uint8)
c_u8pp = ctypes.POINTER(c_u8p)


MAX_META = 8


class dlic_opts(ctypes.Structure):
    _fields_ = [("precision", ctypes.c_uint32), ("group_rows", ctypes.c_uint32),
                ("tile_w", ctypes.c_uint32), ("tile_h", ctypes.c_uint32),
                ("n_meta", ctypes.c_uint32), ("meta", ctypes.POINTER(ctypes.c_float)),
                ("volume_depth", ctypes.c_uint32)]


class dlic_header(ctypes.Structure):
    _fields_ = [("width", ctypes.c_uint32), ("height", ctypes.c_uint32), ("precision", ctypes.c_uint32),
                ("group_rows", ctypes.c_uint32), ("tile_w", ctypes.c_uint32), ("tile_h", ctypes.c_uint32),
                ("n_streams", ctypes.c_uint32), ("n_units", ctypes.c_uint32), ("numerics", ctypes.c_uint32),
                ("depth", ctypes.c_uint32),
                ("n_meta", ctypes.c_uint32), ("meta", ctypes.c_float * MAX_META),
                ("model_sha256", ctypes.c_uint8 * 32),
                ("payload_bytes", ctypes.c_uint64), ("header_bytes", ctypes.c_uint64), ("bits", ctypes.c_uint32)]


def _sig(lib, name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_vp = ctypes.c_void_p
_st = ctypes.c_int


def _setup(lib):
    _sig(lib, "dlic_status_str", ctypes.c_char_p, _st)
    _sig(lib, "dlic_last_error", ctypes.c_char_p)
    _sig(lib, "dlic_free", None, _vp)
    _sig(lib, "dlic_model_load", _st, _vp, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(_vp))
    _sig(lib, "dlic_model_from_arrays", _st, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32),
         ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.c_int, ctypes.POINTER(_vp))
    _sig(lib, "dlic_model_free", None, _vp)
    _sig(lib, "dlic_model_sha256", _st, _vp, _vp)
    _sig(lib, "dlic_model_blob_check", _st, _vp, ctypes.c_size_t, _vp)
    _sig(lib, "dlic_encode", _st, _vp, _vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_size_t,
         ctypes.POINTER(dlic_opts), c_u8pp, ctypes.POINTER(ctypes.c_size_t))
    _sig(lib, "dlic_decode", _st, _vp, _vp, ctypes.c_size_t, _vp, ctypes.c_size_t)
    _sig(lib, "dlic_peek", _st, _vp, ctypes.c_size_t, ctypes.POINTER(dlic_header))
    _sig(lib, "dlic_max_container_bytes", ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(dlic_opts))
    _sig(lib, "dlic_encode_batch", _st, _vp, _vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
         ctypes.POINTER(dlic_opts), c_u8pp, ctypes.POINTER(ctypes.c_size_t), _vp)
    _sig(lib, "dlic_decode_batch", _st, _vp, _vp, ctypes.c_size_t, _vp, ctypes.c_uint32, _vp, ctypes.c_size_t)
    _sig(lib, "dlic_encode_batch_device", _st, _vp, _vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
         ctypes.POINTER(dlic_opts), _vp, ctypes.c_size_t, _vp, _vp)
    _sig(lib, "dlic_decode_batch_device", _st, _vp, _vp, _vp, _vp, ctypes.c_uint32, ctypes.POINTER(dlic_header), _vp,
         _vp, _vp)
    _sig(lib, "dlic_rans_encode_tables", _st, _vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(dlic_opts), _vp,
         c_u8pp, ctypes.POINTER(ctypes.c_size_t))
    _sig(lib, "dlic_rans_decode_tables", _st, _vp, ctypes.c_size_t, _vp, _vp)
    _sig(lib, "dlic_debug_mlp", _st, _vp, _vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(dlic_opts),
         _vp, _vp, _vp, _vp)
    _sig(lib, "dlic_info", _st, ctypes.c_char_p, ctypes.c_size_t)
    _sig(lib, "dlic_set_timing", None, ctypes.c_int)
    _sig(lib, "dlic_last_kernel_ms", ctypes.c_double, ctypes.c_char_p)
    _sig(lib, "dlic_numerics_rev", ctypes.c_uint32)
    _sig(lib, "dlic_unit_streams", _st, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(dlic_opts), ctypes.c_uint32,
         ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32))
    _sig(lib, "dlic_encode_units", _st, _vp, _vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_size_t,
         ctypes.POINTER(dlic_opts), ctypes.c_uint32, ctypes.c_uint32, c_u8pp, ctypes.POINTER(ctypes.c_size_t), _vp)
    _sig(lib, "dlic_container_build", _st, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(dlic_opts), _vp, _vp,
         ctypes.c_uint32, _vp, ctypes.c_size_t, c_u8pp, ctypes.POINTER(ctypes.c_size_t))
    _sig(lib, "dlic_decode_units", _st, _vp, _vp, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint32, _vp,
         ctypes.c_size_t)
    _sig(lib, "dlic_encode_volume", _st, _vp, _vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
         ctypes.POINTER(dlic_opts), c_u8pp, ctypes.POINTER(ctypes.c_size_t))
    _sig(lib, "dlic_decode_volume", _st, _vp, _vp, ctypes.c_size_t, _vp, ctypes.c_size_t)


def _L():
    """The loaded libdlic.so (first call loads it; raises ImportError if unbuilt)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libdlic.so not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(nvcc -gencode arch=compute_100a,code=sm_100a)")
        lib = ctypes.CDLL(LIB_PATH)
        _setup(lib)
        _lib = lib
    return _lib


class DlicError(RuntimeError):
    def __init__(self, status, detail):
        self.status = int(status)
        super().__init__("%s (%d): %s" % (_L().dlic_status_str(status).decode(), status, detail))


STATUS = {0: "DLIC_OK", 1: "DLIC_E_INVALID_ARG", 2: "DLIC_E_SHAPE_MISMATCH", 3: "DLIC_E_NONCAUSAL_WINDOW",
          4: "DLIC_E_CORRUPT_MODEL", 5: "DLIC_E_VERSION_MISMATCH", 6: "DLIC_E_CORRUPT_CONTAINER",
          7: "DLIC_E_MODEL_HASH_MISMATCH", 8: "DLIC_E_STREAM_UNDERFLOW", 9: "DLIC_E_SUM_MISMATCH",
          10: "DLIC_E_ZERO_FREQUENCY", 11: "DLIC_E_BUFFER_TOO_SMALL", 12: "DLIC_E_CUDA",
          13: "DLIC_E_OUT_OF_MEMORY", 14: "DLIC_E_UNSUPPORTED_MODEL"}


def _check(s):
    if s != 0:
        raise DlicError(s, _L().dlic_last_error().decode(errors="replace"))


def _opts(precision=PREC_BF16, group_rows=32, tile=(0, 0), meta=None, volume_depth=0):
    """meta: raw metadata reals, (n_meta,) for one image or (n, n_meta) for a
    batch.  volume_depth: 0 = 2D images, D = volumes of D slices.  The
    returned struct keeps the float32 array alive."""
    o = dlic_opts(precision, group_rows, tile[0], tile[1], 0, None, volume_depth)
    if meta is not None:
        m = np.ascontiguousarray(np.asarray(meta, dtype=np.float32))
        o._meta_keep = m
        o.n_meta = m.shape[-1] if m.ndim else 1
        o.meta = m.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    return o


def _take(ptr, n) -> bytes:
    b = ctypes.string_at(ptr, n)
    _L().dlic_free(ptr)
    return b


class Model:
    """Owns a dlic_model* (uploaded weights)."""

    def __init__(self, handle, device):
        self._h = _vp(handle)
        self.device = device

    @property
    def handle(self):
        return self._h

    def sha256(self) -> bytes:
        out = (ctypes.c_uint8 * 32)()
        _check(_L().dlic_model_sha256(self._h, out))
        return bytes(out)

    def close(self):
        if self._h:
            _L().dlic_model_free(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ models
def dlic_model_load(blob: bytes, device: int = 0) -> Model:
    h = _vp()
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(_L().dlic_model_load(buf, len(blob), device, ctypes.byref(h)))
    return Model(h.value, device)


def dlic_model_from_arrays(layers, device: int = 0) -> Model:
    dims = [layers[0][0].shape[0]] + [w.shape[1] for w, _ in layers]
    ws = [np.ascontiguousarray(w, np.float32) for w, _ in layers]
    bs = [np.ascontiguousarray(b, np.float32) for _, b in layers]
    cd = (ctypes.c_uint32 * len(dims))(*dims)
    wp = (_vp * len(ws))(*[w.ctypes.data for w in ws])
    bp = (_vp * len(bs))(*[b.ctypes.data for b in bs])
    h = _vp()
    _check(_L().dlic_model_from_arrays(len(ws), cd, wp, bp, device, ctypes.byref(h)))
    return Model(h.value, device)


def dlic_model_blob_check(blob: bytes) -> bytes:
    out = (ctypes.c_uint8 * 32)()
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(_L().dlic_model_blob_check(buf, len(blob), out))
    return bytes(out)


# ------------------------------------------------------------------ codec
def _pixels(a) -> np.ndarray:
    """u16 arrays stay u16 (12-bit alphabet: a P12 model's images), anything
    else becomes u8."""
    a = np.asarray(a)
    return np.ascontiguousarray(a, dtype=np.uint16 if a.dtype == np.uint16 else np.uint8)


def _pix_dtype(hd) -> type:
    return np.uint16 if hd.get("bits", 8) == 12 else np.uint8


def dlic_encode(model: Model, img: np.ndarray, precision=PREC_BF16, group_rows=32, tile=(0, 0),
                meta=None) -> bytes:
    """img (H, W): u8, or u16 (values < 4096) for a 12-bit (P12) model."""
    img = _pixels(img)
    assert img.ndim == 2
    h, w = img.shape
    out = c_u8p()
    n = ctypes.c_size_t()
    o = _opts(precision, group_rows, tile, meta)
    _check(_L().dlic_encode(model.handle, img.ctypes.data, w, h, w, ctypes.byref(o), ctypes.byref(out),
                            ctypes.byref(n)))
    return _take(out, n.value)


def dlic_peek(bits: bytes) -> dict:
    hd = dlic_header()
    _check(_L().dlic_peek(bits, len(bits), ctypes.byref(hd)))
    d = {k: getattr(hd, k) for k, _ in dlic_header._fields_ if k not in ("model_sha256", "meta")}
    d["model_sha256"] = bytes(hd.model_sha256)
    d["meta"] = np.array(hd.meta[:hd.n_meta], dtype=np.float32)
    return d


def dlic_decode(model: Model, bits: bytes) -> np.ndarray:
    hd = dlic_peek(bits)
    img = np.empty((hd["height"], hd["width"]), _pix_dtype(hd))
    _check(_L().dlic_decode(model.handle, bits, len(bits), img.ctypes.data, img.nbytes))
    return img


def dlic_encode_batch(model: Model, imgs: np.ndarray, precision=PREC_BF16, group_rows=32, tile=(0, 0), meta=None,
                      volume_depth=0):
    """imgs (n, H, W) u8 host -> (blob, sizes): the containers back to back
    (n, or n / volume_depth volumes).  meta: raw metadata reals per container."""
    imgs = _pixels(imgs)
    n, h, w = imgs.shape
    out = c_u8p()
    tot = ctypes.c_size_t()
    sizes = np.zeros(n // volume_depth if volume_depth else n, np.uint64)
    o = _opts(precision, group_rows, tile, meta, volume_depth)
    _check(_L().dlic_encode_batch(model.handle, imgs.ctypes.data, n, w, h, ctypes.byref(o), ctypes.byref(out),
                                  ctypes.byref(tot), sizes.ctypes.data))
    return _take(out, tot.value), [int(x) for x in sizes]


def dlic_decode_batch(model: Model, blob: bytes, sizes) -> np.ndarray:
    """containers back to back (sizes[i] bytes each) -> (n, H, W) u8 (a volume
    container contributes its depth slices)."""
    sizes = [int(x) for x in sizes]
    offs = np.zeros(len(sizes), np.uint64)
    offs[1:] = np.cumsum(sizes[:-1])
    hd = dlic_peek(blob[:sizes[0]])
    imgs = np.empty((len(sizes) * max(1, hd["depth"]), hd["height"], hd["width"]), _pix_dtype(hd))
    _check(_L().dlic_decode_batch(model.handle, blob, len(blob), offs.ctypes.data, len(sizes), imgs.ctypes.data,
                                  imgs.nbytes))
    return imgs


def dlic_max_container_bytes(width, height, precision=PREC_BF16, group_rows=32, tile=(0, 0), meta=None,
                             volume_depth=0) -> int:
    """Per container (a volume container holds volume_depth slices)."""
    o = _opts(precision, group_rows, tile, meta, volume_depth)
    return int(_L().dlic_max_container_bytes(width, height, ctypes.byref(o)))


# ------------------------------------------------------------------ parity taps
def dlic_rans_encode_tables(fc: np.ndarray, precision=PREC_BF16, group_rows=32, tile=(0, 0),
                            model_sha: bytes | None = None, meta=None) -> bytes:
    """fc (H, W), or (D, H, W) for a volume container."""
    fc = np.ascontiguousarray(fc, dtype=np.uint32)
    h, w = fc.shape[-2:]
    out = c_u8p()
    n = ctypes.c_size_t()
    o = _opts(precision, group_rows, tile, meta, fc.shape[0] if fc.ndim == 3 else 0)
    sha = ctypes.create_string_buffer(model_sha, 32) if model_sha else None
    _check(_L().dlic_rans_encode_tables(fc.ctypes.data, w, h, ctypes.byref(o), sha, ctypes.byref(out),
                                        ctypes.byref(n)))
    return _take(out, n.value)


def dlic_rans_decode_tables(bits: bytes, freq_tables: np.ndarray) -> np.ndarray:
    hd = dlic_peek(bits)
    ft = np.ascontiguousarray(freq_tables, dtype=np.uint16)
    shape = ((hd["depth"],) if hd["depth"] else ()) + (hd["height"], hd["width"])
    assert ft.shape == shape + (256,)
    img = np.empty(shape, np.uint8)
    _check(_L().dlic_rans_decode_tables(bits, len(bits), ft.ctypes.data, img.ctypes.data))
    return img


def dlic_debug_mlp(model: Model, img: np.ndarray, precision=PREC_BF16, group_rows=32, tile=(0, 0),
                   logits=True, probs=True, freqs=True, fc=True, meta=None) -> dict:
    """img (H, W), or (D, H, W) for a volume (3D window); u16 for a 12-bit
    (P12) model, whose tables have 4096 entries."""
    img = _pixels(img)
    h, w = img.shape[-2:]
    lead = img.shape[:-2]
    out = {}
    A = 4096 if img.dtype == np.uint16 else 256
    lg = np.empty(lead + (h, w, A), np.float32) if logits else None
    pb = np.empty(lead + (h, w, A), np.float32) if probs else None
    fq = np.empty(lead + (h, w, A), np.uint16) if freqs else None
    f = np.empty(lead + (h, w), np.uint32) if fc else None
    o = _opts(precision, group_rows, tile, meta, img.shape[0] if img.ndim == 3 else 0)
    _check(_L().dlic_debug_mlp(model.handle, img.ctypes.data, w, h, ctypes.byref(o),
                               lg.ctypes.data if logits else None, pb.ctypes.data if probs else None,
                               fq.ctypes.data if freqs else None, f.ctypes.data if fc else None))
    for k, v in (("logits", lg), ("probs", pb), ("freqs", fq), ("fc", f)):
        if v is not None:
            out[k] = v
    return out


# ------------------------------------------------------------------ device batch (torch memory/streams)
def _stream_handle(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return _vp(s.cuda_stream)


def dlic_encode_batch_device(model: Model, d_imgs, precision=PREC_BF16, group_rows=32, tile=(0, 0),
                             d_out=None, d_sizes=None, stream=None, meta=None, volume_depth=0):
    """d_imgs: torch uint8 (uint16 for a P12 model) CUDA tensor (n, H, W).  Returns (d_out, d_sizes, stride):
    container i occupies d_out[i*stride : i*stride + d_sizes[i]]."""
    import torch
    n, h, w = d_imgs.shape
    stride = dlic_max_container_bytes(w, h, precision, group_rows, tile, meta, volume_depth)
    if stride == 0:
        raise DlicError(1, "unsupported options")
    nc = n // volume_depth if volume_depth else n
    if d_out is None:
        d_out = torch.empty(nc * stride, dtype=torch.uint8, device=d_imgs.device)
    if d_sizes is None:
        d_sizes = torch.empty(nc, dtype=torch.int64, device=d_imgs.device)
    o = _opts(precision, group_rows, tile, meta, volume_depth)
    _check(_L().dlic_encode_batch_device(model.handle, _vp(d_imgs.data_ptr()), n, w, h, ctypes.byref(o),
                                         _vp(d_out.data_ptr()), d_out.numel(), _vp(d_sizes.data_ptr()),
                                         _stream_handle(stream)))
    return d_out, d_sizes, stride


def dlic_decode_batch_device(model: Model, d_bits, h_offsets, h_lengths, header: dict, d_imgs, d_status,
                             stream=None):
    """d_bits: torch uint8 CUDA tensor holding n containers at byte offsets
    h_offsets, each exactly h_lengths bytes (host ints); header: dlic_peek() of
    container 0; d_imgs: torch uint8 CUDA (n, H, W) output; d_status: int32
    CUDA (n,), zeroed by the caller (required: per-image errors land there)."""
    offs = np.ascontiguousarray(np.asarray(h_offsets, dtype=np.uint64))
    lens = np.ascontiguousarray(np.asarray(h_lengths, dtype=np.uint64))
    assert lens.shape == offs.shape
    hd = dlic_header()
    for k, _ in dlic_header._fields_:
        if k == "model_sha256":
            ctypes.memmove(hd.model_sha256, header["model_sha256"], 32)
        elif k == "meta":
            for i, v in enumerate(header.get("meta", [])):
                hd.meta[i] = float(v)
        else:
            setattr(hd, k, header.get(k, 8) if k == "bits" else header[k])
    _check(_L().dlic_decode_batch_device(model.handle, _vp(d_bits.data_ptr()), offs.ctypes.data, lens.ctypes.data,
                                         len(offs), ctypes.byref(hd), _vp(d_imgs.data_ptr()),
                                         _vp(d_status.data_ptr()) if d_status is not None else None,
                                         _stream_handle(stream)))


# ------------------------------------------------------------------ unit ranges (one image across GPUs)
def dlic_unit_streams(width, height, unit_lo, unit_hi, precision=PREC_BF16, group_rows=32, tile=(0, 0), meta=None):
    """(first_stream, n_streams) of units [unit_lo, unit_hi)."""
    a, b = ctypes.c_uint32(), ctypes.c_uint32()
    o = _opts(precision, group_rows, tile, meta)
    _check(_L().dlic_unit_streams(width, height, ctypes.byref(o), unit_lo, unit_hi, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def dlic_encode_units(model: Model, img: np.ndarray, unit_lo: int, unit_hi: int, precision=PREC_BF16,
                      group_rows=32, tile=(0, 0), meta=None):
    """Code units [unit_lo, unit_hi) of img -> (payload bytes, stream sizes list)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    _, ns = dlic_unit_streams(w, h, unit_lo, unit_hi, precision, group_rows, tile, meta)
    sizes = np.zeros(ns, np.uint32)
    out = c_u8p()
    n = ctypes.c_size_t()
    o = _opts(precision, group_rows, tile, meta)
    _check(_L().dlic_encode_units(model.handle, img.ctypes.data, w, h, w, ctypes.byref(o), unit_lo, unit_hi,
                                  ctypes.byref(out), ctypes.byref(n), sizes.ctypes.data))
    return _take(out, n.value), [int(x) for x in sizes]


def dlic_container_build(width, height, model_sha: bytes, stream_sizes, payload: bytes, precision=PREC_BF16,
                         group_rows=32, tile=(0, 0), meta=None) -> bytes:
    sz = np.ascontiguousarray(np.asarray(stream_sizes, dtype=np.uint32))
    out = c_u8p()
    n = ctypes.c_size_t()
    o = _opts(precision, group_rows, tile, meta)
    sha = ctypes.create_string_buffer(model_sha, 32)
    _check(_L().dlic_container_build(width, height, ctypes.byref(o), sha, sz.ctypes.data, len(sz), payload,
                                     len(payload), ctypes.byref(out), ctypes.byref(n)))
    return _take(out, n.value)


def dlic_decode_units(model: Model, bits: bytes, unit_lo: int, unit_hi: int, img: np.ndarray | None = None):
    """Decode units [unit_lo, unit_hi) into img (allocated zeroed if None)."""
    hd = dlic_peek(bits)
    if img is None:
        img = np.zeros((hd["height"], hd["width"]), np.uint8)
    assert img.flags.c_contiguous and img.dtype == np.uint8
    _check(_L().dlic_decode_units(model.handle, bits, len(bits), unit_lo, unit_hi, img.ctypes.data, img.size))
    return img


def dlic_encode_volume(model: Model, vol: np.ndarray, precision=PREC_BF16, group_rows=32, tile=(0, 0),
                       meta=None) -> bytes:
    """vol (D, H, W) u8 -> one volume container (3D window)."""
    vol = np.ascontiguousarray(vol, dtype=np.uint8)
    d, h, w = vol.shape
    out = c_u8p()
    n = ctypes.c_size_t()
    o = _opts(precision, group_rows, tile, meta)
    _check(_L().dlic_encode_volume(model.handle, vol.ctypes.data, w, h, d, ctypes.byref(o), ctypes.byref(out),
                                   ctypes.byref(n)))
    return _take(out, n.value)


def dlic_decode_volume(model: Model, bits: bytes) -> np.ndarray:
    hd = dlic_peek(bits)
    vol = np.empty((hd["depth"], hd["height"], hd["width"]), np.uint8)
    _check(_L().dlic_decode_volume(model.handle, bits, len(bits), vol.ctypes.data, vol.size))
    return vol


def dlic_numerics_rev() -> int:
    return int(_L().dlic_numerics_rev())


# ------------------------------------------------------------------ misc
def dlic_info() -> str:
    buf = ctypes.create_string_buffer(1024)
    _check(_L().dlic_info(buf, 1024))
    return buf.value.decode()


def dlic_set_timing(enable: bool):
    _L().dlic_set_timing(1 if enable else 0)


def dlic_last_kernel_ms(name: str) -> float:
    return float(_L().dlic_last_kernel_ms(name.encode()))
