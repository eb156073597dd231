"""GPU parity: the CUDA path (through the C-ABI) against the oracle.

Bars (north_star / DESIGN.md):
  * rANS fed the same integer tables -> bit-identical container bytes;
  * GPU decode reconstructs every image bit-exactly;
  * fp32 path logits within 1e-4 relative (per row, L_inf / max|logit|) of the
    fp64 oracle; bf16 path logits within BF16_TOL of the oracle's bf16
    emulation (tolerance derived in DESIGN.md);
  * integer tables == oracle Q1 of the GPU-exported probabilities (same
    precision decides the integer, fp32);
  * bf16-path payload bpp within +0.5% of the fp32 path.
"""

import numpy as np
import pytest

import synth
from oracle import codec, container, mlp, model_io, quant, streams, window

pytestmark = pytest.mark.gpu

# bf16 path vs the oracle's bf16 definition (per row, L_inf / max|logit|).
# Measured on 77k rows of the production encoder (scripts/measure_tol.py,
# profiles/r2_tol.txt): median 1.7e-7, p99 2.6e-7, p99.9 9.2e-4, max 3.6e-3.
# Rows whose bf16 activation roundings all agree with the oracle's differ only
# by the fp32 accumulation order (~1e-6); a row where one hidden activation
# rounds the other way (the fp32 sum sits within ~1e-6 of a bf16 midpoint)
# moves by up to 2^-8 |w a| / |z| per flip.  Bars: max 8e-3
# (2.2x the worst row seen) and p99 <= 1e-5 (the flip-free population).
BF16_TOL = 8e-3
BF16_P99 = 1e-5


@pytest.fixture(scope="module")
def dl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2207_05152_b200 as m
    return m


@pytest.fixture(scope="module")
def trained(dl, trained_blob):
    return dl.dlic_model_load(trained_blob, 0)


def _rand_tables(h, w, seed, alpha=0.3):
    rng = np.random.default_rng(seed)
    ft = np.zeros((h, w, 256), np.int64)
    img = np.zeros((h, w), np.uint8)
    for r in range(h):
        for c in range(w):
            p = rng.dirichlet(np.full(256, alpha)).astype(np.float32)
            ft[r, c] = quant.q1(p)
            img[r, c] = rng.choice(256, p=ft[r, c] / 65536)
    ct = np.cumsum(ft, -1) - ft
    idx = img.astype(np.int64)[..., None]
    fs = np.take_along_axis(ft, idx, -1)[..., 0]
    cs = np.take_along_axis(ct, idx, -1)[..., 0]
    return ft, img, fs, cs


@pytest.mark.parametrize("h,w,g,tile", [(1, 1, 32, (0, 0)), (7, 1, 1, (0, 0)), (1, 40, 32, (0, 0)),
                                         (33, 17, 32, (0, 0)), (45, 29, 4, (0, 0)), (40, 50, 8, (16, 12)),
                                         (64, 96, 16, (0, 0)), (20, 9, 2, (5, 7))])
def test_rans_bit_exact_vs_oracle_same_tables(dl, h, w, g, tile):
    ft, img, fs, cs = _rand_tables(h, w, seed=h * 1000 + w)
    sha = bytes(range(32))
    ob = codec.encode_with_tables(fs, cs, w, h, 1, g, tile[0], tile[1], sha, dl.dlic_numerics_rev())
    fc = (fs | (cs << 16)).astype(np.uint32)
    gb = dl.dlic_rans_encode_tables(fc, precision=1, group_rows=g, tile=tile, model_sha=sha)
    assert gb == ob
    # GPU decode of the oracle's stream, fed the same full tables
    assert np.array_equal(dl.dlic_rans_decode_tables(ob, ft.astype(np.uint16)), img)
    # and the oracle decodes it too (self-check of the fixture)
    assert np.array_equal(codec.decode_with_tables(ob, ft), img)


def test_rans_decode_detects_corruption(dl):
    ft, img, fs, cs = _rand_tables(24, 20, seed=5)
    ob = codec.encode_with_tables(fs, cs, 20, 24, 1, 8, 0, 0, bytes(32), dl.dlic_numerics_rev())
    hdr = container.parse(ob)
    bad = bytearray(ob)
    bad[hdr["header_bytes"] + 6] ^= 0x10
    with pytest.raises(dl.DlicError):
        dl.dlic_rans_decode_tables(bytes(bad), ft.astype(np.uint16))


def _oracle_logits(layers, img, prec, rows=None, cols=None):
    h, w = img.shape
    if rows is None:
        rows, cols = np.divmod(np.arange(h * w), w)
    x = window.features(window.gather_many(img, rows, cols))
    return mlp.forward_fp64(layers, x) if prec == 0 else mlp.forward_bf16(layers, x)


@pytest.mark.parametrize("prec", [0, 1])
def test_mlp_logits_vs_oracle(dl, trained, trained_blob, prec):
    layers = model_io.load(trained_blob)
    img = synth.natural_like(61, 37, seed=11)      # several 128-pixel tiles, ragged tail
    out = dl.dlic_debug_mlp(trained, img, precision=prec)
    ref = _oracle_logits(layers, img, prec).reshape(37, 61, 256)
    rel = np.abs(out["logits"] - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)
    tol = 1e-4 if prec == 0 else BF16_TOL
    assert rel.max() <= tol, (prec, float(rel.max()))
    if prec == 1:
        assert np.quantile(rel, 0.99) <= BF16_P99, float(np.quantile(rel, 0.99))
    # integer tables follow exactly from the exported probabilities (fp32 decides)
    f_or = quant.q1(out["probs"].reshape(-1, 256)).reshape(37, 61, 256)
    assert np.array_equal(out["freqs"].astype(np.int64), f_or)
    # probabilities are the softmax of the exported logits
    p_ref = quant.softmax_fp64(out["logits"].astype(np.float64))
    assert np.abs(out["probs"] - p_ref).max() < 2e-6
    # fc of the true symbol agrees with the exported table
    c = np.cumsum(f_or, -1) - f_or
    idx = img.astype(np.int64)[..., None]
    assert np.array_equal(out["fc"] & 0xFFFF, np.take_along_axis(f_or, idx, -1)[..., 0])
    assert np.array_equal(out["fc"] >> 16, np.take_along_axis(c, idx, -1)[..., 0])


def test_tiled_mlp_uses_tile_borders(dl, trained, trained_blob):
    layers = model_io.load(trained_blob)
    img = synth.natural_like(40, 30, seed=3)
    out = dl.dlic_debug_mlp(trained, img, precision=0, tile=(16, 12), probs=False, freqs=False, fc=False)
    ref = np.zeros((30, 40, 256))
    for (x0, y0, tw, th) in container.tiles(40, 30, 16, 12):
        sub = np.ascontiguousarray(img[y0:y0 + th, x0:x0 + tw])
        ref[y0:y0 + th, x0:x0 + tw] = _oracle_logits(layers, sub, 0).reshape(th, tw, 256)
    rel = np.abs(out["logits"] - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)
    assert rel.max() <= 1e-4


@pytest.mark.parametrize("prec", [1, 0])
@pytest.mark.parametrize("h,w,g,tile", [(1, 1, 32, (0, 0)), (1, 13, 32, (0, 0)), (9, 1, 4, (0, 0)),
                                         (5, 8, 1, (0, 0)), (32, 32, 32, (0, 0)), (70, 45, 16, (0, 0)),
                                         (50, 70, 32, (24, 20)), (130, 40, 8, (0, 0))])
def test_roundtrip_and_oracle_bytes(dl, trained, trained_blob, prec, h, w, g, tile):
    img = synth.natural_like(w, h, seed=h + 7 * w)
    bits = dl.dlic_encode(trained, img, precision=prec, group_rows=g, tile=tile)
    assert np.array_equal(dl.dlic_decode(trained, bits), img)
    fc = dl.dlic_debug_mlp(trained, img, precision=prec, group_rows=g, tile=tile, logits=False, probs=False,
                           freqs=False)["fc"]
    ob = codec.encode_with_tables((fc & 0xFFFF).astype(np.int64), (fc >> 16).astype(np.int64), w, h, prec, g,
                                  tile[0], tile[1], model_io.digest(trained_blob), dl.dlic_numerics_rev())
    assert ob == bits
    hd = dl.dlic_peek(bits)
    assert hd["precision"] == prec and hd["group_rows"] == g and hd["header_bytes"] + hd["payload_bytes"] == len(bits)


def test_wide_unit_uses_clusters(dl, trained):
    # W = 700 -> 234 rows per front -> 4-CTA cluster (64 slots each); W = 1100 -> 367 rows -> 8 CTAs
    for w, h in ((700, 40), (1100, 24)):
        img = synth.natural_like(w, h, seed=w)
        for prec in (1, 0):
            bits = dl.dlic_encode(trained, img, precision=prec)
            assert np.array_equal(dl.dlic_decode(trained, bits), img)


def test_gpu_stream_decodes_with_oracle_given_gpu_tables(dl, trained):
    img = synth.natural_like(48, 40, seed=21)
    bits = dl.dlic_encode(trained, img, precision=1, group_rows=8)
    ft = dl.dlic_debug_mlp(trained, img, precision=1, group_rows=8, logits=False, probs=False, fc=False)["freqs"]
    assert np.array_equal(codec.decode_with_tables(bits, ft.astype(np.int64)), img)


def test_determinism_and_faults(dl, trained, trained_blob):
    img = synth.natural_like(64, 48, seed=9)
    a = dl.dlic_encode(trained, img)
    assert a == dl.dlic_encode(trained, img) == dl.dlic_encode(trained, img)
    other = dl.dlic_model_load(model_io.save(synth.he_uniform_layers(mlp.P100K, seed=99)), 0)
    with pytest.raises(dl.DlicError) as e:
        dl.dlic_decode(other, a)
    assert e.value.status == 7
    hd = dl.dlic_peek(a)
    rng = np.random.default_rng(0)
    caught = 0
    for _ in range(10):
        bad = bytearray(a)
        pos = int(rng.integers(hd["header_bytes"], len(a)))
        bad[pos] ^= 1 << int(rng.integers(0, 8))
        try:
            out = dl.dlic_decode(trained, bytes(bad))
            caught += int(not np.array_equal(out, img)) and 0
        except dl.DlicError:
            caught += 1
    assert caught >= 9
    with pytest.raises(dl.DlicError):
        dl.dlic_decode(trained, a[:-2])


def test_c2_full_size_bf16_roundtrip_sampled_oracle_and_bpp_gate(dl, trained, trained_blob):
    """BASELINE configs[1] at full size in the bench's launch configuration."""
    layers = model_io.load(trained_blob)
    img = synth.config_images("C2", count=1)[0]
    b16 = dl.dlic_encode(trained, img, precision=1)
    b32 = dl.dlic_encode(trained, img, precision=0)
    assert np.array_equal(dl.dlic_decode(trained, b16), img)
    assert np.array_equal(dl.dlic_decode(trained, b32), img)
    p16 = dl.dlic_peek(b16)["payload_bytes"]
    p32 = dl.dlic_peek(b32)["payload_bytes"]
    assert p16 <= 1.005 * p32, (p16, p32)            # bf16 gate (north_star, Q18)
    # sampled oracle check at full size: 512 pixels
    rng = np.random.default_rng(0)
    sel = rng.choice(img.size, 512, replace=False)
    rows, cols = np.divmod(sel, img.shape[1])
    out = dl.dlic_debug_mlp(trained, img, precision=1, probs=False, freqs=False, fc=False)
    g = out["logits"][rows, cols]
    ref = _oracle_logits(layers, img, 1, rows, cols)
    rel = np.abs(g - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)
    assert rel.max() <= BF16_TOL and np.quantile(rel, 0.99) <= BF16_P99


def test_batch_device_api_matches_single(dl, trained):
    import torch
    imgs = synth.mri_like_slices(6, 256, seed0=3)[:, :96, :80].copy()
    d_imgs = torch.from_numpy(imgs).cuda()
    d_out, d_sizes, stride = dl.dlic_encode_batch_device(trained, d_imgs, precision=1)
    torch.cuda.synchronize()
    sizes = d_sizes.cpu().numpy()
    host = d_out.cpu().numpy()
    offs = []
    for i in range(6):
        single = dl.dlic_encode(trained, imgs[i], precision=1)
        got = host[i * stride: i * stride + sizes[i]].tobytes()
        assert got == single
        offs.append(i * stride)
    hdr = dl.dlic_peek(host[:sizes[0]].tobytes())
    d_dec = torch.empty_like(d_imgs)
    d_st = torch.zeros(6, dtype=torch.int32, device="cuda")
    dl.dlic_decode_batch_device(trained, d_out, offs, [int(x) for x in sizes], hdr, d_dec, d_st)
    torch.cuda.synchronize()
    assert d_st.cpu().numpy().tolist() == [0] * 6
    assert np.array_equal(d_dec.cpu().numpy(), imgs)


def test_host_batch_api_matches_single(dl, trained, trained_blob):
    """dlic_encode_batch / dlic_decode_batch: each container byte-identical to a
    single-image dlic_encode (images are independent units); lossless decode;
    the model hash is checked before pixel work."""
    imgs = synth.mri_like_slices(5, 256, seed0=4)[:, :70, :90].copy()
    blob, sizes = dl.dlic_encode_batch(trained, imgs, precision=1, tile=(40, 32))
    assert sum(sizes) == len(blob)
    off = 0
    for i in range(5):
        assert blob[off:off + sizes[i]] == dl.dlic_encode(trained, imgs[i], precision=1, tile=(40, 32))
        off += sizes[i]
    assert np.array_equal(dl.dlic_decode_batch(trained, blob, sizes), imgs)
    other = dl.dlic_model_load(model_io.save(synth.he_uniform_layers(mlp.P100K, seed=98)), 0)
    with pytest.raises(dl.DlicError) as e:
        dl.dlic_decode_batch(other, blob, sizes)
    assert e.value.status == 7
    bad = bytearray(blob)
    bad[sizes[0] + dl.dlic_peek(blob[sizes[0]:sizes[0] + sizes[1]])["header_bytes"] + 3] ^= 0x40   # payload of image 1
    with pytest.raises(dl.DlicError):
        dl.dlic_decode_batch(trained, bytes(bad), sizes)
