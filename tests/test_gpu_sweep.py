"""GPU coverage of the configurations round 1 left untested (VERDICT r1 "What's
weak" 4), through the C-ABI:

  * a seeded random sweep of 112 shapes across every decode-cluster boundary
    (slots = ceil(W/3) against 64 * nc: W = 192/193, 384/385, 768/769,
    1536/1537 and 3072, i.e. 1, 2, 4, 8 and 16 CTAs), H from 1 to ~600, every
    G, tiles on and off, both precisions -- lossless round trip everywhere,
    container byte-identical to the oracle's coder fed the GPU tables where
    the pure-Python oracle is fast enough;
  * the untiled C4 image (1920x1080: 640 rows per front -> a 16-CTA
    non-portable cluster) with the oracle-byte check;
  * C2 decoded 50 times while a bf16 GEMM stream keeps the other SMs busy;
  * the unit-range calls (one image's tiles split as across GPUs) against the
    whole-image container;
  * the container's numerics revision and the device decoder's length checks
    (a corrupt size table must never make the decoder read outside its
    container);
  * the production encoder's debug tap against the production run.
The wavefront ordering these cover is P:87; the per-row coder instances P:103.
"""

import numpy as np
import pytest

import synth
from oracle import codec, container, model_io

pytestmark = pytest.mark.gpu


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


def _sweep_cases(n=112, seed=2024):
    """Deterministic shapes: cluster-boundary widths first, then random ones."""
    rng = np.random.default_rng(seed)
    widths = [1, 2, 3, 8, 9, 10, 191, 192, 193, 194, 383, 384, 385, 386, 767, 768, 769, 770,
              1535, 1536, 1537, 1538, 2200, 3070, 3071, 3072]
    cases = []
    for i in range(n):
        w = widths[i] if i < len(widths) else int(rng.integers(1, 1100))
        if i < len(widths):   # boundary widths: tall enough to fill several CTAs' slots, or short
            hmax = max(1, min(600, 600_000 // w))
            h = hmax if i % 2 == 0 else int(rng.integers(1, 40))
        else:
            hmax = max(1, min(600, 250_000 // w))
            h = int(rng.choice([1, 2, 3, int(rng.integers(1, hmax + 1)), hmax])) if i % 3 else int(rng.integers(1, 40))
        g = int(rng.choice([1, 2, 4, 8, 16, 32]))
        tiled = rng.random() < 0.3 and w > 4 and h > 4
        tile = (int(rng.integers(3, w)), int(rng.integers(3, h))) if tiled else (0, 0)
        while -(-(tile[1] or h) // g) > 200:   # the decoder keeps <= ~250 group cursors in shared memory
            g *= 2
        # fp32 (CUDA-core engine, ~0.14 ms per front) only on shapes with few fronts
        prec = 0 if (rng.random() < 0.25 and w + 3 * h < 1500) else 1
        kind = rng.choice(["natural", "uniform", "smooth", "const"])
        cases.append((w, h, g, tile, prec, str(kind), i))
    return cases


def _img(w, h, kind, seed):
    if kind == "natural":
        return synth.natural_like(w, h, seed=seed)
    if kind == "const":
        return np.full((h, w), seed % 256, np.uint8)
    return synth.random_image(w, h, seed=seed, kind=kind)


@pytest.mark.parametrize("w,h,g,tile,prec,kind,i", _sweep_cases())
def test_random_shape_sweep(dl, trained, trained_blob, w, h, g, tile, prec, kind, i):
    img = _img(w, h, kind, i)
    bits = dl.dlic_encode(trained, img, precision=prec, group_rows=g, tile=tile)
    assert np.array_equal(dl.dlic_decode(trained, bits), img)
    hd = dl.dlic_peek(bits)
    assert (hd["width"], hd["height"], hd["group_rows"], hd["precision"]) == (w, h, g, prec)
    assert hd["numerics"] == dl.dlic_numerics_rev()
    if w * h <= 40_000:   # the pure-Python oracle coder: ~0.1 s per 10k px
        fc = dl.dlic_debug_mlp(trained, img, precision=prec, group_rows=g, tile=tile, logits=False, probs=False,
                               freqs=False)["fc"]
        ob = codec.encode_with_tables((fc & 0xFFFF).astype(np.int64), (fc >> 16).astype(np.int64), w, h, prec, g,
                                      tile[0], tile[1], model_io.digest(trained_blob), dl.dlic_numerics_rev())
        assert ob == bits


def test_too_many_groups_per_unit_is_rejected_up_front(dl, trained):
    img = synth.natural_like(8, 600, seed=1)
    assert dl.dlic_max_container_bytes(8, 600, 1, 1) == 0
    with pytest.raises(dl.DlicError) as e:
        dl.dlic_encode(trained, img, precision=1, group_rows=1)
    assert e.value.status == 1
    assert np.array_equal(dl.dlic_decode(trained, dl.dlic_encode(trained, img, group_rows=4)), img)


def test_c4_untiled_16_cta_cluster(dl, trained, trained_blob):
    """1920x1080 as ONE unit: ceil(1920/3) = 640 rows on the widest front ->
    nc = 16 CTAs of 64 slots (non-portable cluster size)."""
    img = synth.config_images("C4", count=1)[0]
    bits = dl.dlic_encode(trained, img, precision=1)
    assert np.array_equal(dl.dlic_decode(trained, bits), img)
    fc = dl.dlic_debug_mlp(trained, img, precision=1, logits=False, probs=False, freqs=False)["fc"]
    ob = codec.encode_with_tables((fc & 0xFFFF).astype(np.int64), (fc >> 16).astype(np.int64), 1920, 1080, 1, 32,
                                  0, 0, model_io.digest(trained_blob), dl.dlic_numerics_rev())
    assert ob == bits


def test_c2_decode_stress_under_concurrent_gemms(dl, trained):
    """50 decodes of C2 while another stream runs bf16 GEMMs on the same GPU:
    the decoder's cross-CTA ordering (cluster barriers, DSMEM halo, TMEM
    double buffers) must not depend on timing."""
    import torch
    img = synth.config_images("C2", count=1)[0]
    bits = dl.dlic_encode(trained, img, precision=1)
    noise = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    with torch.cuda.stream(noise):
        for _ in range(3000):          # ~0.1 ms each: longer than the 50 decodes
            c = a @ b
    for k in range(50):
        out = dl.dlic_decode(trained, bits)
        assert np.array_equal(out, img), k
    noise.synchronize()
    del c


def test_unit_range_calls_match_whole_image(dl, trained, trained_blob):
    """C4 in 384x360 tiles (15 units) split into 3 unit ranges, as 3 GPUs
    would code it: payloads + sizes framed by dlic_container_build equal the
    single-call container; each range decodes its own tiles only."""
    img = synth.config_images("C4", count=1)[0]
    tile = (384, 360)
    whole = dl.dlic_encode(trained, img, precision=1, tile=tile)
    n_units = dl.dlic_peek(whole)["n_units"]
    assert n_units == 15
    ranges = [(0, 4), (4, 9), (9, 15)]
    payload, sizes = b"", []
    for lo, hi in ranges:
        p, s = dl.dlic_encode_units(trained, img, lo, hi, precision=1, tile=tile)
        assert sum(s) == len(p)
        payload += p
        sizes += s
    built = dl.dlic_container_build(1920, 1080, model_io.digest(trained_blob), sizes, payload, 1, 32, tile)
    assert built == whole
    out = np.zeros_like(img)
    for lo, hi in ranges:
        dl.dlic_decode_units(trained, whole, lo, hi, out)
    assert np.array_equal(out, img)
    part = dl.dlic_decode_units(trained, whole, 4, 9)        # only tiles 4..8 are written
    tiles = container.tiles(1920, 1080, *tile)
    for u, (x0, y0, tw, th) in enumerate(tiles):
        got = part[y0:y0 + th, x0:x0 + tw]
        if 4 <= u < 9:
            assert np.array_equal(got, img[y0:y0 + th, x0:x0 + tw])
        else:
            assert not got.any()


def test_numerics_revision_is_checked_before_pixel_work(dl, trained):
    img = synth.natural_like(64, 40, seed=4)
    bits = bytearray(dl.dlic_encode(trained, img))
    assert bits[22] | (bits[23] << 8) == dl.dlic_numerics_rev()
    bits[22] ^= 1
    with pytest.raises(dl.DlicError) as e:
        dl.dlic_decode(trained, bytes(bits))
    assert e.value.status == 5
    with pytest.raises(dl.DlicError) as e:
        dl.dlic_decode_batch(trained, bytes(bits), [len(bits)])
    assert e.value.status == 5


def test_device_decode_checks_lengths_and_size_tables(dl, trained):
    """a truncated container or a corrupt size table must be
    reported in d_status, never read past the container."""
    import torch
    imgs = synth.mri_like_slices(3, 256, seed0=8)[:, :64, :96].copy()
    d_imgs = torch.from_numpy(imgs).cuda()
    d_out, d_sizes, stride = dl.dlic_encode_batch_device(trained, d_imgs, precision=1)
    torch.cuda.synchronize()
    sizes = [int(x) for x in d_sizes.cpu()]
    hdr = dl.dlic_peek(d_out[:sizes[0]].cpu().numpy().tobytes())
    offs = [i * stride for i in range(3)]
    d_dec = torch.zeros_like(d_imgs)
    # (a) container 1 declared 2 bytes short
    st = torch.zeros(3, dtype=torch.int32, device="cuda")
    dl.dlic_decode_batch_device(trained, d_out, offs, [sizes[0], sizes[1] - 2, sizes[2]], hdr, d_dec, st)
    torch.cuda.synchronize()
    s = st.cpu().tolist()
    assert s[0] == 0 and s[2] == 0 and s[1] == 6
    # (b) container 2's first stream size rewritten to a huge value
    bad = d_out.clone()
    o = offs[2] + 60
    bad[o:o + 4] = torch.tensor([0xF0, 0xFF, 0xFF, 0x7F], dtype=torch.uint8)
    st.zero_()
    dl.dlic_decode_batch_device(trained, bad, offs, sizes, hdr, d_dec, st)
    torch.cuda.synchronize()
    s = st.cpu().tolist()
    assert s[0] == 0 and s[1] == 0 and s[2] != 0
    # the context is healthy afterwards: a clean decode still works
    st.zero_()
    dl.dlic_decode_batch_device(trained, d_out, offs, sizes, hdr, d_dec, st)
    torch.cuda.synchronize()
    assert st.cpu().tolist() == [0, 0, 0] and torch.equal(d_dec, d_imgs)
    with pytest.raises(dl.DlicError) as e:        # d_status is required
        dl.dlic_decode_batch_device(trained, d_out, offs, sizes, hdr, d_dec, None)
    assert e.value.status == 1


def test_production_encoder_debug_tap_equals_production_run(dl, trained):
    """dlic_debug_mlp's bf16 exports come from k_enc_pp<DBG=true>; the tables
    it reports for the true symbols are exactly what the production launch
    (k_enc_pp<false>, no exports) codes."""
    for (w, h, tile) in ((61, 37, (0, 0)), (130, 70, (40, 32))):
        img = synth.natural_like(w, h, seed=w)
        full = dl.dlic_debug_mlp(trained, img, precision=1, tile=tile)
        prod = dl.dlic_debug_mlp(trained, img, precision=1, tile=tile, logits=False, probs=False, freqs=False)
        assert np.array_equal(full["fc"], prod["fc"])
        f = full["freqs"].astype(np.int64)
        c = np.cumsum(f, -1) - f
        idx = img.astype(np.int64)[..., None]
        assert np.array_equal(prod["fc"] & 0xFFFF, np.take_along_axis(f, idx, -1)[..., 0])
        assert np.array_equal(prod["fc"] >> 16, np.take_along_axis(c, idx, -1)[..., 0])
