"""Oracle pins for the 12-bit alphabet (§8(f) f3).

P:184-186 — MRI "information is captured in one 12-bit channel, leading to
4096 possible shades of gray"; P:207-208 — "our final model has 4096 output
layer neurons".  Readings: R15 features v / 4096; R16 the network
P12 = 78 -> 256x5 -> 4096; R17 the table Q1' with n = 4096 and a 64-unit
guard (scale 61376); container byte 7 = 12.

Pins independent of the oracle's own formulas: hand-derived tables for the
uniform and one-hot PDFs, brute-force window features, the information
content of a uniform model in closed form, exhaustive round trips, and the
sequential raster decoder against the wavefront decoder.
"""

import math

import numpy as np
import pytest

import synth
from oracle import codec, container, mlp, model_io, quant, window


def test_q1_4096_uniform_pdf_by_hand():
    # p_i = 2^-12 exactly; 2^-12 * 61376 = 14.984375 exactly -> f = 1 + 14 = 15;
    # sum = 4096 * 15 = 61440, residual 4096 on the last symbol
    f = quant.q1(np.full(4096, 2.0 ** -12, np.float32))
    assert f[:4095].tolist() == [15] * 4095 and f[4095] == 15 + 4096
    c = quant.cdf(f)
    assert c[0] == 0 and c[4095] == 15 * 4095


def test_q1_4096_one_hot_shows_the_guard():
    # p_0 = 1: f_0 = 1 + 61376, others 1; sum 61377 + 4095 = 65472 -> R = 64
    p = np.zeros(4096, np.float32)
    p[0] = 1.0
    f = quant.q1(p)
    assert f[0] == 61377 and f[4095] == 1 + 64 and np.all(f[1:4095] == 1)


def test_q1_8bit_scale_unchanged():
    # the 8-bit definition keeps guard 1 (scale 65279): one-hot -> f_7 = 65280,
    # 255 ones: sum 65535, residual 1 on symbol 255
    p = np.zeros(256, np.float32)
    p[7] = 1.0
    f = quant.q1(p)
    assert f[7] == 65280 and f[255] == 2 and f.sum() == 65536


def test_q1_4096_total_and_floor_on_fp32_softmaxes():
    rng = np.random.default_rng(3)
    for scale in (0.1, 3.0, 20.0, 200.0):
        lg = (rng.standard_normal((64, 4096)) * scale).astype(np.float32)
        p = quant.softmax_fp64(lg).astype(np.float32)
        f = quant.q1(p)
        assert np.all(f.sum(-1) == 65536) and np.all(f >= 1)


def test_features_12bit_brute_force():
    img = np.arange(4096, dtype=np.uint16).reshape(64, 64)
    rows, cols = np.divmod(np.arange(64 * 64), 64)
    x = window.net_inputs(img, rows, cols, bits=12)
    for k in (0, 65, 2000, 4095):
        r, c = divmod(k, 64)
        want = [(img[r + dr, c + dc] if 0 <= r + dr < 64 and 0 <= c + dc < 64 else 0) / 4096.0
                for dr, dc in window.OFFSETS]
        assert x[k].tolist() == want


def test_bf16_definition_rounds_12bit_inputs():
    # 4095/4096 = 1 - 2^-12 has 12 significant bits: RN to bf16 gives 1.0;
    # 257/4096 = 2^-4 (1 + 2^-8) is a tie -> even -> 2^-4
    assert mlp.bf16_round(np.array([4095 / 4096.0]))[0] == 1.0
    assert mlp.bf16_round(np.array([257 / 4096.0]))[0] == 0.0625
    assert mlp.bf16_round(np.array([384 / 4096.0]))[0] == 384 / 4096.0


def _small12(seed=0, bias_scale=0.1):
    return synth.he_uniform_layers((78, 16, 16, 16, 16, 16, 4096), seed=seed, bias_scale=bias_scale)


def test_p12_parameter_count():
    assert mlp.n_params(mlp.P12) == 1_336_064


def test_uniform_model_information_content_closed_form():
    # zero weights and biases: every table is the uniform one above, so the
    # information content is sum_s (16 - log2 f_s) with f = 15 (4111 for 4095)
    img = synth.mri_like_volume(24, 1, seed=2, bits=12)[0]
    img[0, 0] = 4095
    blob = model_io.save(synth.zero_layers((78, 8, 8, 8, 8, 8, 4096)))
    fs, _ = codec.unit_tables_by_front(model_io.load_net(blob), 0, img)
    want = sum(16 - math.log2(4111 if v == 4095 else 15) for v in img.ravel())
    assert codec.payload_bits_estimate(fs) == pytest.approx(want, rel=1e-12)
    bits = codec.encode(img, blob, 0, 1)
    hdr = container.parse(bits)
    payload = sum(len(s) for s in hdr["streams"])
    # rANS: within 2 flushed words per row + <1 word per row of slack
    assert 8 * payload >= want and 8 * payload <= want + 24 * (32 + 16)


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("h,w,g,tile", [(9, 13, 1, (0, 0)), (17, 11, 4, (0, 0)), (12, 20, 2, (8, 7))])
def test_12bit_roundtrip(prec, h, w, g, tile):
    img = synth.mri_like_volume(max(h, w), 1, seed=h * w, bits=12)[0][:h, :w].copy()
    img[0, -1] = 4095
    blob = model_io.save(_small12(seed=h))
    bits = codec.encode(img, blob, prec, g, *tile)
    assert bits[7] == 12 and container.parse(bits)["bits"] == 12
    out = codec.decode(bits, blob)
    assert out.dtype == np.uint16 and np.array_equal(out, img)


def test_12bit_raster_decoder_matches_wavefront():
    img = synth.mri_like_volume(16, 1, seed=5, bits=12)[0][:7, :10].copy()
    blob = model_io.save(_small12(seed=1))
    bits = codec.encode(img, blob, 0, 1)
    assert np.array_equal(codec.raster_decode(bits, blob), img)


def test_12bit_tables_decoder_and_alphabet_checks():
    img = synth.mri_like_volume(16, 1, seed=6, bits=12)[0][:8, :9].copy()
    blob = model_io.save(_small12(seed=2))
    bits = codec.encode(img, blob, 1, 2)
    _, _, f, _ = codec.all_pixel_tables(model_io.load_net(blob), 1, img)
    assert np.array_equal(codec.decode_with_tables(bits, f.reshape(8, 9, 4096)), img)
    with pytest.raises(ValueError):                       # value outside the alphabet
        bad = img.copy()
        bad[0, 0] = 4096
        codec.encode(bad, blob)
    as8 = bytearray(bits)
    as8[7] = 0                                            # the header claims 8-bit pixels
    with pytest.raises(container.CorruptContainer):       # ... but the model has 4096 outputs
        codec.decode(bytes(as8), blob)
    blob8 = model_io.save(synth.he_uniform_layers((78, 8, 8, 8, 8, 8, 256), seed=0))
    with pytest.raises(ValueError):                       # 12-bit pixels need 4096 outputs
        codec.encode(img, blob8)


def test_8bit_containers_keep_byte7_zero():
    img = synth.natural_like(10, 6, seed=1)
    blob = model_io.save(synth.he_uniform_layers((78, 8, 8, 8, 8, 8, 256), seed=0))
    bits = codec.encode(img, blob)
    assert bits[7] == 0 and container.parse(bits)["bits"] == 8
    bad = bytearray(bits)
    bad[7] = 11
    with pytest.raises(container.CorruptContainer):
        container.parse(bytes(bad))
