"""Pins for the oracle codec, container and model file: losslessness,
wavefront == raster equivalence, uniform-model rate, rate consistency,
fault detection."""

import numpy as np
import pytest

import synth
from oracle import codec, container, mlp, model_io, quant, rans, streams, train


def _small_model(seed, dims=(78, 16, 16, 256)):
    return model_io.save(synth.he_uniform_layers(dims, seed=seed, bias_scale=0.3))


@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (6, 1), (5, 8), (13, 9), (33, 20), (40, 3)])
def test_roundtrip_shapes(shape):
    h, w = shape
    blob = _small_model(h * 100 + w)
    img = synth.random_image(w, h, seed=h + w, kind="smooth")
    for prec in (0, 1):
        for g in sorted({1, 3, 32, h}):
            b = codec.encode(img, blob, prec, g)
            assert np.array_equal(codec.decode(b, blob), img)


def test_roundtrip_random_models_and_tiles():
    rng = np.random.default_rng(0)
    for i in range(8):
        h, w = (int(v) for v in rng.integers(2, 30, 2))
        blob = _small_model(1000 + i)
        img = synth.random_image(w, h, seed=i, kind=["uniform", "smooth", "const"][i % 3])
        tw, th = int(rng.integers(1, w + 1)), int(rng.integers(1, h + 1))
        b = codec.encode(img, blob, i % 2, int(rng.integers(1, 9)), tw, th)
        hdr = container.parse(b)
        assert len(hdr["streams"]) == sum(streams.n_groups(t[3], hdr["group_rows"])
                                           for t in container.tiles(w, h, tw, th))
        assert np.array_equal(codec.decode(b, blob), img)


def test_raster_decoder_equals_wavefront_decoder():
    blob = _small_model(7)
    img = synth.random_image(19, 14, seed=7, kind="smooth")
    b = codec.encode(img, blob, 0, 1)
    assert np.array_equal(codec.raster_decode(b, blob), img)
    assert np.array_equal(codec.decode(b, blob), img)


def test_uniform_model_costs_eight_bits_per_pixel():
    blob = model_io.save(synth.zero_layers(mlp.P100K))
    img = synth.random_image(37, 21, seed=3)
    b = codec.encode(img, blob, 0, 32)
    hdr = container.parse(b)
    payload = sum(len(s) for s in hdr["streams"])
    lanes = 21
    # uniform p: f = 255 (511 for symbol 255): log2(65536/255) = 8.0056 bits per
    # symbol (exactly 8 - log2(255/256) for every symbol of this image below 255);
    # per-lane flush overhead in (2, 4] bytes
    info = sum(16 - np.log2(511 if v == 255 else 255) for v in img.reshape(-1)) / 8
    assert info + 2 * lanes - 1 <= payload <= info + 4 * lanes + 1
    assert np.array_equal(codec.decode(b, blob), img)


def test_encode_with_tables_equals_encode_and_is_deterministic():
    blob = _small_model(9)
    img = synth.random_image(20, 11, seed=9, kind="smooth")
    layers = model_io.load(blob)
    fs, cs = codec.unit_tables_by_front(layers, 0, img)
    a = codec.encode_with_tables(fs, cs, 20, 11, 0, 4, 0, 0, model_io.digest(blob))
    assert a == codec.encode(img, blob, 0, 4) == codec.encode(img, blob, 0, 4)


def test_decode_with_tables_matches():
    blob = _small_model(10)
    img = synth.random_image(15, 12, seed=10, kind="smooth")
    b = codec.encode(img, blob, 1, 5)
    layers = model_io.load(blob)
    _, _, f, _ = codec.all_pixel_tables(layers, 1, img)
    assert np.array_equal(codec.decode_with_tables(b, f.reshape(12, 15, 256)), img)


def test_fault_detection():
    blob = _small_model(11)
    other = _small_model(12)
    img = synth.random_image(24, 16, seed=11, kind="smooth")
    b = codec.encode(img, blob, 0, 8)
    with pytest.raises(codec.ModelHashMismatch):
        codec.decode(b, other)
    hdr = container.parse(b)
    rng = np.random.default_rng(11)
    detected = 0
    for _ in range(20):
        bad = bytearray(b)
        pos = int(rng.integers(hdr["header_bytes"], len(b)))
        bad[pos] ^= 1 << int(rng.integers(0, 8))
        try:
            out = codec.decode(bytes(bad), blob)
            detected += int(not np.array_equal(out, img)) * 0
        except (streams.CorruptStream, rans.Underflow, AssertionError):
            detected += 1
    assert detected >= 18
    with pytest.raises(container.CorruptContainer):
        codec.decode(b[:-2], blob)
    with pytest.raises(container.CorruptContainer):
        container.parse(b"XLIC" + b[4:])


def test_model_file_roundtrip_and_corruption():
    layers = synth.he_uniform_layers(mlp.P100K, seed=1)
    blob = model_io.save(layers)
    back = model_io.load(blob)
    assert all(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) for a, b in zip(layers, back))
    assert len(blob) == 8 + 2 + 6 * 10 + 4 * mlp.n_params(mlp.P100K) + 2 + 32
    bad = bytearray(blob)
    bad[100] ^= 4
    with pytest.raises(model_io.CorruptModel):
        model_io.load(bytes(bad))


def test_trained_fixture_rate_consistency(trained_blob):
    """Payload bpp <= vloss + 0.05 + flush overhead; P:110 vloss
    "indicative for the compression performance ... excluding header"."""
    layers = model_io.load(trained_blob)
    img = synth.natural_like(96, 64, seed=4242)
    x, y = train.dataset([img])
    vl = train.vloss_bits(layers, x, y)
    b = codec.encode(img, trained_blob, 0, 32)
    hdr = container.parse(b)
    payload_bits = 8 * sum(len(s) for s in hdr["streams"])
    n = img.size
    assert payload_bits / n <= vl + 0.05 + 32 * 64 / n
    assert vl < 6.0            # briefly trained: well below the 8-bit uniform cost
    assert np.array_equal(codec.decode(b, trained_blob), img)


def test_q1_tables_from_logits_shapes():
    lg = np.zeros((3, 256), np.float32)
    p, f, c = quant.tables_from_logits(lg)
    assert np.all(f[:, :255] == 255) and np.all(f[:, 255] == 511) and np.all(c[:, 1] == 255)
