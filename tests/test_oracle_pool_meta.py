"""Pins for the §8(f) f4 additions to the oracle: optional average pooling
between dense layers ("two optional pooling layers"; reading R11 = SPEC
S:249) and metadata input features (reading R12 = SPEC S:252).
Hand-derived values, special cases that reduce to the unpooled / metadata-free
network, and the container's uncompressed metadata block."""

import numpy as np
import pytest

import synth
from oracle import codec, container, mlp, model_io, window


def test_avg_pool_hand_derived():
    # x = [1, 2]; z1 = [1, 2, 2, 4] - [0, 0, 3, 0] -> relu -> [1, 2, 0, 4];
    # pool g = 2 (contiguous pairs) -> [1.5, 2.0]; out = 1.5 * 1 + 2.0 * 10 + 0.25 = 21.75
    w1 = np.array([[1, 0, 2, 0], [0, 1, 0, 2]], np.float32)
    b1 = np.array([0, 0, -3, 0], np.float32)
    w2 = np.array([[1], [10]], np.float32)
    b2 = np.array([0.25], np.float32)
    layers = [(w1, b1), (w2, b2)]
    x = np.array([[1.0, 2.0]])
    for f in (mlp.forward_fp64, mlp.forward_fp32, mlp.forward_bf16):
        assert float(f(layers, x, pool=[2, 0])[0, 0]) == 21.75
    # strided (non-contiguous) grouping would give (1 + 0)/2 * 1 + (2 + 4)/2 * 10 + .25 = 30.75
    assert float(mlp.forward_fp64(layers, x, pool=[2, 0])[0, 0]) != 30.75
    # g = 4 averages all four: 7/4 -> w2 must then be 1 x 1
    layers4 = [(w1, b1), (np.array([[2]], np.float32), b2)]
    assert float(mlp.forward_fp64(layers4, x, pool=[4, 0])[0, 0]) == 3.75


def test_bf16_pool_averages_bf16_activations_without_rerounding():
    # activations 1 and 1 + 2^-7 (both bf16); their average 1 + 2^-8 is NOT a
    # bf16 value and must reach the next layer unrounded (weight 1, bias 0)
    layers = [(np.array([[1, 1]], np.float32), np.array([0, 2.0 ** -7], np.float32)),
              (np.array([[1]], np.float32), np.array([0], np.float32))]
    assert float(mlp.forward_bf16(layers, np.array([[1.0]]), pool=[2, 0])[0, 0]) == 1 + 2.0 ** -8


def test_pool_is_the_unpooled_network_with_folded_weights():
    # avg pooling is linear: layer l+1 after pooling g == an unpooled layer whose
    # row k is W[k // g] / g (the GPU engines run this form)
    rng = np.random.default_rng(0)
    dims = [(78, 128), (64, 128), (128, 128), (32, 128), (128, 128), (128, 256)]
    layers = [(rng.normal(size=d).astype(np.float32) / 8, rng.normal(size=d[1]).astype(np.float32) / 8) for d in dims]
    pool = [2, 0, 4, 0, 0, 0]
    folded = [layers[0]]
    for l in range(1, 6):
        g = pool[l - 1] or 1
        w, b = layers[l]
        folded.append((np.repeat(w, g, axis=0) / g, b))
    x = rng.integers(0, 256, size=(64, 78)) / 256.0
    a = mlp.forward_fp64(layers, x, pool)
    f = mlp.forward_fp64(folded, x)
    assert np.allclose(a, f, rtol=1e-12, atol=1e-12)


def test_model_file_round_trips_pool_and_metadata_and_rejects_bad_chains():
    rng = np.random.default_rng(1)
    layers = [(rng.normal(size=(81, 16)).astype(np.float32), np.zeros(16, np.float32)),
              (rng.normal(size=(8, 256)).astype(np.float32), np.zeros(256, np.float32))]
    blob = model_io.save(layers, pool=[2, 0], meta_range=[(0.0, 2.0), (1.0, 5.0), (-1.0, 1.0)])
    net = model_io.load_net(blob)
    assert net["pool"] == [2, 0] and [tuple(r) for r in net["meta_range"]] == [(0.0, 2.0), (1.0, 5.0), (-1.0, 1.0)]
    assert all(np.array_equal(a[0], b[0]) for a, b in zip(net["layers"], layers))
    with pytest.raises(model_io.CorruptModel):   # 16 / 4 = 4 != 8
        model_io.load_net(model_io.save(layers, pool=[4, 0]))


def test_metadata_features_hand_derived():
    # (28 - 0) / (56 - 0) = 0.5 ; (3.5 - 1) / (6 - 1) = 0.5 ; (-1 - -1) / 2 = 0
    m = window.meta_features([28.0, 3.5, -1.0], [(0.0, 56.0), (1.0, 6.0), (-1.0, 1.0)])
    assert m.tolist() == [0.5, 0.5, 0.0]
    img = np.arange(12, dtype=np.uint8).reshape(3, 4)
    x = window.net_inputs(img, np.array([2]), np.array([3]), m)
    assert x.shape == (1, 81) and x[0, 78:].tolist() == [0.5, 0.5, 0.0]
    assert x[0, 77] == img[2, 2] / 256.0                      # tap (0,-1) stays the last window feature
    with pytest.raises(ValueError):
        window.meta_features([1.0], [(0.0, 1.0), (0.0, 1.0)])


def _meta_model(zero_meta_weights, seed=3):
    base = synth.he_uniform_layers((78, 16, 256), seed=seed)
    w0, b0 = base[0]
    rng = np.random.default_rng(seed)
    wm = np.zeros((3, 16), np.float32) if zero_meta_weights else rng.normal(size=(3, 16)).astype(np.float32)
    layers = [(np.concatenate([w0, wm]), b0), base[1]]
    return base, model_io.save(layers, meta_range=[(0.0, 2.0), (0.0, 10.0), (0.0, 1.0)])


def test_zero_metadata_weights_reduce_to_the_metadata_free_model():
    base, blob = _meta_model(True)
    img = synth.random_image(13, 9, seed=2, kind="smooth")
    a = container.parse(codec.encode(img, blob, 1, 4, meta=[1.0, 3.0, 0.25]))
    b = container.parse(codec.encode(img, model_io.save(base), 1, 4))
    assert a["streams"] == b["streams"]


def test_metadata_is_stored_uncompressed_and_drives_the_tables():
    _, blob = _meta_model(False)
    img = synth.random_image(13, 9, seed=2, kind="smooth")
    m = [1.0, 3.0, 0.25]
    bits = codec.encode(img, blob, 1, 4, meta=m)
    hdr = container.parse(bits)
    assert hdr["meta"].tolist() == m
    # the block is 4 + 4 n bytes between the size table and the streams
    n_streams = len(hdr["streams"])
    assert hdr["header_bytes"] == container.HEADER_FIXED + 4 * n_streams + 4 + 4 * len(m)
    assert np.array_equal(codec.decode(bits, blob), img)          # re-read from the container
    other = container.parse(codec.encode(img, blob, 1, 4, meta=[0.0, 9.0, 1.0]))
    assert other["streams"] != hdr["streams"]                     # the metadata enters the network
    with pytest.raises(ValueError):
        codec.encode(img, blob, 1, 4, meta=[1.0])
