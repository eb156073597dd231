"""Pins for §8(f) f2 in the oracle: the 2-layer 3D window (Fig. 6
right; reading R13) and the overlapped 3D wavefront (reading R14),
the volume codec and container (window id 2)."""

import itertools

import numpy as np
import pytest

import synth
from oracle import codec, container, model_io, schedule, window


def test_3d_window_geometry():
    assert len(window.OFFSETS_3D) == 9 and window.N_INPUTS_3D == 87
    assert set(window.OFFSETS_3D) == set(itertools.product((-1, 0, 1), (-1, 0, 1)))
    # the pixel directly below the target is tap 4 (row-major box)
    assert window.OFFSETS_3D[4] == (0, 0)


def test_slice_lag_is_minimal_by_brute_force():
    """Every lower-layer tap (z-1, r+dr, c+dc) must be decoded strictly before
    (z, r, c) under step_3d; LAG3D = 5 works, 4 does not (it misses the tap
    (r+1, c+1), decoded 4 steps after (r, c) in its own slice)."""
    h, w = 7, 9

    def ok(lag3d):
        for r in range(h):
            for c in range(w):
                s = schedule.step_3d(1, r, c, lag3d)
                for dr, dc in window.OFFSETS_3D:
                    rr, cc = r + dr, c + dc
                    if 0 <= rr < h and 0 <= cc < w and schedule.step_3d(0, rr, cc, lag3d) >= s:
                        return False
        return True
    assert schedule.LAG3D == 5 and ok(5) and not ok(4)
    assert schedule.n_fronts_3d(256, 256, 35) == 256 + 3 * 255 + 5 * 34


def test_gather_3d_hand_values():
    prev = np.arange(20, dtype=np.uint8).reshape(4, 5)
    x = window.gather_many_3d(prev, np.array([0, 3]), np.array([0, 4]), (4, 5))
    # (0,0): box rows -1..1, cols -1..1 -> fill above/left
    assert x[0].tolist() == [0, 0, 0, 0, 0, 1, 0, 5, 6]
    # (3,4): bottom-right corner
    assert x[1].tolist() == [13, 14, 0, 18, 19, 0, 0, 0, 0]
    assert window.gather_many_3d(None, np.array([1]), np.array([1]), (4, 5)).tolist() == [[0] * 9]


def _models(seed=4):
    """(3D model with zero lower-layer weights, the same network as a 2D model)."""
    base = synth.he_uniform_layers((78, 16, 256), seed=seed, bias_scale=0.05)
    w0, b0 = base[0]
    z3 = [(np.concatenate([w0, np.zeros((9, 16), np.float32)]), b0), base[1]]
    return model_io.save(z3), model_io.save(base)


@pytest.mark.parametrize("tile", [(0, 0), (7, 5)])
def test_zero_lower_weights_reduce_each_slice_to_the_2d_codec(tile):
    b3, b2 = _models()
    vol = np.stack([synth.random_image(11, 9, seed=z, kind="smooth") for z in range(3)])
    hv = container.parse(codec.encode_volume(vol, b3, 1, 4, *tile))
    assert hv["window"] == container.WINDOW_3D and hv["depth"] == 3
    sps = container.streams_per_slice(11, 9, tile[0], tile[1], 4)
    for z in range(3):
        h2 = container.parse(codec.encode(vol[z], b2, 1, 4, *tile))
        assert hv["streams"][z * sps:(z + 1) * sps] == h2["streams"]


@pytest.mark.parametrize("d,h,w,g,tile", [(1, 5, 7, 4, (0, 0)), (3, 9, 11, 2, (0, 0)), (2, 12, 10, 32, (6, 5))])
def test_volume_round_trip_and_lower_layer_matters(d, h, w, g, tile):
    layers = synth.he_uniform_layers((87, 16, 256), seed=d + h, bias_scale=0.05)
    blob = model_io.save(layers)
    rng = np.random.default_rng(h)
    base = synth.random_image(w, h, seed=1, kind="smooth").astype(np.int64)
    vol = np.stack([np.clip(base + rng.integers(-2, 3, size=base.shape), 0, 255) for _ in range(d)]).astype(np.uint8)
    bits = codec.encode_volume(vol, blob, 1, g, *tile)
    assert np.array_equal(codec.decode_volume(bits, blob), vol)
    if d > 1:   # a different slice below changes slice 1's tables (the 3D taps are inputs)
        vol2 = vol.copy()
        vol2[0] = 255 - vol2[0]
        sps = container.streams_per_slice(w, h, tile[0], tile[1], g)
        a = container.parse(bits)["streams"][sps:2 * sps]
        b = container.parse(codec.encode_volume(vol2, blob, 1, g, *tile))["streams"][sps:2 * sps]
        assert a != b


def test_volume_container_framing():
    layers = synth.he_uniform_layers((87, 8, 256), seed=1)
    blob = model_io.save(layers)
    vol = np.zeros((4, 6, 5), np.uint8)
    bits = codec.encode_volume(vol, blob, 1, 2)
    hdr = container.parse(bits)
    assert hdr["depth"] == 4 and len(hdr["streams"]) == 4 * 3
    bad = bytearray(bits)
    bad[6] = 1                         # as a 2D container the stream count is wrong
    with pytest.raises(container.CorruptContainer):
        container.parse(bytes(bad))


def test_table_iii_first_frame_vs_complete_context():
    """P:259-279 Table III: 256x256x35, first frame 0.2799 s vs complete
    0.3374 s (ratio 1.205) for the ~350K net.  Our R14 schedule: the first
    slice completes after 1021 fronts, the volume after 1021 + 34*5 = 1191
    (ratio 1.167); the paper's window/lag are not stated (context, not a pin)."""
    first = schedule.n_fronts(256, 256)
    full = schedule.n_fronts_3d(256, 256, 35)
    assert first == 1021 and full == 1191
    assert abs(0.3374 / 0.2799 - 1.2054) < 1e-3
