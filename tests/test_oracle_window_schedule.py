"""Pins for oracle.window and oracle.schedule against the paper and SPEC examples."""

import itertools

import numpy as np

from conftest import golden
from oracle import schedule, window


def test_window_geometry_matches_fig6():
    facts = golden("paper_facts.json")["window"]
    assert len(window.OFFSETS) == 9 * 9 - 3 == 78
    assert (window.TARGET_ROW, window.TARGET_COL) == (facts["target_row"], facts["target_col"])
    # every cell of the 9x9 box that precedes the target in raster order, and nothing else
    box = {(br - 8, bc - 6) for br in range(9) for bc in range(9)}
    kept = set(window.OFFSETS)
    assert kept <= box
    assert box - kept == {(0, 0), (0, 1), (0, 2)}
    for dr, dc in window.OFFSETS:                      # causal
        assert dr < 0 or (dr == 0 and dc < 0)
    assert list(window.OFFSETS) == sorted(window.OFFSETS)   # row-major order
    assert window.OFFSETS[0] == (-8, -6) and window.OFFSETS[-1] == (0, -1)


def test_gather_spec_examples_and_fill():
    for ex in golden("spec_wavefront.json")["extract_batch"]:
        img = np.array(ex["image"], dtype=np.uint8)
        j = window.OFFSETS.index(tuple(ex["offset"]))
        assert window.gather(img, *ex["pos"])[j] == ex["value"]
    img = np.full((3, 3), 7, np.uint8)
    g = window.gather(img, 0, 0)
    assert g.sum() == 0                                # everything causal is outside -> fill 0
    g = window.gather(img, 2, 2)
    # inside: rows 0..1 cols 0..2 (dc in [-2, 0]) + row 2 cols 0..1
    assert g.sum() == 7 * (2 * 3 + 2)


def test_gather_many_equals_gather():
    rng = np.random.default_rng(0)
    img = rng.integers(0, 256, (13, 11), dtype=np.uint8)
    rr, cc = np.divmod(np.arange(13 * 11), 11)
    many = window.gather_many(img, rr, cc)
    for i in range(len(rr)):
        assert np.array_equal(many[i], window.gather(img, rr[i], cc[i]))


def test_features_exact_in_bf16_and_fp32():
    from oracle import mlp
    v = np.arange(256)
    x = window.features(v)
    assert np.array_equal(mlp.bf16_round(x), x)
    assert np.array_equal(x.astype(np.float32).astype(np.float64), x)


def test_minimal_row_lag_brute_force():
    # strict precedence: every offset must land on a strictly smaller step
    def ok(lag):
        return all(dc + lag * dr < 0 for dr, dc in window.OFFSETS)
    assert not ok(1) and not ok(2) and ok(3) and ok(4)
    assert [o for o in window.OFFSETS if o[1] + 2 * o[0] >= 0] == [(-1, 2)]
    assert schedule.LAG == 3 == schedule.row_lag()


def test_spec_lag_and_schedule_examples():
    g = golden("spec_wavefront.json")
    for ex in g["compute_lags"]:
        assert schedule.row_lag([tuple(o) for o in ex["offsets"]]) == ex["row_lag"]
    for ex in g["build_schedule"]:
        assert schedule.n_fronts(ex["width"], ex["height"], ex["row_lag"]) == ex["steps"]
        if "step2" in ex:
            assert schedule.front(2, ex["width"], ex["height"], ex["row_lag"]) == [tuple(p) for p in ex["step2"]]


def test_front_count_and_rows():
    assert schedule.n_fronts(768, 512) == 2301          # C2
    assert schedule.n_fronts(32, 32) == 125
    assert schedule.n_fronts(256, 256) == 1021
    mx = max(len(schedule.front(t, 768, 512)) for t in range(0, 2301, 7))
    assert mx == 256


def test_partition_causality_and_closed_form():
    rng = np.random.default_rng(1)
    for _ in range(40):
        h, w = (int(v) for v in rng.integers(1, 17, 2))
        seen = {}
        for t in range(schedule.n_fronts(w, h)):
            lo, hi = schedule.front_rows(t, w, h)
            pix = schedule.front(t, w, h)
            assert [p[0] for p in pix] == list(range(lo, hi + 1))
            for p in pix:
                assert p not in seen
                seen[p] = t
        assert len(seen) == h * w
        for (r, c), t in seen.items():
            for dr, dc in window.OFFSETS:
                q = (r + dr, c + dc)
                if q in seen:
                    assert seen[q] < t


def test_wavefront_order_is_raster_order_within_each_row():
    # sequential equivalence: within one lane (row) the front order
    # visits columns ascending, exactly like raster order.
    for h, w in itertools.product([1, 3, 9], [1, 2, 10]):
        order = [p for t in range(schedule.n_fronts(w, h)) for p in schedule.front(t, w, h)]
        for r in range(h):
            assert [c for rr, c in order if rr == r] == list(range(w))
