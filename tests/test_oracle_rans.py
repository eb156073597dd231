"""Pins for oracle.rans and oracle.streams (SPEC worked examples, exhaustive
tiny-alphabet round trips, the entropy bound and the size bound)."""

import itertools
import math

import numpy as np
import pytest

from conftest import golden
from oracle import quant, rans, streams


def _tab(freqs):
    return list(freqs), list(quant.cdf(np.array(freqs)))


def test_spec_symbol_table_examples():
    for ex in golden("spec_rans.json")["build_symbol_table"]:
        f = np.array(ex["freqs"])
        if "error" in ex:
            assert f.sum() != 1 << ex["k"]
        else:
            assert list(quant.cdf(f)) == ex["cums"] and f.sum() == 1 << ex["k"]


def test_spec_update_formula_examples():
    g = golden("spec_rans.json")
    for ex in g["encode_symbol"]:
        freqs, cums = _tab(ex["freqs"])
        s = ex["sym"]
        assert rans.encode_symbol_raw(ex["x"], freqs[s], cums[s], ex["k"]) == ex["out"]
    for ex in g["decode_symbol"]:
        freqs, cums = _tab(ex["freqs"])
        assert rans.decode_symbol_raw(ex["x"], freqs, cums, ex["k"]) == (ex["sym"], ex["out"])


def test_spec_sequence_examples():
    g = golden("spec_rans.json")["encode_sequence"]
    t = _tab(g[0]["freqs"])
    assert len(rans.words_to_bytes(rans.encode_sequence([], [], g[0]["k"]))) == g[0]["bytes"]
    words = rans.encode_sequence(g[1]["symbols"], [t, t], g[1]["k"])
    out, xf, pos = rans.decode_sequence(words, [t, t], g[1]["k"])
    assert out == g[1]["symbols"] and xf == rans.L and pos == len(words)


def _compositions(total, parts):
    for cut in itertools.combinations(range(1, total), parts - 1):
        b = (0,) + cut + (total,)
        yield [b[i + 1] - b[i] for i in range(parts)]


def test_exhaustive_tiny_alphabets():
    k = 4
    tables = [t for n in (1, 2, 3) for t in _compositions(16, n)]
    rng = np.random.default_rng(0)
    tables += [list(t) for t in rng.permutation(list(_compositions(16, 4)))[:20]]
    n_checked = 0
    for freqs in tables:
        tab = _tab(freqs)
        n = len(freqs)
        for length in range(0, 6 if n <= 3 else 5):
            for seq in itertools.product(range(n), repeat=length):
                words = rans.encode_sequence(list(seq), [tab] * length, k)
                out, xf, pos = rans.decode_sequence(words, [tab] * length, k)
                assert out == list(seq) and xf == rans.L and pos == len(words)
                n_checked += 1
    assert n_checked > 30000


def test_varying_tables_k16_roundtrip():
    rng = np.random.default_rng(1)
    for _ in range(30):
        n = int(rng.integers(1, 300))
        tabs, syms = [], []
        for _ in range(n):
            a = int(rng.integers(2, 257))
            p = rng.dirichlet(np.full(a, float(rng.choice([0.05, 0.5, 5.0]))))
            f = quant.q1(p.astype(np.float32))
            tabs.append((list(f), list(quant.cdf(f))))
            syms.append(int(rng.choice(a, p=f / f.sum())))
        words = rans.encode_sequence(syms, tabs)
        out, xf, pos = rans.decode_sequence(words, tabs)
        assert out == syms and xf == rans.L and pos == len(words)


def test_entropy_bound_iid():
    ex = golden("spec_rans.json")["encode_sequence"][2]
    rng = np.random.default_rng(2)
    n = 100000
    tab = _tab(ex["iid_freqs"])
    syms = list(rng.choice(3, size=n, p=np.array(ex["iid_freqs"]) / 65536))
    words = rans.encode_sequence(syms, [tab] * n, ex["k"])
    bits = 16 * len(words) / n
    assert bits <= ex["entropy_bits"] + 0.01 + 32 / n
    assert bits >= ex["entropy_bits"] - 0.01


def test_compressed_size_equals_information_within_a_few_bytes():
    """north_star: compressed size equal to the summed -log2 p within a few bytes.
    Derivation: bytes = 4 + 2*words and 16*words = 16 + info - log2(x_final)
    up to the floor() slack, with log2(x_final) in [16, 32) -> bytes - info/8 in (2, 4]."""
    rng = np.random.default_rng(3)
    for scale in (0.6, 1.5, 4.0, 10.0):
        for _ in range(3):
            n = 768
            i = np.arange(256)
            tabs, syms, info = [], [], 0.0
            for _ in range(n):
                mu = rng.uniform(20, 230)
                logits = -np.abs(i - mu) / scale
                f = quant.q1(quant.softmax_fp64(logits).astype(np.float32))
                s = int(rng.choice(256, p=f / 65536))
                tabs.append((list(f), list(quant.cdf(f))))
                syms.append(s)
                info += -math.log2(f[s] / 65536)
            b = 2 * len(rans.encode_sequence(syms, tabs))
            assert 2.0 - 0.05 <= b - info / 8 <= 4.0 + 0.05, (scale, b - info / 8)


def test_truncated_stream_underflows():
    tab = _tab([1000] + [64536 // 255] * 254 + [64536 - (64536 // 255) * 254])
    assert sum(tab[0]) == 65536
    syms = [1 + (i % 200) for i in range(200)]
    words = rans.encode_sequence(syms, [tab] * 200)
    with pytest.raises(rans.Underflow):
        rans.decode_sequence(words[:len(words) // 2], [tab] * 200)


def test_group_streams_roundtrip_and_invariants():
    rng = np.random.default_rng(4)
    for _ in range(25):
        h, w = (int(v) for v in rng.integers(1, 40, 2))
        g = int(rng.choice([1, 3, 32, h]))
        a = int(rng.choice([2, 3, 16, 256]))
        ft = np.zeros((h, w, a), np.int64)
        img = np.zeros((h, w), np.uint8)
        for r in range(h):
            for c in range(w):
                p = rng.dirichlet(np.full(a, 0.3)).astype(np.float32)
                ft[r, c] = quant.q1(p)
                img[r, c] = rng.choice(a, p=ft[r, c] / 65536)
        ct = np.cumsum(ft, -1) - ft
        idx = img.astype(np.int64)[..., None]
        fs = np.take_along_axis(ft, idx, -1)[..., 0]
        cs = np.take_along_axis(ct, idx, -1)[..., 0]
        sts = streams.encode_unit(fs, cs, g)
        assert len(sts) == streams.n_groups(h, g)
        out = streams.decode_unit_with_tables(sts, ft, g)   # also checks end states / cursors
        assert np.array_equal(out, img)
