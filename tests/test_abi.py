"""C-ABI checks that need no GPU: the library builds and loads, exports every
symbol include/dlic.h declares, and its host-only parsers agree with the
independent oracle (SHA-256 of model files, container framing)."""

import hashlib
import os
import re

import numpy as np
import pytest

import synth
from conftest import ROOT
from oracle import codec, container, mlp, model_io


@pytest.fixture(scope="module")
def dl():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2207_05152_b200 as m
    return m


def test_exports_every_declared_symbol(dl):
    hdr = open(os.path.join(ROOT, "include", "dlic.h")).read()
    names = set(re.findall(r"\b(dlic_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 20
    for n in sorted(names):
        assert hasattr(dl._L(), n), n


def test_model_blob_hash_agrees_with_hashlib(dl, trained_blob):
    for blob in (trained_blob, model_io.save(synth.he_uniform_layers((78, 9, 256), seed=2))):
        assert dl.dlic_model_blob_check(blob) == hashlib.sha256(blob[:-32]).digest() == model_io.digest(blob)
    bad = bytearray(trained_blob)
    bad[77] ^= 1
    with pytest.raises(dl.DlicError) as e:
        dl.dlic_model_blob_check(bytes(bad))
    assert e.value.status == 4


def test_peek_agrees_with_oracle_container(dl):
    blob = model_io.save(synth.he_uniform_layers((78, 8, 256), seed=1))
    for (h, w, g, tile) in ((9, 14, 4, (0, 0)), (23, 30, 8, (10, 7)), (1, 1, 32, (0, 0))):
        img = synth.random_image(w, h, seed=h, kind="smooth")
        b = codec.encode(img, blob, 1, g, *tile)
        ref = container.parse(b)
        got = dl.dlic_peek(b)
        assert (got["width"], got["height"], got["group_rows"], got["precision"]) == (w, h, g, 1)
        assert (got["tile_w"], got["tile_h"]) == tile
        assert got["n_streams"] == len(ref["streams"])
        assert got["payload_bytes"] == sum(len(s) for s in ref["streams"])
        assert got["header_bytes"] == ref["header_bytes"]
        assert got["model_sha256"] == model_io.digest(blob)
        assert got["n_units"] == len(container.tiles(w, h, *tile))
        assert dl.dlic_max_container_bytes(w, h, 1, g, tile) >= len(b)
        with pytest.raises(dl.DlicError):
            dl.dlic_peek(b[:-1])


def test_invalid_options_rejected(dl):
    assert dl.dlic_max_container_bytes(100, 100, 1, 3) == 0          # G must divide 32
    assert dl.dlic_max_container_bytes(4000, 10, 1, 32) == 0         # untiled width > 3072
    assert dl.dlic_max_container_bytes(4000, 10, 1, 32, (768, 720)) > 0
    assert dl._L().dlic_status_str(7) == b"model hash mismatch"


def test_no_cpu_fallback_without_gpu(dl, trained_blob):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(dl.DlicError) as e:
        dl.dlic_model_load(trained_blob, 0)
    assert e.value.status == 12


def test_info_reports(dl):
    s = dl.dlic_info()
    assert "sm_100a" in s and "bf16_tcgen05" in s


def test_container_build_and_unit_streams_agree_with_oracle_framing(dl):
    """Host-only framing calls (no GPU): dlic_container_build frames the same
    bytes as the oracle's container writer given the same streams, and
    dlic_unit_streams partitions the streams by unit (tile-major, Q16)."""
    rng = np.random.default_rng(3)
    for (w, h, g, tile) in ((40, 30, 8, (16, 12)), (13, 5, 32, (0, 0)), (100, 70, 4, (30, 33))):
        units = container.tiles(w, h, *tile)
        streams = []
        per_unit = []
        for (_, _, tw, th) in units:
            k = -(-th // g)
            per_unit.append(k)
            streams += [rng.integers(0, 256, 2 * int(rng.integers(2, 40)), dtype=np.uint8).tobytes() for _ in range(k)]
        sha = bytes(rng.integers(0, 256, 32, dtype=np.uint8))
        num = dl.dlic_numerics_rev()
        ref = container.write(w, h, 1, g, tile[0], tile[1], sha, streams, num)
        got = dl.dlic_container_build(w, h, sha, [len(s) for s in streams], b"".join(streams), 1, g, tile)
        assert got == ref
        assert dl.dlic_peek(got)["numerics"] == num and container.parse(got)["numerics"] == num
        first = 0
        for u, k in enumerate(per_unit):
            assert dl.dlic_unit_streams(w, h, u, u + 1, 1, g, tile) == (first, k)
            first += k
        assert dl.dlic_unit_streams(w, h, 0, len(units), 1, g, tile) == (0, len(streams))
        with pytest.raises(dl.DlicError):
            dl.dlic_unit_streams(w, h, 0, len(units) + 1, 1, g, tile)
        with pytest.raises(dl.DlicError):   # sizes must sum to the payload
            dl.dlic_container_build(w, h, sha, [len(s) for s in streams], b"".join(streams)[:-2], 1, g, tile)


def test_peek_rejects_other_container_versions(dl):
    blob = model_io.save(synth.he_uniform_layers((78, 8, 256), seed=1))
    b = bytearray(codec.encode(synth.random_image(9, 7, seed=1, kind="smooth"), blob, 1, 4))
    assert dl.dlic_peek(bytes(b))["numerics"] == 0            # the oracle's own arithmetic
    b[4] = 1                                                   # round-1 layout
    with pytest.raises(dl.DlicError) as e:
        dl.dlic_peek(bytes(b))
    assert e.value.status == 5
