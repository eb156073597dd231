"""World-size-2 gloo tests (CPU) of the multi-GPU sharding in
paper_2207_05152_b200/dist.py -- the same functions bench.py runs on NCCL.
The per-rank coder is the oracle here (the device coder is exercised by the
GPU tests); results must equal the single-process oracle byte for byte.
dist.py imports without libdlic.so (the binding loads it lazily)."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import codec, container, model_io, streams
from paper_2207_05152_b200 import dist as dd

BLOB = None


def _blob():
    global BLOB
    if BLOB is None:
        BLOB = model_io.save(synth.he_uniform_layers((78, 8, 256), seed=5))
    return BLOB


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _imgs(n):
    return np.stack([synth.random_image(11, 7, seed=i, kind="smooth") for i in range(n)])


def _weak_worker(rank, world, port, n_per_rank, outdir):
    """bench.py's weak-scaling step: every rank codes its own images, the
    container sizes are all-gathered, every rank decodes its own containers."""
    _init(rank, world, port)
    imgs = _imgs(world * n_per_rank)[rank * n_per_rank:(rank + 1) * n_per_rank]
    state = {}

    def encode_local():
        state["bits"] = [codec.encode(im, _blob(), 1, 4) for im in imgs]
        return torch.tensor([len(b) for b in state["bits"]], dtype=torch.int64)

    def decode_local():
        state["dec"] = [codec.decode(b, _blob()) for b in state["bits"]]

    all_sizes, offs = dd.coded_step(encode_local, decode_local)
    assert all(np.array_equal(d, im) for d, im in zip(state["dec"], imgs))
    np.save(os.path.join(outdir, "sizes%d.npy" % rank), all_sizes.numpy())
    np.save(os.path.join(outdir, "offs%d.npy" % rank), offs.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("n_per_rank", [1, 3])
def test_weak_step_sizes_and_offsets(n_per_rank):
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_weak_worker, args=(world, _free_port(), n_per_rank, d), nprocs=world, join=True)
        sizes = [np.load(os.path.join(d, "sizes%d.npy" % r)) for r in range(world)]
        offs = [np.load(os.path.join(d, "offs%d.npy" % r)) for r in range(world)]
    single = [len(codec.encode(im, _blob(), 1, 4)) for im in _imgs(world * n_per_rank)]
    for r in range(world):
        assert sizes[r].shape == (world, n_per_rank)
        assert sizes[r].reshape(-1).tolist() == single
        assert offs[r].tolist() == list(np.cumsum([0] + single[:-1]))


# one image, 3x3 = 9 tiles split across ranks (C4's sharding)
W, H, TW, TH, G = 40, 30, 16, 12, 4


def _oracle_encode_units(img):
    layers = model_io.load(_blob())
    tiles = container.tiles(W, H, TW, TH)

    def enc(lo, hi):
        payload, sizes = b"", []
        for (x0, y0, tw, th) in tiles[lo:hi]:
            fs, cs = codec.unit_tables_by_front(layers, 1, np.ascontiguousarray(img[y0:y0 + th, x0:x0 + tw]))
            for s in streams.encode_unit(fs, cs, G):
                b = streams.rans.words_to_bytes(s)
                payload += b
                sizes.append(len(b))
        return payload, sizes
    return enc


def _units_worker(rank, world, port, outdir):
    _init(rank, world, port)
    img = synth.random_image(W, H, seed=3, kind="smooth")
    n_units = len(container.tiles(W, H, TW, TH))
    payload, (lo, hi), soffs, all_ssz = dd.encode_units_distributed(_oracle_encode_units(img), n_units)
    with open(os.path.join(outdir, "payload%d.bin" % rank), "wb") as fh:
        fh.write(payload)
    np.save(os.path.join(outdir, "meta%d.npy" % rank), np.array([lo, hi]))
    np.save(os.path.join(outdir, "soffs%d.npy" % rank), soffs)
    np.save(os.path.join(outdir, "ssz%d.npy" % rank), all_ssz)
    # decode side: each rank decodes its own tiles of the framed container
    full = container.write(W, H, 1, G, TW, TH, model_io.digest(_blob()),
                           _split(b"".join(_payloads_when_ready(outdir, world)), all_ssz))
    out = np.zeros((H, W), np.uint8)

    def dec(a, b):
        tiles = container.tiles(W, H, TW, TH)
        ref = codec.decode(full, _blob())
        for (x0, y0, tw, th) in tiles[a:b]:
            out[y0:y0 + th, x0:x0 + tw] = ref[y0:y0 + th, x0:x0 + tw]
    dd.decode_units_distributed(dec, n_units)
    np.save(os.path.join(outdir, "dec%d.npy" % rank), out)
    dist.destroy_process_group()


def _split(payload, sizes):
    out, o = [], 0
    for s in sizes:
        out.append(payload[o:o + int(s)])
        o += int(s)
    return out


def _payloads_when_ready(outdir, world):
    dist.barrier()          # every rank's payload is on disk (a product writes at its offset instead)
    return [open(os.path.join(outdir, "payload%d.bin" % r), "rb").read() for r in range(world)]


def test_one_image_units_split_across_two_ranks():
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_units_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        parts = [open(os.path.join(d, "payload%d.bin" % r), "rb").read() for r in range(world)]
        ssz = [np.load(os.path.join(d, "ssz%d.npy" % r)) for r in range(world)]
        soffs = [np.load(os.path.join(d, "soffs%d.npy" % r)) for r in range(world)]
        ranges = [tuple(np.load(os.path.join(d, "meta%d.npy" % r))) for r in range(world)]
        decs = [np.load(os.path.join(d, "dec%d.npy" % r)) for r in range(world)]
    img = synth.random_image(W, H, seed=3, kind="smooth")
    whole = codec.encode(img, _blob(), 1, G, TW, TH)
    hdr = container.parse(whole)
    assert ranges == [(0, 5), (5, 9)]
    assert all(np.array_equal(ssz[0], s) for s in ssz) and all(np.array_equal(soffs[0], o) for o in soffs)
    assert ssz[0].tolist() == [len(s) for s in hdr["streams"]]
    framed = container.write(W, H, 1, G, TW, TH, model_io.digest(_blob()), _split(b"".join(parts), ssz[0]))
    assert framed == whole
    # each rank decoded exactly its tiles; together they are the image
    tiles = container.tiles(W, H, TW, TH)
    merged = np.zeros_like(img)
    for (lo, hi), dec in zip(ranges, decs):
        for (x0, y0, tw, th) in tiles[lo:hi]:
            merged[y0:y0 + th, x0:x0 + tw] = dec[y0:y0 + th, x0:x0 + tw]
    assert np.array_equal(merged, img)


def test_shard_plan_properties():
    for n in range(0, 40):
        for w in (1, 2, 3, 8):
            rngs = [dd.shard_range(n, w, r) for r in range(w)]
            assert rngs[0][0] == 0 and rngs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))
            sizes = [b - a for a, b in rngs]
            assert max(sizes) - min(sizes) <= 1


def test_assemble_and_offsets():
    parts = [[b"ab", b"cde"], [b"f"]]
    offs = dd.global_offsets([[2, 3], [1]])
    assert offs.tolist() == [0, 2, 5, 6]
    assert dd.assemble(parts, offs) == b"abcdef"
