"""World-size-2 gloo tests (CPU) of the multi-GPU sharding logic: shard plan,
the single size all_gather, global offsets and batch assembly.  The per-rank
encoder is the oracle here (the device encoder is exercised by the GPU tests);
the result must equal the single-process batch byte for byte."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import codec, model_io


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_img, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2207_05152_b200 import dist as dd
    blob = model_io.save(synth.he_uniform_layers((78, 8, 256), seed=5))
    imgs = np.stack([synth.random_image(11, 7, seed=i, kind="smooth") for i in range(n_img)])

    def enc(shard):
        return [codec.encode(im, blob, 1, 4) for im in shard]

    mine, first, offs = dd.encode_batch_distributed(enc, imgs)
    # every rank writes its containers into its own byte range (no payload exchange)
    with open(os.path.join(outdir, "part%d.bin" % rank), "wb") as fh:
        np.save(fh, np.array([first, len(mine)]))
        for b in mine:
            np.save(fh, np.frombuffer(b, np.uint8))
    np.save(os.path.join(outdir, "offs%d.npy" % rank), offs)
    dist.destroy_process_group()


@pytest.mark.parametrize("n_img", [3, 4, 1])
def test_two_rank_batch_equals_single_process(n_img):
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), n_img, d), nprocs=world, join=True)
        offs = [np.load(os.path.join(d, "offs%d.npy" % r)) for r in range(world)]
        assert all(np.array_equal(offs[0], o) for o in offs)       # every rank agrees
        parts = []
        for r in range(world):
            with open(os.path.join(d, "part%d.bin" % r), "rb") as fh:
                first, cnt = np.load(fh)
                parts.append([np.load(fh).tobytes() for _ in range(cnt)])
        from paper_2207_05152_b200 import dist as dd
        batch = dd.assemble(parts, offs[0])
    blob = model_io.save(synth.he_uniform_layers((78, 8, 256), seed=5))
    single = [codec.encode(synth.random_image(11, 7, seed=i, kind="smooth"), blob, 1, 4) for i in range(n_img)]
    assert batch == b"".join(single)
    assert list(np.diff(offs[0])) == [len(b) for b in single]


def test_shard_plan_properties():
    from paper_2207_05152_b200 import dist as dd
    for n in range(0, 40):
        for w in (1, 2, 3, 8):
            rngs = [dd.shard_range(n, w, r) for r in range(w)]
            assert rngs[0][0] == 0 and rngs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))
            sizes = [b - a for a, b in rngs]
            assert max(sizes) - min(sizes) <= 1
