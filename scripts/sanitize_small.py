"""Small encode/decode round trips for compute-sanitizer runs (racecheck/memcheck):
every engine -- P100K bf16 and fp32 (bf16x3), P350K, the 12-bit P12, the 3D
window on a 4-slice volume, pooling + metadata.
python scripts/sanitize_small.py [engine ...]   (default: all)"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2207_05152_b200 as dl
import synth


def load(name):
    return dl.dlic_model_load(open(os.path.join(ROOT, "fixtures", name), "rb").read(), 0)


def p100k():
    m = load("p100k_trained.dlicmdl")
    for (w, h, tile) in ((40, 30, (0, 0)), (700, 12, (0, 0)), (50, 40, (24, 20))):
        img = synth.natural_like(w, h, seed=w + h)
        for prec in (1, 0):
            b = dl.dlic_encode(m, img, precision=prec, tile=tile)
            assert np.array_equal(dl.dlic_decode(m, b), img), (w, h, prec)


def p350k():
    m = load("p350k_seeded.dlicmdl")
    for (w, h) in ((40, 30), (700, 12)):
        img = synth.natural_like(w, h, seed=w * h)
        b = dl.dlic_encode(m, img)
        assert np.array_equal(dl.dlic_decode(m, b), img), (w, h)


def p12():
    m = load("p12_seeded.dlicmdl")
    img = synth.mri_like_volume(48, 1, seed=3, bits=12)[0][:20, :37].copy()
    b = dl.dlic_encode(m, img)
    assert np.array_equal(dl.dlic_decode(m, b), img)


def vol():
    m = load("p100k_3d.dlicmdl")
    imgs = synth.mri_like_volume(40, 4, seed=5)
    for prec in (1, 0):
        blob, sizes = dl.dlic_encode_batch(m, imgs, precision=prec, volume_depth=4)
        assert np.array_equal(dl.dlic_decode_batch(m, blob, sizes), imgs), prec


def pool_meta():
    m = load("p100k_pool_meta.dlicmdl")
    img = synth.natural_like(45, 33, seed=9)
    for prec in (1, 0):
        b = dl.dlic_encode(m, img, precision=prec, meta=[0.9, 3.0, 1.25])
        assert np.array_equal(dl.dlic_decode(m, b), img), prec


ALL = {"p100k": p100k, "p350k": p350k, "p12": p12, "vol": vol, "pool_meta": pool_meta}
for name in sys.argv[1:] or list(ALL):
    ALL[name]()
    print(name, "ok", flush=True)
