"""Write fixture weights with the ORACLE trainer only (no GPU code involved).

fixtures/p100k_trained.dlicmdl — P100K (78->128x5->256) briefly trained on
synthetic "natural-like" crops (SURVEY §8(d) C2 generator, sigma_tex=2,
sigma_n=1), as north_star allows ("briefly trained by the oracle on synthetic
smooth-plus-noise images").  Run: python scripts/make_fixtures.py
fixtures/p100k_pool_meta.dlicmdl — the §8(f) f4 network (78 + 3 metadata
inputs -> 128 -> [avg 2] -> 128 -> 128 -> [avg 2] -> 128 -> 128 -> 256),
seeded He-uniform weights (the GPU tests' model); written alone by
python scripts/make_fixtures.py pool_meta
"""

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
from oracle import mlp, model_io, train  # noqa: E402


def main():
    rng = np.random.default_rng(12345)
    crops = []
    for s in range(16):
        img = synth.natural_like(768, 512, seed=1000 + s)
        for _ in range(6):
            y = int(rng.integers(0, 512 - 128))
            x = int(rng.integers(0, 768 - 128))
            crops.append(np.ascontiguousarray(img[y:y + 128, x:x + 128]))
    x, y = train.dataset(crops)
    held = synth.natural_like(768, 512, seed=999)
    xv, yv = train.dataset([held[:128, :256]])
    layers = synth.he_uniform_layers(mlp.P100K, seed=7)
    t = time.time()
    layers, hist = train.train(layers, x, y, epochs=int(os.environ.get("EPOCHS", "16")), batch=4096,
                               lr=1e-3, seed=0)
    print("train %.1fs loss/epoch %s" % (time.time() - t, ["%.3f" % h for h in hist]))
    print("held-out vloss %.4f bits" % train.vloss_bits(layers, xv, yv))
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "fixtures",
                       "p100k_trained.dlicmdl")
    with open(out, "wb") as fh:
        fh.write(model_io.save(layers))
    print("wrote", out)


POOL = [2, 0, 2, 0, 0, 0]
META_RANGE = [(0.0, 2.0), (0.0, 10.0), (0.5, 6.0)]


def p100k_3d():
    """fixtures/p100k_3d.dlicmdl: the §8(f) f2 network (87 = 78 + the 3x3 box
    of the slice below -> 128x5 -> 256), seeded He-uniform weights."""
    layers = synth.he_uniform_layers((87, 128, 128, 128, 128, 128, 256), seed=11, bias_scale=0.1)
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "fixtures", "p100k_3d.dlicmdl")
    with open(out, "wb") as fh:
        fh.write(model_io.save(layers))
    print("wrote", out)


def p350k():
    """fixtures/p350k_seeded.dlicmdl: the §8(f) f1 network P350K (78 -> 256x5
    -> 256, reading R4), seeded He-uniform weights with biases (the GPU
    tests' and bench's model)."""
    layers = synth.he_uniform_layers(mlp.P350K, seed=3, bias_scale=0.1)
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "fixtures", "p350k_seeded.dlicmdl")
    with open(out, "wb") as fh:
        fh.write(model_io.save(layers))
    print("wrote", out)


def p12():
    """fixtures/p12_seeded.dlicmdl: the §8(f) f3 network P12 (78 -> 256x5 ->
    4096, 12-bit alphabet, reading R16), seeded He-uniform weights with biases
    (the GPU tests' and bench's model)."""
    layers = synth.he_uniform_layers(mlp.P12, seed=5, bias_scale=0.1)
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "fixtures", "p12_seeded.dlicmdl")
    with open(out, "wb") as fh:
        fh.write(model_io.save(layers))
    print("wrote", out)


def pool_meta():
    layers = synth.he_uniform_pooled(81, [128, 128, 128, 128, 128, 256], POOL, seed=7, bias_scale=0.1)
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "fixtures",
                       "p100k_pool_meta.dlicmdl")
    with open(out, "wb") as fh:
        fh.write(model_io.save(layers, pool=POOL, meta_range=META_RANGE))
    print("wrote", out)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "pool_meta":
        pool_meta()
    elif len(sys.argv) > 1 and sys.argv[1] == "3d":
        p100k_3d()
    elif len(sys.argv) > 1 and sys.argv[1] == "p350k":
        p350k()
    elif len(sys.argv) > 1 and sys.argv[1] == "p12":
        p12()
    else:
        main()
        pool_meta()
        p100k_3d()
        p350k()
        p12()
