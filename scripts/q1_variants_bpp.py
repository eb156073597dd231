"""Cost of the quantiser reading R5 (Q1', residual on symbol 255) against the
survey's Q1 (residual on the first argmax, scale 2^16 - 256) and against the
ideal code length of the unquantised PDF, on the C2 image with the trained
P100K fixture.  Oracle-only (fp64 network, fp64 softmax rounded to fp32);
prints information content in bits per pixel (the rANS payload is this plus
the per-lane flush, R6).

python scripts/q1_variants_bpp.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import synth
from oracle import mlp, model_io, quant, window


def q1_argmax(p, k=16):
    """Survey Q1: f = 1 + floor(fl32(p) * fl32(2^k - 256)),
    residual R = 2^k - sum f added to the first argmax of f."""
    p = np.asarray(p, np.float32)
    f = 1 + np.floor(p * np.float32((1 << k) - p.shape[-1])).astype(np.int64)
    r = (1 << k) - f.sum(-1)
    a = f.argmax(-1)
    f[np.arange(f.shape[0]), a] += r
    assert np.all(f.sum(-1) == 1 << k) and np.all(f >= 1)
    return f


def main():
    blob = open(os.path.join(os.path.dirname(__file__), "..", "fixtures", "p100k_trained.dlicmdl"), "rb").read()
    layers = model_io.load(blob)
    img = synth.config_images("C2", count=1)[0]
    h, w = img.shape
    sym = img.reshape(-1).astype(np.int64)
    bits = {"ideal": 0.0, "q1prime": 0.0, "q1_argmax": 0.0}
    chunk = 32768
    for s in range(0, h * w, chunk):
        idx = np.arange(s, min(s + chunk, h * w))
        rows, cols = np.divmod(idx, w)
        lg = mlp.forward_fp64(layers, window.features(window.gather_many(img, rows, cols))).astype(np.float32)
        p = quant.softmax_fp64(lg).astype(np.float32)
        ys = sym[idx]
        pd = p.astype(np.float64)
        bits["ideal"] += -np.log2(pd[np.arange(len(idx)), ys] / pd.sum(-1)).sum()
        for name, f in (("q1prime", quant.q1(p)), ("q1_argmax", q1_argmax(p))):
            bits[name] += -np.log2(f[np.arange(len(idx)), ys] / 65536.0).sum()
    npx = h * w
    for k, v in bits.items():
        print("%-10s %.5f bpp" % (k, v / npx))
    print("Q1' - Q1(argmax) = %+.5f bpp (%+.3f%%)" % ((bits["q1prime"] - bits["q1_argmax"]) / npx,
                                                     100 * (bits["q1prime"] / bits["q1_argmax"] - 1)))


if __name__ == "__main__":
    main()
