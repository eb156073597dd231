"""Debug: localise a round-trip failure (encoder bytes vs oracle; decoder status)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2207_05152_b200 as dl
import synth
from oracle import codec, model_io
blob = open("fixtures/p100k_trained.dlicmdl", "rb").read()
m = dl.dlic_model_load(blob, 0)
for (h, w, g) in [(1, 1, 32), (1, 2, 32), (1, 13, 32), (2, 1, 32), (5, 8, 1)]:
    for prec in (0, 1):
        img = synth.natural_like(w, h, seed=h + 7 * w)
        bits = dl.dlic_encode(m, img, precision=prec, group_rows=g)
        fc = dl.dlic_debug_mlp(m, img, precision=prec, group_rows=g, logits=False, probs=False, freqs=False)["fc"]
        ob = codec.encode_with_tables((fc & 0xFFFF).astype(np.int64), (fc >> 16).astype(np.int64), w, h, prec, g,
                                      0, 0, model_io.digest(blob), dl.dlic_numerics_rev())
        try:
            d = dl.dlic_decode(m, bits)
            res = "ok" if np.array_equal(d, img) else "MISMATCH %s vs %s" % (d.ravel()[:8], img.ravel()[:8])
        except Exception as e:
            res = "ERR " + str(e)[:60]
        print(h, w, g, prec, "enc==oracle" if ob == bits else "ENC DIFF", res, img.ravel()[:6])
