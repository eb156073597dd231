import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2207_05152_b200 as dl
import synth
blob = open("fixtures/p100k_trained.dlicmdl", "rb").read()
m = dl.dlic_model_load(blob, 0)
prec = int(sys.argv[1]); w = int(sys.argv[2])
img = synth.natural_like(w, 1, seed=1 + 7 * w)
out = dl.dlic_debug_mlp(m, img, precision=prec, probs=False, freqs=False, fc=False)
print("ENC logits px0:", " ".join("%.6g" % v for v in out["logits"].reshape(-1, 256)[0]), file=sys.stderr)
bits = dl.dlic_encode(m, img, precision=prec)
try:
    dl.dlic_decode(m, bits)
except Exception as e:
    print("decode:", e, file=sys.stderr)
