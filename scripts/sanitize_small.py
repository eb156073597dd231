"""Small encode/decode round trips for compute-sanitizer runs (racecheck/memcheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2207_05152_b200 as dl
import synth
blob = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "fixtures", "p100k_trained.dlicmdl"), "rb").read()
m = dl.dlic_model_load(blob, 0)
for (w, h, tile) in ((40, 30, (0, 0)), (700, 12, (0, 0)), (50, 40, (24, 20))):
    img = synth.natural_like(w, h, seed=w + h)
    for prec in (1, 0):
        b = dl.dlic_encode(m, img, precision=prec, tile=tile)
        assert np.array_equal(dl.dlic_decode(m, b), img), (w, h, prec)
print("ok")
