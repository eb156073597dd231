"""One C2 encode + decode (for ncu captures): python scripts/prof_once.py [bf16|fp32] [config]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2207_05152_b200 as dl
import synth
prec = 1 if (len(sys.argv) < 2 or sys.argv[1] == "bf16") else 0
cfg = sys.argv[2] if len(sys.argv) > 2 else "C2"
blob = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "fixtures", "p100k_trained.dlicmdl"), "rb").read()
m = dl.dlic_model_load(blob, 0)
img = synth.config_images(cfg, 1)[0]
tile = {"C4": (384, 360), "C5": (768, 720)}.get(cfg, (0, 0))
b = dl.dlic_encode(m, img, precision=prec, tile=tile)
d = dl.dlic_decode(m, b)
assert (d == img).all()
print("ok", len(b))
