"""Issuer-side cycle breakdown of the P350K streamed-weight engine (encoder
k_enc_mlp<2>): DLIC_PROF_STREAM=1 python scripts/prof_stream.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2207_05152_b200 as dl
import synth
name = os.environ.get("DLIC_MODEL_FILE", "p350k_seeded.dlicmdl")
blob = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "fixtures", name), "rb").read()
m = dl.dlic_model_load(blob, 0)
img = synth.config_images("C2", 1)[0]
if "p12" in name:  # 12-bit MRI-like slice
    img = synth.mri_like_volume(256, 1, seed=0, bits=12)[0]
for _ in range(3):
    fc = dl.dlic_debug_mlp(m, img, logits=False, probs=False, freqs=False)["fc"]
