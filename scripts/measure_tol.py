"""Measured logit errors of both GPU paths against the oracle (test images of
tests/test_gpu_parity.py), and the bf16/fp32 payload ratio on C2.
python scripts/measure_tol.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2207_05152_b200 as dl
import synth
from oracle import mlp, model_io, window
blob = open("fixtures/p100k_trained.dlicmdl", "rb").read()
layers = model_io.load(blob)
m = dl.dlic_model_load(blob, 0)
for seed, (w, h) in [(11, (61, 37)), (3, (128, 96))]:
    img = synth.natural_like(w, h, seed=seed)
    rows, cols = np.divmod(np.arange(h * w), w)
    x = window.features(window.gather_many(img, rows, cols))
    for prec in (0, 1):
        out = dl.dlic_debug_mlp(m, img, precision=prec, probs=False, freqs=False, fc=False)
        ref = mlp.forward_fp64(layers, x) if prec == 0 else mlp.forward_bf16(layers, x)
        got = out["logits"].reshape(-1, 256)
        rel = np.abs(got - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)
        print("%dx%d prec %d: max row rel err %.3g, median %.3g" % (w, h, prec, rel.max(), np.median(rel)))
img = synth.config_images("C2", 1)[0]
b32 = dl.dlic_encode(m, img, precision=0)
b16 = dl.dlic_encode(m, img, precision=1)
p32 = dl.dlic_peek(b32)["payload_bytes"]
p16 = dl.dlic_peek(b16)["payload_bytes"]
print("C2 payload fp32 %d bf16 %d ratio %.5f" % (p32, p16, p16 / p32))
