"""Measured logit errors of both GPU paths against the oracle, as quantiles of
the per-row relative L_inf error (the statistic the parity tests bound), over
several images; bf16 logits come from the production encoder k_enc_pp (its
debug exports).  Also the bf16/fp32 payload ratio on C2.
python scripts/measure_tol.py [p350k]   (p350k: the seeded P350K of
tests/test_gpu_p350k.py, bf16 only, streamed-weight engine)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2207_05152_b200 as dl
import synth
from oracle import mlp, model_io, window
P350K = len(sys.argv) > 1 and sys.argv[1] == "p350k"
if P350K:
    layers = synth.he_uniform_layers(mlp.P350K, seed=3, bias_scale=0.1)
    blob = model_io.save(layers)
else:
    blob = open("fixtures/p100k_trained.dlicmdl", "rb").read()
    layers = model_io.load(blob)
m = dl.dlic_model_load(blob, 0)
PRECS = (1,) if P350K else (0, 1)
allrel = {0: [], 1: []}
for seed, (w, h) in [(11, (61, 37)), (3, (128, 96)), (5, (200, 150)), (7, (256, 128))]:
    img = synth.natural_like(w, h, seed=seed)
    rows, cols = np.divmod(np.arange(h * w), w)
    x = window.features(window.gather_many(img, rows, cols))
    for prec in PRECS:
        out = dl.dlic_debug_mlp(m, img, precision=prec, probs=False, freqs=False, fc=False)
        ref = mlp.forward_fp64(layers, x) if prec == 0 else mlp.forward_bf16(layers, x)
        got = out["logits"].reshape(-1, 256)
        rel = np.abs(got - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)
        allrel[prec].append(rel)
for prec in PRECS:
    r = np.concatenate(allrel[prec])
    q = np.quantile(r, [0.5, 0.9, 0.99, 0.999, 0.9999])
    print("%s prec %d rows %d: median %.3g p90 %.3g p99 %.3g p99.9 %.3g p99.99 %.3g max %.3g  frac>1e-5 %.2e "
          "frac>1e-3 %.2e" % ("P350K" if P350K else "P100K", prec, r.size, q[0], q[1], q[2], q[3], q[4], r.max(),
                              (r > 1e-5).mean(), (r > 1e-3).mean()))
if P350K:
    sys.exit(0)
img = synth.config_images("C2", 1)[0]
b32 = dl.dlic_encode(m, img, precision=0)
b16 = dl.dlic_encode(m, img, precision=1)
p32 = dl.dlic_peek(b32)["payload_bytes"]
p16 = dl.dlic_peek(b16)["payload_bytes"]
print("C2 payload fp32 %d bf16 %d ratio %.5f" % (p32, p16, p16 / p32))
