"""Decode-kernel time only (no correctness assertion: for timing experiments
with deliberately broken variant builds).  python scripts/time_decode.py [C2] lib.so ..."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, numpy as np
sys.path.insert(0, %r)
import paper_2207_05152_b200 as dl, synth
cfg = %r
blob = open(%r, "rb").read()
m = dl.dlic_model_load(blob, 0)
img = synth.config_images(cfg, 1)[0]
tile = {"C4": (384, 360), "C5": (768, 720)}.get(cfg, (0, 0))
dl.dlic_set_timing(True)
b = dl.dlic_encode(m, img, precision=1, tile=tile)
ts = []; ok = True
for i in range(8):
    try:
        d = dl.dlic_decode(m, b); ok = ok and bool((d == img).all())
    except dl.DlicError:
        ok = False
    ts.append(dl.dlic_last_kernel_ms("decode"))
print(json.dumps({"decode_ms": sorted(ts)[len(ts)//2], "ok": ok}))
'''
args = sys.argv[1:]
cfg = "C2"
if args and not args[0].endswith(".so"):
    cfg = args.pop(0)
blob = os.path.join(ROOT, "fixtures", "p100k_trained.dlicmdl")
for rep in range(2):
    for lib in args:
        env = dict(os.environ, DLIC_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg, blob)], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        print(lib, line[-1] if line else out.stderr[-400:])
