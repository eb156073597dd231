"""Time C2 (or another config) round trips for several builds of libdlic.so
(experiments): python scripts/variant_bench.py [config] lib1.so lib2.so ...
Each library runs in its own process (DLIC_LIB), reps alternate between them."""
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
ts = []; te = []
for i in range(8):
    b = dl.dlic_encode(m, img, precision=1, tile=tile); te.append(dl.dlic_last_kernel_ms("mlp"))
    d = dl.dlic_decode(m, b); ts.append(dl.dlic_last_kernel_ms("decode"))
    assert (d == img).all()
print(json.dumps({"decode_ms": sorted(ts)[len(ts)//2], "mlp_ms": sorted(te)[len(te)//2], "bytes": len(b)}))
'''
args = sys.argv[1:]
cfg = "C2"
if args and not args[0].endswith(".so"):
    cfg = args.pop(0)
blob = os.path.join(ROOT, "fixtures", "p100k_trained.dlicmdl")
res = {a: [] for a in args}
for rep in range(2):
    for lib in args:
        env = dict(os.environ, DLIC_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg, blob)], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        res[lib].append(json.loads(line[-1]) if line else {"error": out.stderr[-400:]})
for lib, r in res.items():
    print(lib, r)
