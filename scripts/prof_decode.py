"""Per-phase decoder clock profile (DLIC_PROF=1; thread 32 of each CTA)
for one or more library builds: python scripts/prof_decode.py [C2] lib.so ..."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys
sys.path.insert(0, %r)
import paper_2207_05152_b200 as dl, synth
cfg = %r
m = dl.dlic_model_load(open(%r, "rb").read(), 0)
img = synth.config_images(cfg, 1)[0]
tile = {"C4": (384, 360), "C5": (768, 720)}.get(cfg, (0, 0))
b = dl.dlic_encode(m, img, precision=1, tile=tile)
for i in range(2):
    d = dl.dlic_decode(m, b)
'''
args = sys.argv[1:]
cfg = "C2"
if args and not args[0].endswith(".so"):
    cfg = args.pop(0)
blob = os.path.join(ROOT, "fixtures", os.environ.get("DLIC_MODEL_FILE", "p100k_trained.dlicmdl"))
for lib in args or [os.path.join(ROOT, "paper_2207_05152_b200", "libdlic.so")]:
    env = dict(os.environ, DLIC_LIB=os.path.abspath(lib), DLIC_PROF="1")
    out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg, blob)], env=env, capture_output=True, text=True)
    print(lib)
    print("\n".join(l for l in out.stderr.splitlines() if "prof" in l)[-600:])
