"""Encoder-MLP and decode kernel times of the 12-bit P12 engine on one
256x256x35 12-bit MRI-like scan (Table III's size), for one or more
libdlic.so builds: python scripts/time_p12.py lib.so ..."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, os
sys.path.insert(0, %r)
os.environ["DLIC_LIB"] = %r
import numpy as np
import paper_2207_05152_b200 as dl, synth
m = dl.dlic_model_load(open(os.path.join(%r, "fixtures", "p12_seeded.dlicmdl"), "rb").read(), 0)
imgs = synth.mri_like_volume(256, 35, seed=0, bits=12)
dl.dlic_set_timing(True)
te, td = [], []
ok = True
for i in range(3):
    blob, sizes = dl.dlic_encode_batch(m, imgs)
    te.append(dl.dlic_last_kernel_ms("mlp"))
    back = dl.dlic_decode_batch(m, blob, sizes)
    td.append(dl.dlic_last_kernel_ms("decode"))
    ok = ok and bool((back == imgs).all())
print(json.dumps({"mlp_ms": sorted(te)[1], "decode_ms": sorted(td)[1], "bytes": len(blob), "ok": ok}))
'''
for lib in sys.argv[1:]:
    out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, os.path.abspath(lib), ROOT)], capture_output=True, text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")]
    print(lib, line[-1] if line else out.stderr[-600:])
