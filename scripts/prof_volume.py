"""Per-phase clock profile (DLIC_PROF=1) of a volume decode vs the same slices
decoded as 2D images; also times both.  python scripts/prof_volume.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2207_05152_b200 as dl
import synth
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
m3 = dl.dlic_model_load(open(os.path.join(root, "fixtures", "p100k_3d.dlicmdl"), "rb").read(), 0)
m2 = dl.dlic_model_load(open(os.path.join(root, "fixtures", "p100k_trained.dlicmdl"), "rb").read(), 0)
d = int(sys.argv[1]) if len(sys.argv) > 1 else 32
vol = synth.mri_like_volume(256, d, seed=3)
dl.dlic_set_timing(True)
bits = dl.dlic_encode_volume(m3, vol)
blob, sizes = dl.dlic_encode_batch(m2, vol)
for name, f in (("volume", lambda: dl.dlic_decode_volume(m3, bits)), ("2d", lambda: dl.dlic_decode_batch(m2, blob, sizes))):
    ts = []
    for _ in range(3):
        out = f()
        ts.append(dl.dlic_last_kernel_ms("decode"))
    assert np.array_equal(out, vol)
    print(name, "decode ms", ["%.3f" % t for t in ts], flush=True)
os.environ["DLIC_PROF"] = "1"
