import sys, os, json
sys.path.insert(0, os.getcwd())
import paper_2207_05152_b200 as dl, synth, numpy as np
blob = open('fixtures/p100k_trained.dlicmdl','rb').read()
m = dl.dlic_model_load(blob, 0)
img = synth.config_images('C2', 1)[0]
dl.dlic_set_timing(True)
ts=[]
for i in range(8):
    b = dl.dlic_encode(m, img, precision=1); ts.append(dl.dlic_last_kernel_ms("rans_enc"))
    assert (dl.dlic_decode(m, b) == img).all()
print(os.environ.get("DLIC_LIB"), sorted(ts)[4], len(b))
