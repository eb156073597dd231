import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2207_05152_b200 as dl, synth
blob = open('fixtures/p100k_trained.dlicmdl','rb').read()
m = dl.dlic_model_load(blob, 0)
img = synth.config_images("C2", 1)[0]
dl.dlic_set_timing(True)
for prec in (1, 0):
    for it in range(3):
        t=time.time(); b = dl.dlic_encode(m, img, precision=prec); te=time.time()-t
        enc = {k: dl.dlic_last_kernel_ms(k) for k in ("mlp","rans_enc","compact")}
        t=time.time(); d = dl.dlic_decode(m, b); td=time.time()-t
        dec = dl.dlic_last_kernel_ms("decode")
        assert (d==img).all()
    print("prec", prec, "bytes", len(b), "bpp %.4f" % (8*len(b)/img.size), "enc wall %.2f ms" % (te*1e3), enc, "dec wall %.2f ms" % (td*1e3), "dec kernel %.3f ms" % dec)
