"""C2 decode time and bpp vs tile shape (bf16): python scripts/probe_tiles.py"""
import sys
sys.path.insert(0, '.')
import paper_2207_05152_b200 as dl, synth
blob = open('fixtures/p100k_trained.dlicmdl', 'rb').read()
m = dl.dlic_model_load(blob, 0)
img = synth.config_images("C2", 1)[0]
dl.dlic_set_timing(True)
base = None
for tile in [(0, 0), (768, 256), (768, 128), (384, 256), (768, 64), (384, 128)]:
    best = 1e9
    for it in range(3):
        b = dl.dlic_encode(m, img, precision=1, tile=tile)
        d = dl.dlic_decode(m, b)
        assert (d == img).all()
        best = min(best, dl.dlic_last_kernel_ms("decode"))
    bpp = 8 * len(b) / img.size
    base = base or bpp
    print("tile %-10s bytes %7d bpp %.4f (%+.2f%%) decode %.3f ms" % (tile, len(b), bpp, 100 * (bpp / base - 1), best))
