"""Decode-kernel and encoder-MLP times of one or more libdlic.so builds (A/B
across commits or experimental variants; no correctness assertion beyond a
lossless flag).  Env: TIME_MODEL (fixture file, default the trained P100K),
TIME_PREC (1 bf16, 0 fp32).
Uses its own minimal ctypes calls (dlic_model_load / dlic_encode /
dlic_decode / dlic_last_kernel_ms), which every build since round 1 exports.
python scripts/time_decode.py [C2|C3|C4|C5] lib.so ..."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, ctypes, numpy as np
sys.path.insert(0, %r)
import synth
lib = ctypes.CDLL(%r)
cfg = %r
blob = open(%r, "rb").read()
img = np.ascontiguousarray(synth.config_images(cfg, 1)[0])
tile = {"C4": (384, 360), "C5": (768, 720)}.get(cfg, (0, 0))
vp = ctypes.c_void_p
m = vp()
assert lib.dlic_model_load(blob, len(blob), 0, ctypes.byref(m)) == 0
opts = (ctypes.c_uint32 * 16)(%d, 32, tile[0], tile[1])      # precision, G, tile; later fields zero
lib.dlic_set_timing(1)
lib.dlic_last_kernel_ms.restype = ctypes.c_double
out = ctypes.POINTER(ctypes.c_uint8)()
n = ctypes.c_size_t()
h, w = img.shape
assert lib.dlic_encode(m, img.ctypes.data, w, h, w, opts, ctypes.byref(out), ctypes.byref(n)) == 0
bits = ctypes.string_at(out, n.value)
dec = np.empty_like(img)
ts = []
ok = True
for i in range(8):
    st = lib.dlic_decode(m, bits, len(bits), dec.ctypes.data, dec.size)
    ok = ok and st == 0 and bool((dec == img).all())
    ts.append(lib.dlic_last_kernel_ms(b"decode"))
tm = []
for i in range(5):
    assert lib.dlic_encode(m, img.ctypes.data, w, h, w, opts, ctypes.byref(out), ctypes.byref(n)) == 0
    ok = ok and ctypes.string_at(out, n.value) == bits
    tm.append(lib.dlic_last_kernel_ms(b"mlp"))
print(json.dumps({"decode_ms": sorted(ts)[len(ts)//2], "mlp_ms": sorted(tm)[len(tm)//2], "ok": ok}))
'''
args = sys.argv[1:]
cfg = "C2"
if args and not args[0].endswith(".so"):
    cfg = args.pop(0)
blob = os.path.join(ROOT, "fixtures", os.environ.get("TIME_MODEL", "p100k_trained.dlicmdl"))
prec = int(os.environ.get("TIME_PREC", "1"))  # 1 bf16, 0 fp32
for rep in range(2):
    for lib in args:
        out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, os.path.abspath(lib), cfg, blob, prec)],
                             capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        print(lib, line[-1] if line else out.stderr[-400:], flush=True)
