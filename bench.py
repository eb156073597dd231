"""bench.py — DLIC hot path on B200: encode + decode Mpixel/s (8-bit gray) and bpp.

One step = one pass of the whole hot path over one
batch of synthetic input: encode every pixel at once (window gather -> MLP ->
softmax/Q1 -> rANS lanes -> compaction) and wavefront-decode the containers
back.  Default workload: BASELINE.json configs[1] (C2, one 768x512 Kodak-shaped
image per GPU), bf16 tcgen05 path, trained P100K weights, G = 32.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dlic|reference]
                  [--config C2] [--batch B] [--precision bf16|fp32]

N > 1: one process per GPU over NCCL.  `bench.py --gpus N` without WORLD_SIZE
in the environment re-launches itself under torch.distributed.run with N
ranks (127.0.0.1 rendezvous); under torchrun WORLD_SIZE must equal N.  Every
rank codes its own images (weak scaling; units are independent, P:103 lanes
never cross images) through paper_2207_05152_b200.dist.coded_step, whose only
collective is the all_gather of container sizes (north_star) -- the function
tests/test_dist.py runs under gloo.  C4 additionally reports one frame's 15
tiles split across the ranks (dist.encode_units_distributed, strong scaling)
under "strong_units".
--impl reference times the CPU oracle (oracle/) on the same workload (rank 0
only; C2: the whole image per step).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOP_PER_PX = 216576            # P100K, SURVEY App. A item 1 (2 * sum K*N)
FLOP_PER_PX_P350K = 695296      # P350K: 2 * (78*256 + 4*256*256 + 256*256)
# per front, layers 2-6 are a dependent MMA chain (layer 1 is issued a front
# early), M=64 tiles costing as M=128 (8192 FLOP/clk/SM): P100K 4 x 8 x 64 +
# 8 x 128 = 3072 cycles; P350K 5 x 16 x 128 = 10240 cycles
FRONT_FLOOR_CYC = {"p350k": 10240, "p12": 4 * 16 * 128 + 2 * 32 * 16 * 64}
# P12 (12-bit, reading R16): 78 -> 256x5 -> 4096; the head is evaluated twice
# (two-pass softmax): algorithmic work counts it once
FLOP_PER_PX_P12 = 2 * (78 * 256 + 4 * 256 * 256 + 256 * 4096)
# model fixtures: (file, metadata reals per image or None, description)
MODELS = {
    "p100k": ("p100k_trained.dlicmdl", None,
              "P100K briefly trained by the oracle (fixtures/p100k_trained.dlicmdl)"),
    "pool-meta": ("p100k_pool_meta.dlicmdl", [0.9, 3.0, 1.25],
                  "P100K-pool-meta: 78+3 metadata inputs, avg-pool 2 after layers 1 and 3, seeded random "
                  "(fixtures/p100k_pool_meta.dlicmdl; pooling folded into the next layer, metadata into a "
                  "per-image layer-1 bias: the tensor-core chain runs P100K's shapes, 216,576 FLOP/px)"),
    "p350k": ("p350k_seeded.dlicmdl", None,
              "P350K: 78 -> 256x5 -> 256 (349,184 parameters, reading R4), seeded He-uniform "
              "(fixtures/p350k_seeded.dlicmdl); bf16 only, weights streamed from L2 through a TMA ring "
              "(engine 2, 695,296 FLOP/px)"),
    "p12": ("p12_seeded.dlicmdl", None,
            "P12: 78 -> 256x5 -> 4096 (12-bit alphabet, 1,336,064 parameters, readings R15-R17), seeded "
            "He-uniform (fixtures/p12_seeded.dlicmdl); bf16 only, streamed weights, two-pass 4096-wide head "
            "(engine 3); images: 12-bit MRI-like slices (u16)"),
    "3d": ("p100k_3d.dlicmdl", None,
           "P100K-3D: 78 + the 3x3 box of the slice below (87 inputs) -> 128x5 -> 256, seeded random "
           "(fixtures/p100k_3d.dlicmdl; the 9 lower taps enter layer 1 through the bias term, 2,304 FLOP/px on "
           "the CUDA cores on top of P100K's 216,576 on the tensor cores)"),
}
CONFIG_DESC = {
    "C1": "C1 32x32 gradient+noise, single stream (G=32=H)",
    "C2": "C2 768x512 Kodak-shaped natural-like, 1 image per GPU per step",
    "C3": "C3 256x256 MRI-like slices",
    "C4": "C4 1920x1080 natural-like, tiles 384x360",
    "C5": "C5 3840x2160 natural-like, tiles 768x720",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dlic", choices=["dlic", "reference"])
    ap.add_argument("--config", default="C2", choices=list(CONFIG_DESC))
    ap.add_argument("--batch", type=int, default=0, help="images per GPU per step (0 = config default)")
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tile", default="", help="WxH independent tiles (default: the config's)")
    ap.add_argument("--no-variants", action="store_true", help="skip the strip-tiled C2 side measurement")
    ap.add_argument("--no-strong", action="store_true", help="skip C4's unit-split (strong scaling) measurement")
    ap.add_argument("--volume", type=int, default=0,
                    help="volume depth: code each group of D consecutive images as one volume (3D window; "
                         "--model 3d; default 32 with it)")
    ap.add_argument("--model", default="p100k", choices=list(MODELS),
                    help="p100k: trained fixture; pool-meta: the f4 network (pooling + 3 metadata inputs)")
    return ap.parse_args()


def relaunch_distributed(args):
    """`--gpus N` (N > 1) outside torchrun: run this script under
    torch.distributed.run with N ranks on this node and return its exit code
    (rank 0 prints the JSON line)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.25)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d (launch N ranks for N GPUs)" % (args.gpus, ws))
    if ws > torch.cuda.device_count():
        raise SystemExit("bench.py: %d ranks but %d visible GPUs" % (ws, torch.cuda.device_count()))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    return ws, rank, local


def synth_volumes(args, rank, n, vd):
    import synth
    vols = [synth.mri_like_volume(256, vd, seed=100 * rank + v) for v in range(n // vd)]
    return np.ascontiguousarray(np.concatenate(vols)[:, :args_h(args), :args_w(args)])


def args_h(args):
    return {"C1": 32, "C2": 512, "C3": 256, "C4": 1080, "C5": 2160}[args.config]


def args_w(args):
    return {"C1": 32, "C2": 768, "C3": 256, "C4": 1920, "C5": 3840}[args.config]


def images_for(args, rank, n):
    import synth
    cfg = args.config
    if args.model == "p12":   # 12-bit MRI-like slices, 256x256 (C3 geometry)
        per = 35               # Table III's scan: 256 x 256 x 35
        vols = [synth.mri_like_volume(256, per, seed=100 * rank + v, bits=12) for v in range((n + per - 1) // per)]
        return np.ascontiguousarray(np.concatenate(vols)[:n, :args_h(args), :args_w(args)])
    if cfg == "C1":
        return np.stack([synth.gradient_noise(32, 32, seed=rank * 1000 + i) for i in range(n)])
    if cfg == "C2":
        return np.stack([synth.c2_image(seed=rank * 1000 + i) for i in range(n)])
    if cfg == "C3":
        return synth.mri_like_slices(n, 256, seed0=rank * 100)
    if cfg == "C4":
        return np.stack([synth.natural_like(1920, 1080, seed=100 + rank * 1000 + i, wavelength_scale=2.5)
                         for i in range(n)])
    return np.stack([synth.natural_like(3840, 2160, seed=200 + rank * 1000 + i, wavelength_scale=5.0)
                     for i in range(n)])


def opts_for(cfg):
    c = {"C1": (32, (0, 0)), "C2": (32, (0, 0)), "C3": (32, (0, 0)), "C4": (32, (384, 360)),
         "C5": (32, (768, 720))}[cfg]
    return c


def tile_for(args):
    g, tile = opts_for(args.config)
    if args.tile:
        w, h = (int(x) for x in args.tile.lower().split("x"))
        tile = (w, h)
    return g, tile


def measure_variant(dl, model, d_imgs, prec, g, tile, reps=5):
    """Decode time (CUDA events inside the library, best of reps) and bpp of
    the same images coded with another tile shape (device batch API)."""
    import torch
    n = d_imgs.shape[0]
    d_out, d_sizes, stride = dl.dlic_encode_batch_device(model, d_imgs, prec, g, tile)
    torch.cuda.synchronize()
    sizes = d_sizes.cpu().numpy()
    hdr = dl.dlic_peek(d_out[:int(sizes[0])].cpu().numpy().tobytes())
    d_dec = torch.empty_like(d_imgs)
    d_status = torch.zeros(n, dtype=torch.int32, device=d_imgs.device)
    offs = [i * stride for i in range(n)]
    lens = [int(x) for x in sizes]
    best = 1e30
    for _ in range(reps):
        dl.dlic_decode_batch_device(model, d_out, offs, lens, hdr, d_dec, d_status)
        torch.cuda.synchronize()
        best = min(best, dl.dlic_last_kernel_ms("decode"))
    assert int(d_status.abs().sum()) == 0 and torch.equal(d_dec, d_imgs), "variant round trip failed"
    px = d_imgs.numel()
    return {"tile": list(tile), "decode_ms": best, "decode_mpx_s": px / (best / 1e3) / 1e6,
            "bpp_total": 8.0 * float(sizes.sum()) / px}


def default_batch(cfg, model=None):
    if model == "p12":
        return 35
    # C3: 512 slices across 8 GPUs = 64 per GPU; C5: "batch of 64" per GPU
    # (960 tiles of 768x720 -> 26 waves of 37 four-CTA clusters: no tail)
    return {"C1": 1, "C2": 1, "C3": 64, "C4": 1, "C5": 64}[cfg]


def cpu_info():
    """CPU model and the BLAS thread count the oracle runs with."""
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
    except Exception:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "blas_threads": blas}


# ------------------------------------------------------------------ reference arm (CPU oracle)
METRIC = "encode+decode Mpixel/s (8-bit gray, round trip) and bpp"


def volume_depth(args):
    if args.model == "3d":
        return args.volume or 32
    return 0


def arm_config(args, n, W, H, tile, g, ws):
    """The config object of the JSON line (both arms)."""
    vd = volume_depth(args)
    extra = {"volume_depth": vd, "volumes_per_gpu": n // vd} if vd else {}
    if args.model == "p12":
        extra = dict(extra, alphabet_bits=12)
    wl = CONFIG_DESC[args.config]
    if args.model == "p12":
        wl = "C3 geometry at the paper's MRI bit depth: 12-bit MRI-like slices 256x256, 35 per GPU (Table III's scan)"
    return dict({"workload": wl, "images_per_gpu": n, "width": W, "height": H,
            "tile": list(tile), "group_rows": g, "precision": args.precision,
            "weights": MODELS[args.model][2],
            "l2": "flushed between timed steps (256 MiB write, untimed)", "parallelism": "dp%d" % ws}, **extra)


def run_reference(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import codec  # the one other place bench.py executes oracle/
    with open(os.path.join(ROOT, "fixtures", MODELS[args.model][0]), "rb") as fh:
        blob = fh.read()
    meta = MODELS[args.model][1]
    img = images_for(args, 0, 1)[0]
    # one whole image per step for C1-C3 (C2: ~10 s of oracle work); larger
    # configs: the top-left 768x512 of the first image (~10 s)
    sh, sw = min(img.shape[0], 512), min(img.shape[1], 768)
    if args.model == "p12":
        sh, sw = 96, 96
    sample = np.ascontiguousarray(img[:sh, :sw])
    prec = 1 if args.precision == "bf16" else 0
    g, _ = opts_for(args.config)
    vd = volume_depth(args)
    if vd:   # the oracle's volume coder on the first 4 slices of a volume (~5-10 s)
        sample = synth_volumes(args, 0, vd, vd)[:4]
        sh, sw = sample.shape[1:]
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if vd:
            b = codec.encode_volume(sample, blob, prec, g, meta=meta)
            out = codec.decode_volume(b, blob)
        else:
            b = codec.encode(sample, blob, prec, g, meta=meta)
            out = codec.decode(b, blob)
        dt = time.perf_counter() - t0
        assert np.array_equal(out, sample)
        if i >= args.warmup:
            times.append(dt)
    ms = statistics.mean(times) * 1e3
    mpx = sample.size / (ms / 1e3) / 1e6
    ci = cpu_info()
    cores = ci["blas_threads"] or ci["logical_cpus"] or 1
    whole = sample.shape == img.shape or vd > 0
    what = ("%d slices %dx%d of a volume (3D window)" % (sample.shape[0], sw, sh)) if vd else None
    line = {
        "impl": "reference", "metric": METRIC, "value": mpx,
        "unit": "Mpixel/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64-accum bf16-emulated" if prec else "f64", "data": "synthetic",
        "config": dict(arm_config(args, default_batch(args.config) if not args.batch else args.batch,
                                  img.shape[1], img.shape[0], tile_for(args)[1], g, ws),
                       sample=("per step the oracle codes " + what) if vd else
                       ("per step the oracle codes one whole %dx%d image (untiled)" % (sw, sh)) if whole
                       else "per step the oracle codes a top-left %dx%d crop of one image (untiled)" % (sw, sh)),
        "cpu_baseline": dict({"value": mpx, "unit": "Mpixel/s", "cores": cores, "kind": "oracle",
                              "sample": what if vd else
                              ("the whole %s image (%dx%d), oracle encode+decode per step" % (args.config, sw, sh))
                              if whole else "top-left %dx%d crop of the %s image, oracle encode+decode per step"
                              % (sw, sh, args.config)}, **ci),
        "e2e": {"value": mpx, "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(args, img):
    """Oracle (as it stands) on a bounded sample of the workload (~10 s)."""
    from oracle import codec
    with open(os.path.join(ROOT, "fixtures", MODELS[args.model][0]), "rb") as fh:
        blob = fh.read()
    sh, sw = min(img.shape[0], 512), min(img.shape[1], 768)   # C2: the whole image (~10-15 s)
    if args.model == "p12":   # 4096 outputs: a 96x96 corner (~10-20 s)
        sh, sw = 96, 96
    sample = np.ascontiguousarray(img[:sh, :sw])
    prec = 1 if args.precision == "bf16" else 0
    vd = volume_depth(args)
    t0 = time.perf_counter()
    if vd:
        sample = synth_volumes(args, 0, vd, vd)[:4]
        b = codec.encode_volume(sample, blob, prec, 32)
        out = codec.decode_volume(b, blob)
    else:
        b = codec.encode(sample, blob, prec, 32, meta=MODELS[args.model][1])
        out = codec.decode(b, blob)
    dt = time.perf_counter() - t0
    assert np.array_equal(out, sample)
    ci = cpu_info()
    cores = ci["blas_threads"] or ci["logical_cpus"] or 1
    return dict({"value": sample.size / dt / 1e6, "unit": "Mpixel/s", "cores": cores, "kind": "oracle",
                 "sample": "top-left %dx%d crop of the %s image: oracle encode+decode (%.1f s)"
                           % (sw, sh, args.config, dt)}, **ci)


def measure_strong_units(dl, model, img, prec, g, tile, ws, rank, dev, args):
    """C4: ONE frame's tiles split across the ranks (strong scaling), through
    the public unit-range calls with host buffers: each rank codes its units
    (dlic_encode_units: H2D of the frame, D2H of its payload), the stream sizes
    are all-gathered (dist.encode_units_distributed), then each rank decodes
    its units (dlic_decode_units).  Timed per frame as the max over ranks."""
    import torch
    from paper_2207_05152_b200 import dist as dd
    h, w = img.shape
    n_units = dl.dlic_peek(dl.dlic_encode(model, img, prec, g, tile))["n_units"]
    out = np.zeros_like(img)
    state = {}

    def enc(lo, hi):
        return dl.dlic_encode_units(model, img, lo, hi, prec, g, tile)

    def frame():
        if ws > 1:
            payload, rng, soffs, all_ssz = dd.encode_units_distributed(enc, n_units)
        else:
            payload, ssz = enc(0, n_units)
            rng, all_ssz = (0, n_units), ssz
        state["rng"] = rng
        # a rank decodes its own units of the container (framed here from
        # the gathered sizes; every payload byte of its range is its own)
        lo, hi = rng
        if hi > lo:
            first, nst = dl.dlic_unit_streams(w, h, lo, hi, prec, g, tile)
            sizes = [int(x) for x in all_ssz]
            full = bytearray(sum(sizes))
            off = sum(sizes[:first])
            full[off:off + len(payload)] = payload
            bits = dl.dlic_container_build(w, h, model.sha256(), sizes, bytes(full), prec, g, tile)
            dl.dlic_decode_units(model, bits, lo, hi, out)

    for _ in range(args.warmup):
        frame()
    times = []
    for _ in range(args.steps):
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        frame()
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
    ms = statistics.mean(times)
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        allt = [torch.empty_like(t) for _ in range(ws)]
        torch.distributed.all_gather(allt, t)
        ms = max(float(x[0]) for x in allt)
    lo, hi = state["rng"]
    tiles = [(x0, y0) for y0 in range(0, h, tile[1]) for x0 in range(0, w, tile[0])]
    for (x0, y0) in tiles[lo:hi]:
        assert np.array_equal(out[y0:y0 + tile[1], x0:x0 + tile[0]], img[y0:y0 + tile[1], x0:x0 + tile[0]])
    return {"scaling": "strong", "what": "one 1920x1080 frame, its %d tiles split across %d rank(s); host buffers, "
            "encode+decode per frame, max over ranks" % (n_units, ws), "ms_per_frame": ms,
            "mpx_s": img.size / (ms / 1e3) / 1e6, "units_per_rank": hi - lo}


# ------------------------------------------------------------------ product arm
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args))
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    ws, rank, local = dist_setup(args)
    import paper_2207_05152_b200 as dl

    dev = torch.device("cuda", local)
    with open(os.path.join(ROOT, "fixtures", MODELS[args.model][0]), "rb") as fh:
        blob = fh.read()
    model = dl.dlic_model_load(blob, local)
    prec = 1 if args.precision == "bf16" else 0
    g, tile = tile_for(args)
    n = args.batch or default_batch(args.config, args.model)
    imgs = images_for(args, rank, n)
    vd = volume_depth(args)
    if vd and n % vd:
        raise SystemExit("bench.py: %d images per GPU is not a multiple of the volume depth %d" % (n, vd))
    if vd:  # slices of a volume: consecutive MRI-like slices of one volume (synth.mri_like_slices)
        imgs = synth_volumes(args, rank, n, vd)
    meta = None if MODELS[args.model][1] is None else np.tile(np.array(MODELS[args.model][1], np.float32), (n, 1))
    _, H, W = imgs.shape
    px_rank = n * H * W
    stream = torch.cuda.current_stream(dev)
    d_imgs = torch.from_numpy(imgs.view(np.int16) if imgs.dtype == np.uint16 else imgs).to(dev)   # (u16: same bytes)
    d_dec = torch.empty_like(d_imgs)
    d_status = torch.zeros(n, dtype=torch.int32, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    dl.dlic_set_timing(True)

    # first pass: planning header + correctness check of this batch
    d_out, d_sizes, stride = dl.dlic_encode_batch_device(model, d_imgs, prec, g, tile, meta=meta, volume_depth=vd)
    torch.cuda.synchronize()
    sizes = d_sizes.cpu().numpy()
    hdr = dl.dlic_peek(d_out[:int(sizes[0])].cpu().numpy().tobytes())
    offs = [i * stride for i in range(len(sizes))]
    lens = [int(x) for x in sizes]       # the encoder is deterministic: every step writes these sizes
    dl.dlic_decode_batch_device(model, d_out, offs, lens, hdr, d_dec, d_status)
    torch.cuda.synchronize()
    assert int(d_status.abs().sum()) == 0 and torch.equal(d_dec, d_imgs), "round trip failed"
    total_bytes = int(sizes.sum())
    payload = total_bytes - len(sizes) * hdr["header_bytes"]

    from paper_2207_05152_b200 import dist as dd

    def encode_local():
        dl.dlic_encode_batch_device(model, d_imgs, prec, g, tile, d_out=d_out, d_sizes=d_sizes, meta=meta,
                                    volume_depth=vd)
        return d_sizes

    def decode_local():
        dl.dlic_decode_batch_device(model, d_out, offs, lens, hdr, d_dec, d_status)

    def step():
        if ws > 1:   # the only collective: all_gather of the container sizes (dist.coded_step)
            dd.coded_step(encode_local, decode_local)
        else:
            encode_local()
            decode_local()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    enc_ms, dec_ms = [], []
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)                    # L2 flush between timed steps (not timed)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            enc_ms.append(dl.dlic_last_kernel_ms("mlp") + dl.dlic_last_kernel_ms("rans_enc")
                          + dl.dlic_last_kernel_ms("compact"))
            dec_ms.append(dl.dlic_last_kernel_ms("decode"))
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = statistics.mean(step_ms)
    t_enc = statistics.mean(enc_ms)
    t_dec = statistics.mean(dec_ms)
    mlp_ms = dl.dlic_last_kernel_ms("mlp")
    if ws > 1:
        t = torch.tensor([ms, t_enc, t_dec], dtype=torch.float64, device=dev)
        allt = [torch.empty_like(t) for _ in range(ws)]
        dist.all_gather(allt, t)
        ms, t_enc, t_dec = (max(float(x[i]) for x in allt) for i in range(3))
    assert int(d_status.abs().sum()) == 0 and torch.equal(d_dec, d_imgs)
    clocks = clk.summary()

    # ---- e2e: public host API, host buffers, H2D/D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        pin_imgs = torch.from_numpy(imgs).pin_memory().numpy()
        e_ms = []
        h2d = d2h = 0
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tot_in = tot_out = 0
            if vd:  # the volume calls: one container per volume
                blob, sizes_e = dl.dlic_encode_batch(model, pin_imgs, prec, g, tile, meta=meta, volume_depth=vd)
                back = dl.dlic_decode_batch(model, blob, sizes_e)
                nb = len(blob)
            elif n == 1:  # the paper's calls: encode(image) -> bits, decode(bits) -> image
                b = dl.dlic_encode(model, pin_imgs[0], prec, g, tile, meta=None if meta is None else meta[0])
                back = dl.dlic_decode(model, b)[None]
                nb = len(b)
            else:  # the same calls over the rank's batch: one H2D and one D2H each way
                blob, sizes = dl.dlic_encode_batch(model, pin_imgs, prec, g, tile, meta=meta)
                back = dl.dlic_decode_batch(model, blob, sizes)
                nb = len(blob)
            tot_in = pin_imgs.nbytes + nb
            tot_out = nb + back.nbytes
            dt = (time.perf_counter() - t0) * 1e3
            if i >= args.warmup:
                e_ms.append(dt)
                h2d, d2h = tot_in, tot_out
            assert np.array_equal(back, pin_imgs)
        em = statistics.mean(e_ms)
        if ws > 1:
            t = torch.tensor([em], dtype=torch.float64, device=dev)
            allt = [torch.empty_like(t) for _ in range(ws)]
            dist.all_gather(allt, t)
            em = max(float(x[0]) for x in allt)
        e2e = {"value": ws * px_rank / (em / 1e3) / 1e6, "unit": "Mpixel/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": em}

    strong = None
    if args.config == "C4" and tile != (0, 0) and not args.no_strong and meta is None:
        strong = measure_strong_units(dl, model, imgs[0], prec, g, tile, ws, rank, dev, args)

    variants = None
    if rank == 0 and ws == 1 and args.config == "C2" and tile == (0, 0) and not args.no_variants and meta is None:
        # the same image as 4 independent 768x128 strips (north_star: "independent
        # image tiles with their own streams"): 1149 instead of 2301 fronts
        variants = {"strips_768x128": measure_variant(dl, model, d_imgs, prec, g, (768, 128))}

    if rank == 0:
        peaks, src = load_peaks()
        # dominant kernel: the wavefront decoder (latency-bound front chain)
        fpp = {"p350k": FLOP_PER_PX_P350K, "p12": FLOP_PER_PX_P12}.get(args.model, FLOP_PER_PX)
        dec_flops = fpp * px_rank
        achieved = dec_flops / (t_dec / 1e3) / 1e12
        # fp32 path runs on CUDA-core FFMA: 148 SMs x 128 FMA/clk x 2 x sm_max
        peak = peaks["bf16_tflops"] if prec == 1 else 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        traffic = None   # dram bytes per k_decode launch from a stored ncu --set full capture (not this run)
        try:
            if args.model != "p100k":
                raise OSError("stored captures are of the P100K decoder")
            with open(os.path.join(ROOT, "profiles", "decode_traffic.json")) as fh:
                traffic = json.load(fh).get("%s_%s" % (args.config, args.precision))
        except (OSError, ValueError):
            pass
        tw, th = (W, H) if tile == (0, 0) else (min(tile[0], W), min(tile[1], H))
        T = tw + 3 * (th - 1)
        floor_ms = T * FRONT_FLOOR_CYC.get(args.model, 3072) / (peaks.get("sm_max_mhz", 1965.0) * 1e3)
        cpu = cpu_baseline_sample(args, imgs[0]) if ws == 1 else None   # N=1 only (contract)
        line = {
            "metric": METRIC,
            "value": ws * px_rank / (ms / 1e3) / 1e6,
            "unit": "Mpixel/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16" if prec == 1 else "f32", "data": "synthetic",
            "config": arm_config(args, n, W, H, tile, g, ws),
            "encode_mpx_s": ws * px_rank / (t_enc / 1e3) / 1e6,
            "decode_mpx_s": ws * px_rank / (t_dec / 1e3) / 1e6,
            "encode_ms": t_enc, "decode_ms": t_dec, "mlp_ms": mlp_ms,
            "bpp_total": 8.0 * total_bytes / px_rank, "bpp_payload": 8.0 * payload / px_rank,
            "roofline": {"kernel": "k_decode<%s>" % ({"p350k": 2, "p12": 3}.get(args.model, args.precision)), "bound": "tensor" if prec == 1 else "alu", "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                         "peak_source": src + (" bf16_tflops" if prec == 1 else " sm_max_mhz x 148 SM x 128 FFMA x 2 (DESIGN.md)"),
                         "traffic_source": "stored ncu --set full capture of this config's k_decode launch "
                                           "(profiles/decode_traffic.json), not measured in this run",
                         "latency_floor_ms": floor_ms, "latency_frac": floor_ms / t_dec},
            # the throughput-bound encoder MLP (all pixels at once) against the same peak
            "roofline_encode": {"kernel": ({"p350k": "k_enc_mlp<2>", "p12": "k_enc_mlp<3>"}.get(args.model, "k_enc_pp"))
                                if prec == 1
                                else "k_enc_mlp<fp32>",
                                "bound": "tensor" if prec == 1 else "alu",
                                "achieved": fpp * px_rank / (mlp_ms / 1e3) / 1e12, "peak": peak,
                                "unit": "TFLOP/s",
                                "frac": fpp * px_rank / (mlp_ms / 1e3) / 1e12 / peak,
                                "note": "M=64 tcgen05 tiles cost as M=128: ceiling 0.5 of peak (DESIGN.md)"},
            "variants": variants,
            "strong_units": strong,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": 6 * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
