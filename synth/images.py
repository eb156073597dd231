"""Seeded 8-bit grayscale image generators (SURVEY.md §8(d) recipes).

All functions return C-contiguous ``numpy.uint8`` arrays of shape (H, W)
(row-major, as the C-ABI expects) and depend only on their arguments.
"""

from __future__ import annotations

import numpy as np


def _box_blur(a: np.ndarray, k: int) -> np.ndarray:
    """k x k box blur with edge replication (separable running sums)."""
    p = k // 2
    b = np.pad(a, p, mode="edge")
    c = np.cumsum(b, axis=0)
    c = np.concatenate([np.zeros((1, c.shape[1])), c], axis=0)
    v = (c[k:] - c[:-k]) / k
    c = np.cumsum(v, axis=1)
    c = np.concatenate([np.zeros((c.shape[0], 1)), c], axis=1)
    return (c[:, k:] - c[:, :-k]) / k


def gradient_noise(width: int = 32, height: int = 32, seed: int = 0) -> np.ndarray:
    """C1: clip(round(64 + 4r + 2c + N(0, 4^2)), 0, 255)."""
    rng = np.random.default_rng(seed)
    r = np.arange(height)[:, None]
    c = np.arange(width)[None, :]
    v = 64.0 + 4.0 * r + 2.0 * c + rng.normal(0.0, 4.0, size=(height, width))
    return np.ascontiguousarray(np.clip(np.rint(v), 0, 255).astype(np.uint8))


def natural_like(width: int = 768, height: int = 512, seed: int = 0,
                 sigma_tex: float = 2.0, sigma_n: float = 1.0,
                 wavelength_scale: float = 1.0) -> np.ndarray:
    """C2/C4/C5 "natural-like" photo stand-in.

    base 128 + 6 random 2D cosines (wavelength 64-512 px x scale, amplitude
    U(20,60)/2) + 3-6 constant-offset ellipses (radii 20-200 px x scale,
    offset +-40, hard edges) + band-limited texture (5x5 box-blurred white
    noise scaled to sigma_tex) + white noise sigma_n; rounded and clipped.
    """
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:height, 0:width].astype(np.float64)
    v = np.full((height, width), 128.0)
    for _ in range(6):
        lam = rng.uniform(64.0, 512.0) * wavelength_scale
        th = rng.uniform(0.0, np.pi)
        ph = rng.uniform(0.0, 2 * np.pi)
        amp = rng.uniform(20.0, 60.0) / 2.0
        v += amp * np.cos(2 * np.pi * (xx * np.cos(th) + yy * np.sin(th)) / lam + ph)
    for _ in range(int(rng.integers(3, 7))):
        cy, cx = rng.uniform(0, height), rng.uniform(0, width)
        ry, rx = rng.uniform(20, 200, size=2) * wavelength_scale
        off = rng.uniform(-40.0, 40.0)
        v += off * ((((yy - cy) / ry) ** 2 + ((xx - cx) / rx) ** 2) <= 1.0)
    tex = _box_blur(rng.normal(0.0, 1.0, size=(height, width)), 5)
    sd = tex.std()
    if sd > 0:
        v += tex * (sigma_tex / sd)
    v += rng.normal(0.0, sigma_n, size=(height, width))
    return np.ascontiguousarray(np.clip(np.rint(v), 0, 255).astype(np.uint8))


def mri_like_volume(size: int = 256, slices: int = 32, seed: int = 0, bits: int = 8) -> np.ndarray:
    """C3 "MRI-like" volume (Fig. 5): (slices, size, size) u8.

    Rician background |N(0,2)+iN(0,2)|, a head ellipse and 3-8 inner ellipses
    whose smooth intensities (40-220) and radii vary smoothly across slices.
    The histogram is heavily skewed toward the dark background.
    bits=12 (the paper's MRI bit depth): every intensity and noise
    scale x16, values in [0, 4095], u16 (the same draws as bits=8).
    """
    sc = float(1 << (bits - 8))
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    out = np.empty((slices, size, size), dtype=np.uint8 if bits == 8 else np.uint16)
    n_in = int(rng.integers(3, 9))
    head = dict(cy=size / 2 + rng.uniform(-8, 8), cx=size / 2 + rng.uniform(-8, 8),
                ry=size * rng.uniform(0.36, 0.44), rx=size * rng.uniform(0.30, 0.38),
                val=rng.uniform(90, 140))
    inner = []
    for _ in range(n_in):
        inner.append(dict(cy=head["cy"] + rng.uniform(-0.5, 0.5) * head["ry"],
                          cx=head["cx"] + rng.uniform(-0.5, 0.5) * head["rx"],
                          ry=rng.uniform(0.05, 0.25) * size, rx=rng.uniform(0.05, 0.25) * size,
                          val=rng.uniform(40, 220), drift=rng.uniform(-0.5, 0.5)))
    for s in range(slices):
        z = (s - slices / 2) / max(slices, 1)
        shrink = np.sqrt(max(1.0 - (2 * z) ** 2 * 0.6, 0.2))
        v = np.abs(rng.normal(0, 2, (size, size)) + 1j * rng.normal(0, 2, (size, size)))
        hm = (((yy - head["cy"]) / (head["ry"] * shrink)) ** 2
              + ((xx - head["cx"]) / (head["rx"] * shrink)) ** 2) <= 1.0
        shade = head["val"] * (1.0 - 0.25 * (((yy - head["cy"]) / size) ** 2 + ((xx - head["cx"]) / size) ** 2))
        v = np.where(hm, shade + rng.normal(0, 3, (size, size)), v)
        for e in inner:
            m = (((yy - e["cy"] - 20 * z * e["drift"]) / (e["ry"] * shrink)) ** 2
                 + ((xx - e["cx"]) / (e["rx"] * shrink)) ** 2) <= 1.0
            v = np.where(m & hm, e["val"] * (1 + 0.3 * z * e["drift"]) + rng.normal(0, 3, (size, size)), v)
        out[s] = np.clip(np.rint(v * sc), 0, (1 << bits) - 1).astype(out.dtype)
    return out


def mri_like_slices(count: int = 512, size: int = 256, seed0: int = 0) -> np.ndarray:
    """C3 batch: 16 volumes x 32 slices (count/32 volumes), (count, size, size) u8."""
    per = 32
    vols = []
    nvol = (count + per - 1) // per
    for v in range(nvol):
        vols.append(mri_like_volume(size, per, seed=seed0 + v))
    return np.ascontiguousarray(np.concatenate(vols, axis=0)[:count])


def random_image(width: int, height: int, seed: int = 0, kind: str = "uniform") -> np.ndarray:
    """Small random test images: 'uniform' i.i.d. bytes, 'smooth' low-noise ramp, 'const'."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.integers(0, 256, size=(height, width), dtype=np.uint8)
    if kind == "const":
        return np.full((height, width), int(rng.integers(0, 256)), dtype=np.uint8)
    r = np.arange(height)[:, None]
    c = np.arange(width)[None, :]
    v = 100 + 3 * r + c + rng.normal(0, 2, size=(height, width))
    return np.ascontiguousarray(np.clip(np.rint(v), 0, 255).astype(np.uint8))


# Concrete workloads of BASELINE.json "configs".
CONFIGS = {
    "C1": dict(width=32, height=32, count=1, group_rows=32, tile=(0, 0)),
    "C2": dict(width=768, height=512, count=1, group_rows=32, tile=(0, 0)),
    "C3": dict(width=256, height=256, count=512, group_rows=32, tile=(0, 0)),
    "C4": dict(width=1920, height=1080, count=1, group_rows=32, tile=(384, 360)),
    "C5": dict(width=3840, height=2160, count=64, group_rows=32, tile=(768, 720)),
}


# C2's texture and noise levels: chosen so that the trained P100K fixture's
# information content on the C2 image lies inside the paper's photo range of
# 3.53-4.27 bpp (Table I): 3.77 bits/px on its top-left 384x256
# (oracle fp64 network, -log2 p of the true symbol); the generator's defaults
# (texture 2, noise 1) give 2.81 there.
C2_SIGMA_TEX = 3.0
C2_SIGMA_N = 2.0


def c2_image(seed: int = 0) -> np.ndarray:
    """The C2 768x512 photo stand-in (natural_like at C2's texture/noise levels)."""
    return natural_like(768, 512, seed=seed, sigma_tex=C2_SIGMA_TEX, sigma_n=C2_SIGMA_N)


def config_images(name: str, count: int | None = None, seed0: int | None = None) -> np.ndarray:
    """(n, H, W) u8 images for config C1..C5 (optionally only the first `count`)."""
    cfg = CONFIGS[name]
    n = cfg["count"] if count is None else count
    if name == "C1":
        return gradient_noise(32, 32, seed=0 if seed0 is None else seed0)[None]
    if name == "C2":
        s0 = 0 if seed0 is None else seed0
        return np.stack([c2_image(seed=s0 + i) for i in range(n)])
    if name == "C3":
        return mri_like_slices(n, 256, seed0=0 if seed0 is None else seed0)
    if name == "C4":
        s0 = 100 if seed0 is None else seed0
        return np.stack([natural_like(1920, 1080, seed=s0 + i, wavelength_scale=2.5) for i in range(n)])
    if name == "C5":
        s0 = 200 if seed0 is None else seed0
        return np.stack([natural_like(3840, 2160, seed=s0 + i, wavelength_scale=5.0) for i in range(n)])
    raise KeyError(name)
