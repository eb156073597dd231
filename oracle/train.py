"""Brief trainer for fixture weights (oracle; test infrastructure only).

P:110 — networks are trained with categorical cross-entropy; "vloss" is that
loss on validation data in bits per pixel.  The paper's data (CLIC 2019
mobile) and weights are unavailable, so north_star allows weights "briefly
trained by the oracle on synthetic smooth-plus-noise images".  Optimiser:
Adam (SPEC S:313 names no other); loss in bits (log base 2).

Plain PyTorch CPU ops serve as the autodiff + matmul library.  Training is
not part of the coder being checked; parity unpinned beyond the SPEC
trainability checks in tests (vloss of a uniform model is exactly 8 bits).
"""

from __future__ import annotations

import numpy as np

from . import mlp, window


def dataset(images, fill: int = 0):
    """One sample per pixel: (78 window features, target value)."""
    xs, ys = [], []
    for img in images:
        h, w = img.shape
        rr, cc = np.divmod(np.arange(h * w), w)
        xs.append(window.gather_many(img, rr, cc, fill).astype(np.float32) / 256.0)
        ys.append(img.reshape(-1).astype(np.int64))
    return np.concatenate(xs), np.concatenate(ys)


def vloss_bits(layers, x: np.ndarray, y: np.ndarray) -> float:
    """Mean -log2 p(target) under the fp64 forward (P:110 vloss)."""
    from . import quant
    lg = mlp.forward_fp64(layers, x)
    p = quant.softmax_fp64(lg)
    return float(np.mean(-np.log2(np.maximum(p[np.arange(len(y)), y], 2.0 ** -30))))


def train(layers, x: np.ndarray, y: np.ndarray, epochs: int = 8, batch: int = 4096,
          lr: float = 1e-3, seed: int = 0, threads: int | None = None):
    import torch
    if threads:
        torch.set_num_threads(threads)
    g = torch.Generator().manual_seed(seed)
    params = []
    for w, b in layers:
        params.append(torch.tensor(np.asarray(w, np.float32), requires_grad=True))
        params.append(torch.tensor(np.asarray(b, np.float32), requires_grad=True))
    opt = torch.optim.Adam(params, lr=lr)
    X = torch.from_numpy(np.ascontiguousarray(x, np.float32))
    Y = torch.from_numpy(np.ascontiguousarray(y, np.int64))
    n = X.shape[0]
    nl = len(layers)
    hist = []
    for _ in range(epochs):
        perm = torch.randperm(n, generator=g)
        tot = 0.0
        for s in range(0, n, batch):
            idx = perm[s:s + batch]
            h = X[idx]
            for i in range(nl):
                h = h @ params[2 * i] + params[2 * i + 1]
                if i < nl - 1:
                    h = torch.relu(h)
            loss = torch.nn.functional.cross_entropy(h, Y[idx]) / np.log(2.0)
            opt.zero_grad()
            loss.backward()
            opt.step()
            tot += float(loss) * len(idx)
        hist.append(tot / n)
    out = [(params[2 * i].detach().numpy().astype(np.float32).copy(),
            params[2 * i + 1].detach().numpy().astype(np.float32).copy()) for i in range(nl)]
    return out, hist
