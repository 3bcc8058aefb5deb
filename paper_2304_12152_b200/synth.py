"""Seeded synthetic contones standing in for the paper's datasets.

BASELINE.json's configs describe the images only by recipe: "a linear ramp
plus N random Gaussian blobs (sigma 8-40 px, amplitude +-0.4) plus M flat
constant rectangles, clipped to [0,1]" (config 2 adds uniform-random step
edges to 10% of the images).  The paper's own images (VOC2012, DIV2K,
"Lenna") are not available, so this generator -- frozen here, seeded per
config -- produces every contone the tests and bench.py use.  It is host-side
input preparation and is never timed.
"""

import numpy as np


def contone(height, width, seed=0, blobs=8, rects=2, step_edge=False):
    """float32 (height, width) contone in [0, 1]."""
    rng = np.random.default_rng(seed)
    ang = rng.uniform(0.0, 2.0 * np.pi)
    lo, hi = rng.uniform(0.0, 0.3), rng.uniform(0.7, 1.0)
    yy = np.arange(height, dtype=np.float64)[:, None]
    xx = np.arange(width, dtype=np.float64)[None, :]
    # linear ramp along a random direction, spanning [lo, hi]
    proj = np.cos(ang) * xx / max(width - 1, 1) + np.sin(ang) * yy / max(height - 1, 1)
    proj = (proj - proj.min()) / max(proj.max() - proj.min(), 1e-12)
    img = lo + (hi - lo) * proj
    for _ in range(blobs):
        cy, cx = rng.uniform(0, height), rng.uniform(0, width)
        sig = rng.uniform(8.0, 40.0)
        amp = rng.uniform(-0.4, 0.4)
        r = int(np.ceil(4.0 * sig))
        y0, y1 = max(0, int(cy) - r), min(height, int(cy) + r + 1)
        x0, x1 = max(0, int(cx) - r), min(width, int(cx) + r + 1)
        if y0 >= y1 or x0 >= x1:
            continue
        gy = np.exp(-((np.arange(y0, y1) - cy) ** 2) / (2 * sig * sig))
        gx = np.exp(-((np.arange(x0, x1) - cx) ** 2) / (2 * sig * sig))
        img[y0:y1, x0:x1] += amp * gy[:, None] * gx[None, :]
    for _ in range(rects):
        rh = int(rng.uniform(0.05, 0.3) * height) + 1
        rw = int(rng.uniform(0.05, 0.3) * width) + 1
        y0 = int(rng.integers(0, max(height - rh, 0) + 1))
        x0 = int(rng.integers(0, max(width - rw, 0) + 1))
        img[y0:y0 + rh, x0:x0 + rw] = rng.uniform(0.0, 1.0)
    if step_edge:
        # a straight step edge between two uniform-random tones
        a, b = rng.uniform(0.0, 1.0, size=2)
        t = rng.uniform(0.0, np.pi)
        off = rng.uniform(-0.3, 0.3)
        side = (np.cos(t) * (xx / width - 0.5) + np.sin(t) * (yy / height - 0.5)) > off
        img = np.where(side, a, b) * 0.5 + img * 0.5
    return np.clip(img, 0.0, 1.0).astype(np.float32)


def config_batch(n, height, width, seed=0, blobs=8, rects=2, step_frac=0.0):
    """n contones (n, height, width); image i uses seed (seed, i)."""
    out = np.empty((n, height, width), dtype=np.float32)
    n_step = int(round(step_frac * n))
    for i in range(n):
        out[i] = contone(height, width, seed=seed * 1_000_003 + i, blobs=blobs,
                         rects=rects, step_edge=i < n_step)
    return out
