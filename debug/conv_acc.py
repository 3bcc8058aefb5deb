import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_gpu_conv_tc import _conv64, _run
from paper_2304_12152_b200.imagecore import Rng
r = Rng(3)
B, H, W = 2, 24, 30
for xs, ws in ((1.0, 0.05), (1e-6, 0.05), (1e-9, 0.05)):
    x = (r.gaussians(B * 32 * H * W).reshape(B, 32, H, W) * xs).astype(np.float32).astype(np.float64)
    w = (r.gaussians(32 * 32 * 9).reshape(32, 32, 3, 3) * ws).astype(np.float32).astype(np.float64)
    ref = _conv64(x, w)
    scale = np.abs(_conv64(np.abs(x), np.abs(w))).max()
    for impl in (0, 1):
        out = _run(impl, x, w)
        e = np.abs(out - ref)
        print(f"x~{xs:g} impl {impl}: max err / scale {e.max() / scale:.2e}, rel (norm) {np.linalg.norm(out - ref) / np.linalg.norm(ref):.2e}")
