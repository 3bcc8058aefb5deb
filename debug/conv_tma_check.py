import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_gpu_conv_tc import _conv64, _run
from paper_2304_12152_b200.imagecore import Rng
for (B, H, W) in [(1, 4, 128), (1, 5, 256), (2, 9, 300)]:
    r = Rng(1)
    x = r.gaussians(B * 32 * H * W).reshape(B, 32, H, W).astype(np.float32).astype(np.float64)
    w = (r.gaussians(32 * 32 * 9).reshape(32, 32, 3, 3) * 0.1).astype(np.float32).astype(np.float64)
    ref = _conv64(x, w)
    out = _run(0, x, w)
    print(B, H, W, np.abs(out - ref).max() / np.abs(ref).max(), flush=True)
