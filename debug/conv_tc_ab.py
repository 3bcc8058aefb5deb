"""Per-launch time of the 32->32 training conv: tcgen05 (impl 0) vs SIMT (1),
B x 256^2.  (Used for the reverted half-channel two-CTA A/B, profile notes.)"""
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
for B in (4, 20):
    H = W = 256
    x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
    bias = torch.randn(32, device='cuda'); out = torch.empty_like(x)
    res = {}
    for impl in (0, 1):
        f = lambda: _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
                              C.c_void_p(bias.data_ptr()), None, None, C.c_void_p(out.data_ptr()), 1, impl, None)
        for _ in range(3): f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): f()
        b.record(); torch.cuda.synchronize()
        res[impl] = (a.elapsed_time(b) / 20 * 1e3, out.clone())
    print(f"B={B}: " + ", ".join(f"impl {k}: {v[0]:.1f} us" for k, v in res.items()),
          " max|tc - simt| =", (res[0][1] - res[1][1]).abs().max().item())
