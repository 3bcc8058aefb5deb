"""conv_tc2 with a residual input, 20 x 256^2, per-launch time for the library in HTB200_LIB (+ max |diff| vs conv_tc)."""
import ctypes as C, sys, os, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
B, H, W = 20, 256, 256
torch.manual_seed(0)
x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
bias = torch.randn(32, device='cuda'); e = torch.randn_like(x)
res = {}
for mode in ("resid", "mask"):
    m = C.c_void_p(e.data_ptr()) if mode == "mask" else None
    r = C.c_void_p(e.data_ptr()) if mode == "resid" else None
    outs = {}
    for impl in (3, 2):
        out = torch.empty_like(x)
        f = lambda: _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
                              C.c_void_p(bias.data_ptr()), m, r, C.c_void_p(out.data_ptr()), 1, impl, None)
        for _ in range(3): f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(30): f()
        b.record(); torch.cuda.synchronize()
        res[(mode, impl)] = a.elapsed_time(b) / 30 * 1e3
        outs[impl] = out
    res[(mode, 'd')] = (outs[3] - outs[2]).abs().max().item()
print(os.environ.get("HTB200_LIB", "base"), {k: round(v, 2) if isinstance(v, float) and v > 1e-3 else v for k, v in res.items()})
