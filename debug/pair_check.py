"""conv_tc2 on CTA pairs (ht_set_conv_pair(1)) vs one CTA per strip and vs
the split-bf16 kernel: every eligible test shape and epilogue, then timing."""
import sys, ctypes as C, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
torch.manual_seed(0)
worst = 0.0
for (B, H, W) in [(1, 7, 300), (3, 9, 128), (3, 6, 132), (4, 5, 136), (2, 11, 256), (8, 3, 128), (5, 2, 252), (4, 1, 128), (1, 40, 128), (20, 256, 256)]:
    for mode in ("plain", "mask", "resid"):
        x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.1
        bias = torch.randn(32, device='cuda'); e = torch.randn_like(x)
        m = C.c_void_p(e.data_ptr()) if mode == "mask" else None
        r = C.c_void_p(e.data_ptr()) if mode == "resid" else None
        outs = []
        for pair, impl in ((1, 3), (0, 3), (0, 2)):
            _lib.call("ht_set_conv_pair", pair)
            out = torch.empty_like(x)
            _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
                      C.c_void_p(bias.data_ptr()), m, r, C.c_void_p(out.data_ptr()), 1, impl, None)
            torch.cuda.synchronize()
            outs.append(out)
        d_pair = (outs[0] - outs[1]).abs().max().item()
        d_ref = (outs[0] - outs[2]).abs().max().item()
        worst = max(worst, d_ref)
        print(B, H, W, mode, "pair vs single", d_pair, "pair vs split-bf16", d_ref, flush=True)
print("worst", worst)
B, H, W = 20, 256, 256
x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
bias = torch.randn(32, device='cuda'); e = torch.randn_like(x); out = torch.empty_like(x)
for mode in ("plain", "resid"):
    r = C.c_void_p(e.data_ptr()) if mode == "resid" else None
    for rep in range(2):
        for pair in (0, 1):
            _lib.call("ht_set_conv_pair", pair)
            f = lambda: _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
                                  C.c_void_p(bias.data_ptr()), None, r, C.c_void_p(out.data_ptr()), 1, 3, None)
            for _ in range(3): f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(30): f()
            b.record(); torch.cuda.synchronize()
            print(mode, "pair", pair, f"{a.elapsed_time(b) / 30 * 1e3:.1f} us")
_lib.call("ht_set_conv_pair", 0)
