"""Per-launch time of the tcgen05 32->32 training conv with the dgrad-style
epilogue (ReLU mask + residual), 20 x 256^2 (CUDA events)."""
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
B, H, W = 20, 256, 256
x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
bias = torch.randn(32, device='cuda'); o = torch.empty_like(x)
mask = torch.randn_like(x); res = torch.randn_like(x)
res_out = []
for name, m, r in (("plain", None, None), ("mask+resid", mask, res)):
    f = lambda: _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
                          C.c_void_p(bias.data_ptr()), C.c_void_p(m.data_ptr()) if m is not None else None,
                          C.c_void_p(r.data_ptr()) if r is not None else None, C.c_void_p(o.data_ptr()), 0, 0, None)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(30): f()
    b.record(); torch.cuda.synchronize()
    res_out.append(f"{name}: {a.elapsed_time(b) / 30 * 1e3:.1f} us")
print(", ".join(res_out))
