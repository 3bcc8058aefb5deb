"""Per-launch time of conv_tc2 (impl 0), 20 x 256^2 plain, for the library in HTB200_LIB."""
import ctypes as C, sys, torch, os
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
B = H = W = 0
B, H, W = 20, 256, 256
x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
bias = torch.randn(32, device='cuda'); out = torch.empty_like(x); res = torch.randn_like(x)
rp = C.c_void_p(res.data_ptr()) if "resid" in sys.argv else None
f = lambda: _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
                      C.c_void_p(bias.data_ptr()), None, rp, C.c_void_p(out.data_ptr()), 1, 3, None)
for _ in range(3): f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(30): f()
b.record(); torch.cuda.synchronize()
print(os.environ.get("HTB200_LIB", "base"), sys.argv[1:], f"{a.elapsed_time(b) / 30 * 1e3:.1f} us")
