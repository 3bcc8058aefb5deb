"""Per-step timeline of the training conv (CTA 0, thread 0): build with
debug/build_variant.sh ctl -DCT_TL, run HTB200_LIB=debug/libhtb200_ctl.so."""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
lib = _lib.load()
B = 20; H = W = 256
x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
bias = torch.randn(32, device='cuda'); o = torch.empty_like(x)
for _ in range(3):
    _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
              C.c_void_p(bias.data_ptr()), None, None, C.c_void_p(o.data_ptr()), 1, 0, None)
torch.cuda.synchronize()
buf = (C.c_longlong * (4096 * 6))()
lib.ht_debug_conv_timeline(buf)
a = np.frombuffer(buf, dtype=np.int64).reshape(4096, 6)
a = a[a[:, 1] > 0][10:-10]
stg = a[:, 0] - a[:, 4]
per = np.diff(a[:, 1])
print("steps", len(a), "period median", int(np.median(per)))
for k, name in ((2, "barrier+issue"), (3, "wait MMA(r)"), (4, "drain"), (5, "split")):
    print(f"  {name:14s} {int(np.median(a[:, k] - a[:, k - 1]))}")
print(f"  {'(stage wait+LDS)':14s} {int(np.median(stg))}")
print(f"  {'store+load':14s} {int(np.median(a[1:, 1] - a[:-1, 5]))}")
