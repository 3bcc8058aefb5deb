"""Per-launch time of the 32->32 weight gradient: tcgen05 (2 / 3 bf16 parts) vs SIMT, 20 x 256^2."""
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
B, H, W = 20, 256, 256
x = torch.randn(B, 32, H, W, device='cuda')
d = torch.randn(B, 32, H, W, device='cuda') * 1e-2
dw = torch.zeros(9216, dtype=torch.float64, device='cuda'); db = torch.zeros(32, dtype=torch.float64, device='cuda')
def run(impl, parts):
    _lib.call("ht_wgrad3x3_32", C.c_void_p(x.data_ptr()), C.c_void_p(d.data_ptr()), B, H, W,
              C.c_void_p(dw.data_ptr()), C.c_void_p(db.data_ptr()), impl, parts, None)
for impl, parts in ((0, 2), (0, 3), (1, 3)):
    for _ in range(3): run(impl, parts)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    a.record()
    for _ in range(n): run(impl, parts)
    b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) / n * 1e3
    fl = 2 * B * H * W * 32 * 288
    print(f"impl {impl} parts {parts}: {us:.1f} us/launch  ({fl / us / 1e6:.1f} TFLOP/s useful fp32-equivalent)")
