"""One 20 x 256^2 weight-gradient launch (2 bf16 parts) after warm-up, for ncu."""
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
B, H, W = 20, 256, 256
x = torch.randn(B, 32, H, W, device='cuda')
d = torch.randn(B, 32, H, W, device='cuda') * 1e-2
dw = torch.zeros(9216, dtype=torch.float64, device='cuda'); db = torch.zeros(32, dtype=torch.float64, device='cuda')
for _ in range(2):
    _lib.call("ht_wgrad3x3_32", C.c_void_p(x.data_ptr()), C.c_void_p(d.data_ptr()), B, H, W,
              C.c_void_p(dw.data_ptr()), C.c_void_p(db.data_ptr()), 0, 2, None)
torch.cuda.synchronize()
