"""One tcgen05 training conv launch pattern for ncu: impl (argv[1]) at 20 x 256^2."""
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
impl = int(sys.argv[1]) if len(sys.argv) > 1 else 0
B = 20; H = W = 256
x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
bias = torch.randn(32, device='cuda'); o = torch.empty_like(x)
for _ in range(4):
    _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
              C.c_void_p(bias.data_ptr()), None, None, C.c_void_p(o.data_ptr()), 1, impl, None)
torch.cuda.synchronize()
