"""One 20 x 256^2 training-conv launch per impl (0: conv_tc2, 2: conv_tc) after
warm-up, for ncu captures: python debug/conv_tc_one2.py [impl ...]."""
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
B = H = 0
B, H, W = 20, 256, 256
x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
bias = torch.randn(32, device='cuda'); resid = torch.randn_like(x); out = torch.empty_like(x)
for impl in [int(a) for a in sys.argv[1:]] or [0, 2]:
    for _ in range(2):
        _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
                  C.c_void_p(bias.data_ptr()), None, C.c_void_p(resid.data_ptr()), C.c_void_p(out.data_ptr()),
                  1, impl, None)
    torch.cuda.synchronize()
