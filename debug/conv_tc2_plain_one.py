"""One plain 20 x 256^2 conv_tc2 launch (bias + ReLU, no epilogue input)
after warm-up, for an ncu --set full capture."""
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
B, H, W = 20, 256, 256
x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
bias = torch.randn(32, device='cuda'); out = torch.empty_like(x)
for _ in range(3):
    _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
              C.c_void_p(bias.data_ptr()), None, None, C.c_void_p(out.data_ptr()), 1, 0, None)
torch.cuda.synchronize()
