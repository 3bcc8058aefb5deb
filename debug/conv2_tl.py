"""Clock64 timeline of conv_tc2 CTA 0 (build: debug/build_variant.sh tl2 -DCT2_TL;
run: HTB200_LIB=debug/libhtb200_tl2.so python debug/conv2_tl.py [B] [resid])."""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
B = int(sys.argv[1]) if len(sys.argv) > 1 else 20
use_res = len(sys.argv) > 2
H = W = 256
x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
bias = torch.randn(32, device='cuda'); resid = torch.randn_like(x); out = torch.empty_like(x)
lib = _lib.load()
import os
if os.environ.get("PAIR"): _lib.call("ht_set_conv_pair", 1)
buf = np.zeros((3, 1024, 6), np.int64)
for it in range(3):
    _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()), C.c_void_p(bias.data_ptr()),
              None, C.c_void_p(resid.data_ptr()) if use_res else None, C.c_void_p(out.data_ptr()), 1, 0, None)
    torch.cuda.synchronize()
lib.ht_debug_conv2_timeline(buf.ctypes.data_as(C.c_void_p))
t0 = buf[buf > 0].min()
n = int((buf[0, :, 4] > 0).sum())
print("rows", n, "total cycles", buf[0, n - 1, 4] - t0)
I, Sp, D = buf[0, :n] - t0, buf[1, :n] - t0, buf[2, :n] - t0
med = lambda a: int(np.median(a))
print("issuer: wait ready", med(I[:, 1] - I[:, 0]), " tma", med(I[:, 2] - I[:, 1]), " wait ring", med(I[:, 3] - I[:, 2]),
      " mma issue", med(I[:, 4] - I[:, 3]), " period", med(np.diff(I[:, 4])))
print("splitter: wait stg", med(Sp[:, 1] - Sp[:, 0]), " ld+max+bar", med(Sp[:, 2] - Sp[:, 1]), " wait Abuf", med(Sp[:, 3] - Sp[:, 2]),
      " split+st+fence", med(Sp[:, 4] - Sp[:, 3]), " period", med(np.diff(Sp[:, 4])))
dv = D[D[:, 4] > 0]
print("drainer: wait mma", med(dv[:, 1] - dv[:, 0]), " tmem ld", med(dv[:, 5] - dv[:, 1]), " ld+release", med(dv[:, 2] - dv[:, 1]), " epi+st", med(dv[:, 3] - dv[:, 2]),
      " load_epi", med(dv[:, 4] - dv[:, 3]), " period", med(np.diff(dv[:, 4])))
for g in range(0, min(n, 12)):
    print(g, "I", I[g, [0, 1, 3, 4]], "S", Sp[g, [0, 1, 4]], "D", D[g, [0, 1, 4]])
