"""Timeline of CTA 0 of the wgrad kernel (build with -DWG_TL): per-tile gaps."""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
lib = _lib.load()
B, H, W = 20, 256, 256
x = torch.randn(B, 32, H, W, device='cuda'); d = torch.randn(B, 32, H, W, device='cuda') * 1e-2
dw = torch.zeros(9216, dtype=torch.float64, device='cuda'); db = torch.zeros(32, dtype=torch.float64, device='cuda')
parts = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for _ in range(3):
    _lib.call("ht_wgrad3x3_32", C.c_void_p(x.data_ptr()), C.c_void_p(d.data_ptr()), B, H, W,
              C.c_void_p(dw.data_ptr()), C.c_void_p(db.data_ptr()), 0, parts, None)
torch.cuda.synchronize()
from cuda.bindings import runtime as rt
libc = C.CDLL(_lib.LIB_PATH)
f = libc.ht_debug_wtl_ptr
f.restype = C.c_void_p
p = f()
t = torch.empty(10 * 1024 * 4, dtype=torch.int64, device='cuda')
rt.cudaMemcpy(t.data_ptr(), p, 10 * 1024 * 4 * 8, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
a = t.cpu().numpy().reshape(10, 1024, 4)
m = a[8]; n = int((m[:, 3] > 0).sum())
base = m[0, 0]
print("MMA warp: tiles", n)
iss = m[:n, 3] - base
wait_full = m[:n, 3] - m[:n, 1]
print(" issue-to-issue cycles: mean %.0f median %.0f" % (np.diff(iss).mean(), np.median(np.diff(iss))))
print(" wait (d_empty) mean %.0f, wait(full)+issue mean %.0f" % ((m[:n, 1] - m[:n, 0]).mean(), wait_full.mean()))
c = a[0]; k = int((c[:, 3] > 0).sum())
print(f"converters (warp 0): wait raw {np.mean(c[:k,2]-c[:k,0]):.0f}, then op_free {np.mean(c[:k,1]-c[:k,2]):.0f}")
print(f"converters (warp 0): tiles {k}  wait(raw+op) {np.mean(c[:k,1]-c[:k,0]):.0f}  convert {np.mean(c[:k,3]-c[:k,1]):.0f}  "
      f"period {np.mean(np.diff(c[:k,0])):.0f}")
fl = a[9]; k = int((fl[:, 3] > 0).sum())
print(f"flushers: chains {k} wait {np.mean(fl[:k,1]-fl[:k,0]):.0f} flush {np.mean(fl[:k,3]-fl[:k,1]):.0f}")
print("first MMA tiles (issue time rel):", iss[:12])
