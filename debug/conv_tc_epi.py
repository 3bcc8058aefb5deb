"""Per-launch time of the tcgen05 32->32 training conv at 20 x 256^2 for each
epilogue the training step uses (CUDA events)."""
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
B, H, W = 20, 256, 256
x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
bias = torch.randn(32, device='cuda'); o = torch.empty_like(x)
mask = torch.randn_like(x); resid = torch.randn_like(x)
p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
cases = {"relu (fwd conv1)": (bias, None, None, 1), "resid (fwd conv2)": (bias, None, resid, 0),
         "mask (bwd conv2^T)": (None, mask, None, 0), "resid (bwd conv1^T)": (None, None, resid, 0),
         "plain": (None, None, None, 0)}
res = {}
for name, (b_, m_, r_, relu) in cases.items():
    f = lambda: _lib.call("ht_conv3x3_32", p(x), B, H, W, p(w), p(b_), p(m_), p(r_), p(o), relu, 0, None)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(30): f()
    b.record(); torch.cuda.synchronize()
    res[name] = round(a.elapsed_time(b) / 30 * 1e3, 1)
print("us per launch:", res)
