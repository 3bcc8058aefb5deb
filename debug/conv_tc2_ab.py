"""Per-launch time of the 32->32 training conv, impl 0 (conv_tc2: scaled fp16
pairs, role-split warps) vs impl 2 (conv_tc: split bf16), B x 256^2, plus
max |difference| between them (CUDA events, interleaved)."""
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
for B in (4, 20):
    H = W = 256
    x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
    bias = torch.randn(32, device='cuda'); resid = torch.randn_like(x)
    outs = {}
    for mode in ("plain", "resid"):
        res = {}
        for rep in range(3):
            for impl in (3, 2):
                out = torch.empty_like(x)
                rp = resid if mode == "resid" else None
                f = lambda: _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
                                      C.c_void_p(bias.data_ptr()), None, None if rp is None else C.c_void_p(rp.data_ptr()),
                                      C.c_void_p(out.data_ptr()), 1, impl, None)
                for _ in range(3): f()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(30): f()
                b.record(); torch.cuda.synchronize()
                res.setdefault(impl, []).append(a.elapsed_time(b) / 30 * 1e3)
                outs[impl] = out
        d = (outs[3] - outs[2]).abs().max().item()
        print(f"B={B} {mode}: " + ", ".join(f"impl {k}: {min(v):.1f} us" for k, v in res.items()), f"max|d|={d:.2e}")
