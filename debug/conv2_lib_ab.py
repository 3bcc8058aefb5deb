"""A/B of conv_tc2 builds: per-launch time (CUDA events, 30 back-to-back
launches, 20 x 256^2) plain and with a residual, plus an output checksum,
each library in its own subprocess, alternating.
    python debug/conv2_lib_ab.py libA.so libB.so [--reps 3]"""
import json, os, subprocess, sys
CHILD = r'''
import ctypes as C, hashlib, sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
B = H = W = 0; B, H, W = 20, 256, 256
g = torch.Generator(device='cuda'); g.manual_seed(1)
x = torch.randn(B, 32, H, W, device='cuda', generator=g); w = torch.randn(32, 32, 3, 3, device='cuda', generator=g) * 0.05
bias = torch.randn(32, device='cuda', generator=g); resid = torch.randn(B, 32, H, W, device='cuda', generator=g)
res = {}
h = hashlib.sha1()
for mode in ("plain", "resid"):
    out = torch.empty_like(x)
    rp = resid if mode == "resid" else None
    f = lambda: _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
                          C.c_void_p(bias.data_ptr()), None, None if rp is None else C.c_void_p(rp.data_ptr()),
                          C.c_void_p(out.data_ptr()), 1, 0, None)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(30): f()
    b.record(); torch.cuda.synchronize()
    res[mode] = round(a.elapsed_time(b) / 30 * 1e3, 1)
    h.update(out.cpu().numpy().tobytes())
res["sum"] = h.hexdigest()[:12]
print(res)
'''
libs = [a for a in sys.argv[1:] if a.endswith('.so')]
reps = int(sys.argv[sys.argv.index('--reps') + 1]) if '--reps' in sys.argv else 3
for _ in range(reps):
    for l in libs:
        pr = subprocess.run([sys.executable, '-c', CHILD], capture_output=True, text=True,
                            env={**os.environ, 'HTB200_LIB': l}, timeout=300)
        print(os.path.basename(l), pr.stdout.strip().splitlines()[-1] if pr.returncode == 0 else pr.stderr[-500:])
