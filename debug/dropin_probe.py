"""Host-side costs of the drop-in rl.halftone pipeline (one chunk = 8 x 512^2):
numpy -> pinned staging copy, pinned H2D, pageable H2D, float64 D2H."""
import time

import numpy as np
import torch

m, H, W = 8, 512, 512
a = np.random.default_rng(0).random((m, H, W), dtype=np.float32)
a64 = a.astype(np.float64)
st = torch.empty((m, H, W), dtype=torch.float32, pin_memory=True)
d = torch.empty((m, H, W), dtype=torch.float32, device="cuda")
o64 = torch.empty((m, H, W), dtype=torch.float64, device="cuda")
h64 = torch.empty((m, H, W), dtype=torch.float64, pin_memory=True)
print("torch threads", torch.get_num_threads())


def t(f, n=20):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print("stage f32 -> pinned  %.3f ms" % t(lambda: st.copy_(torch.from_numpy(a))))
print("stage f64 -> pinned  %.3f ms" % t(lambda: st.copy_(torch.from_numpy(a64))))
print("np.copyto f32        %.3f ms" % t(lambda: np.copyto(st.numpy(), a)))
print("H2D pinned           %.3f ms" % t(lambda: d.copy_(st, non_blocking=True)))
print("H2D pageable         %.3f ms" % t(lambda: d.copy_(torch.from_numpy(a), non_blocking=True)))
print("D2H f64 pinned       %.3f ms" % t(lambda: h64.copy_(o64, non_blocking=True)))
for nt in (4, 8, 16):
    torch.set_num_threads(nt)
    print(f"stage f32 threads={nt}  %.3f ms" % t(lambda: st.copy_(torch.from_numpy(a))))

# the whole drop-in call at config-2 size for several chunk counts
import sys
sys.path.insert(0, '.')
from paper_2304_12152_b200 import rl, synth  # noqa: E402
from paper_2304_12152_b200.imagecore import Rng  # noqa: E402
from paper_2304_12152_b200.nn import PolicyNetwork  # noqa: E402
torch.set_num_threads(8)
net = PolicyNetwork(32, 16)
net.init_params(Rng(0), std=0.01)
B = 64
c = synth.config_batch(B, 512, 512, seed=2)
z = np.random.default_rng(1).standard_normal((B, 512, 512)).astype(np.float32)
cd, zd = torch.from_numpy(c).cuda(), torch.from_numpy(z).cuda()
hdev = torch.empty((B, 512, 512), dtype=torch.uint8, device="cuda")
ws = net.halftone_device(cd, zd, h_out=hdev)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    net.halftone_device(cd, zd, h_out=hdev, workspace=ws)
e1.record()
torch.cuda.synchronize()
print("device-only %.2f ms" % (e0.elapsed_time(e1) / 3))
for ch in (4, 8, 16, 32):
    rl._PIPE_CHUNKS = ch
    out = rl.halftone(net, c, z)
    del out
    t0 = time.perf_counter()
    for _ in range(3):
        out = rl.halftone(net, c, z)
        del out
    print(f"chunks={ch}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms per call")
t0 = time.perf_counter()
x = torch.empty((B, 512, 512), dtype=torch.float64, pin_memory=True)
print("pinned alloc %.2f ms" % ((time.perf_counter() - t0) * 1e3))
