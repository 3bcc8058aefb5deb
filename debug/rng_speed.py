import sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200.imagecore import Rng
for n in (262144, 4194304, 34799360):
    out = torch.empty(n, dtype=torch.float32, device='cuda')
    r = Rng(1)
    r.gaussians_device(n, out=out); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): r.gaussians_device(n, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"n={n}: {ms:.3f} ms  {n / ms / 1e6:.1f} Msamples/s")
