"""Device RNG kernel times at config-5 sizes: 16 gaussian maps of 256^2, 1M uniforms."""
import sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200.imagecore import Rng, gaussian_maps_device
r = Rng(3)
starts = []
for i in range(16):
    starts.append(r.state_words()); r.jump(65536)
for _ in range(3):
    gaussian_maps_device(starts, 256, 256, device='cuda'); Rng(5).uniforms_device(1 << 20, device='cuda')
torch.cuda.synchronize()
a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
a.record()
for _ in range(10): gaussian_maps_device(starts, 256, 256, device='cuda')
b.record()
for _ in range(10): Rng(5).uniforms_device(1 << 20, device='cuda')
c.record(); torch.cuda.synchronize()
print(f"gaussian maps 16 x 256^2: {a.elapsed_time(b) / 10 * 1e3:.1f} us; uniforms 1M: {b.elapsed_time(c) / 10 * 1e3:.1f} us")
