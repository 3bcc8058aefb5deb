"""Device RNG launches at training-step sizes: 20 noise maps of 256^2 from
recorded stream states (gaussian_maps_device) and 16 x 256^2 uniforms."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200 import imagecore
r = Rng(1)
n = 256 * 256
states = []
for m in range(20):
    states.append(r.state_words()); r.uniforms(3)
u = torch.empty(16 * n, dtype=torch.float64, device='cuda')
def maps(): imagecore.gaussian_maps_device(states, 256, 256, dtype=torch.float32)
def unif(): Rng(2).uniforms_device(16 * n, out=u)
for f, name in ((maps, "20 gaussian maps of 256^2"), (unif, "16 x 256^2 uniforms")):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
