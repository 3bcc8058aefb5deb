"""Device-resident K1 throughput vs batch size (config-2 images), CUDA events:
what one rank sees when config 2's 64 images are split over N GPUs."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import synth
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import PolicyNetwork
net = PolicyNetwork(32, 16); net.init_params(Rng(0), std=0.01)
for B in [int(x) for x in sys.argv[1:]] or [8, 16, 32, 64]:
    c = torch.from_numpy(synth.config_batch(B, 512, 512, seed=2)).cuda()
    z = torch.randn(B, 512, 512, device='cuda')
    h = torch.empty((B, 512, 512), dtype=torch.uint8, device='cuda')
    ws = net.halftone_device(c, z, h_out=h)
    for _ in range(3): net.halftone_device(c, z, h_out=h, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): net.halftone_device(c, z, h_out=h, workspace=ws)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"B={B:3d}: {ms:7.3f} ms/step  {B * 512 * 512 / ms / 1e3:8.1f} Mpx/s")
