"""Config-1 style latency (one image, device-resident, L2 flushed) for a
library build: python debug/latency_sweep.py [size ...]"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import synth
from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_device
from paper_2304_12152_b200.nn import PolicyNetwork
net = PolicyNetwork(32, 16); net.init_params(Rng(0), std=0.01)
flush = torch.empty(64 << 20, dtype=torch.float32, device='cuda')
out = {}
for S in [int(x) for x in sys.argv[1:]] or [64, 128, 256, 512]:
    c = torch.from_numpy(synth.contone(S, S, seed=0)).cuda()[None]
    z = gaussian_noise_map_device(Rng(0), S, S, device='cuda')[None]
    h = torch.empty((1, S, S), dtype=torch.uint8, device='cuda')
    ws = net.halftone_device(c, z, h_out=h, check=True)
    ts = []
    for _ in range(23):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); net.halftone_device(c, z, h_out=h, workspace=ws); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    out[S] = round(float(np.median(ts[3:])), 4)
print("latency_ms", out)
