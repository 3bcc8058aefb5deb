"""Checksum of K1's p and h for a fixed 8 x 512^2 batch, to confirm that a
timing variant of the library (HTB200_LIB=...) computes the same bits."""
import hashlib, sys, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import synth
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import PolicyNetwork
net = PolicyNetwork(32, 16); net.init_params(Rng(0), std=0.05)
c = torch.from_numpy(synth.config_batch(8, 512, 512, seed=2)).cuda()
g = torch.Generator(device='cuda'); g.manual_seed(5)
z = torch.randn(8, 512, 512, device='cuda', generator=g)
h = torch.empty((8, 512, 512), dtype=torch.uint8, device='cuda')
p = torch.empty((8, 512, 512), dtype=torch.float32, device='cuda')
net.halftone_device(c, z, h_out=h, p_out=p)
torch.cuda.synchronize()
print(hashlib.sha1(p.cpu().numpy().tobytes() + h.cpu().numpy().tobytes()).hexdigest()[:16])
