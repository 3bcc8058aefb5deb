import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import rl
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import PolicyNetwork
net = PolicyNetwork(32, int(sys.argv[1]) if len(sys.argv) > 1 else 16)
net.init_params(Rng(0), std=0.05)
H = W = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = np.full((H, W), 0.5); z = np.zeros((H, W))
h, p = rl.halftone(net, c, z)
print("ok", p.mean())
