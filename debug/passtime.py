import ctypes as C, os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib, synth
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import PolicyNetwork
lib = _lib.load()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
NB = int(os.environ.get("HT_NB", "16"))
net = PolicyNetwork(32, NB); net.init_params(Rng(0), std=0.01)
c = torch.from_numpy(synth.config_batch(B, 512, 512, seed=2)).cuda()
z = torch.randn(B, 512, 512, device='cuda')
h = torch.empty((B, 512, 512), dtype=torch.uint8, device='cuda')
ws = net.halftone_device(c, z, h_out=h)
for _ in range(3): net.halftone_device(c, z, h_out=h, workspace=ws)
torch.cuda.synchronize()
_lib.call("ht_timing_enable", 1)
for _ in range(5): net.halftone_device(c, z, h_out=h, workspace=ws)
torch.cuda.synchronize()
_lib.call("ht_timing_enable", 0)
tags = (C.c_int * 256)(); ms = (C.c_float * 256)(); n = C.c_int(0)
_lib.call("ht_timing_read", tags, ms, 256, C.byref(n))
d = {}
for i in range(n.value): d.setdefault(tags[i], []).append(ms[i])
print(sys.argv[2] if len(sys.argv) > 2 else '', {k: round(float(np.mean(v)), 4) for k, v in sorted(d.items())})
