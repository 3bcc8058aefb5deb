import ctypes as C, sys, numpy as np, torch, json
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib, synth
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import PolicyNetwork
lib = _lib.load()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
net = PolicyNetwork(32, 16); net.init_params(Rng(0), std=0.01)
c = torch.from_numpy(synth.config_batch(B, 512, 512, seed=2)).cuda()
z = torch.randn(B, 512, 512, device='cuda')
h = torch.empty((B, 512, 512), dtype=torch.uint8, device='cuda')
ws = net.halftone_device(c, z, h_out=h); torch.cuda.synchronize()
buf = (C.c_longlong * (4 * 4 * 16384))()
lib.ht_debug_timeline.restype = C.c_int
# run only the first two passes' worth by timing a full call; the buffer keeps the
# LAST pass that wrote each slot, so record per pass by calling with timing off
lib.ht_debug_timeline(buf)  # clear
net.halftone_device(c, z, h_out=h, workspace=ws); torch.cuda.synchronize()
lib.ht_debug_timeline(buf)
a = np.frombuffer(buf, dtype=np.int64).reshape(4, 16384, 4)
np.save('gpurun_out/timeline.npy', a)
print('saved')
