import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib, synth
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import PolicyNetwork
lib = _lib.load()
B = 16
net = PolicyNetwork(32, int(sys.argv[1]) if len(sys.argv) > 1 else 16); net.init_params(Rng(0), std=0.01)
c = torch.from_numpy(synth.config_batch(B, 512, 512, seed=2)).cuda()
z = torch.randn(B, 512, 512, device='cuda')
h = torch.empty((B, 512, 512), dtype=torch.uint8, device='cuda')
ws = net.halftone_device(c, z, h_out=h); torch.cuda.synchronize()
buf = (C.c_longlong * 128)()
# profile the mid pass: run a net whose LAST pass is a mid pass is not possible,
# so run NB=16 and read (the last writer is the output pass); then NB such that..
lib.ht_debug_prof(buf)
# v4 step order: 0 loop top, 1 acc_full wait, 2 tmem ld, 3 act+link+pack+init,
# 4 layer-0 loader, 6 st-wait+named bar, 7 a_full wait, 8 mma issue, 9 pre-hand-off,
# 10 a_empty wait, 11 sts, 12 fence.proxy, 13 arrive, 5 tail (global store)
names = ["loop", "acc_full wait", "tmem ld", "act/link/init", "loader", "tail/gstore", "group bar", "a_full wait", "mma issue", "pre-handoff", "a_empty wait", "sts", "fence.proxy", "arrive", "act", "link_empty wait"]
for g in range(4):
    for w in range(2):
        v = list(buf)[16 * (2 * g + w):16 * (2 * g + w) + 16]
        tot = sum(v)
        if not tot: continue
        steps = int(sys.argv[2]) if len(sys.argv) > 2 else 0
        print("group", g, "warp", w, "total", tot, " ".join(f"{n}={100*x/tot:.1f}%" for n, x in zip(names, v) if x))
