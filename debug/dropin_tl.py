"""Host timeline of one pipelined rl.halftone call (64 x 512^2): when each
chunk's retire wait, staging and launch happen, and when the GPU finished it."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2304_12152_b200 import rl, synth  # noqa: E402
from paper_2304_12152_b200.imagecore import Rng  # noqa: E402
from paper_2304_12152_b200.nn import PolicyNetwork  # noqa: E402

net = PolicyNetwork(32, 16)
net.init_params(Rng(0), std=0.01)
B = 64
c = synth.config_batch(B, 512, 512, seed=2)
z = np.random.default_rng(1).standard_normal((B, 512, 512)).astype(np.float32)
print(c.dtype, z.dtype, torch.get_num_threads())
marks = []
orig_sync = torch.cuda.Event.synchronize
orig_hd = net.halftone_device


def ev_sync(self):
    t0 = time.perf_counter()
    orig_sync(self)
    marks.append(("wait", t0, time.perf_counter()))


def hd(*a, **k):
    t0 = time.perf_counter()
    r = orig_hd(*a, **k)
    marks.append(("launch", t0, time.perf_counter()))
    return r


torch.cuda.Event.synchronize = ev_sync
net.halftone_device = hd
for it in range(3):
    marks.clear()
    T0 = time.perf_counter()
    out = rl.halftone(net, c, z)
    T1 = time.perf_counter()
    del out
print("total %.2f ms" % ((T1 - T0) * 1e3))
for n, a, b in marks:
    print(f"{n:7s} {1e3 * (a - T0):7.2f} -> {1e3 * (b - T0):7.2f}  ({1e3 * (b - a):.2f})")
