"""Timeline of the K1 mid pass (CTA 0), v4 group roles.

Build:  debug/build_variant.sh tl -DHT_TIMELINE
Run:    HTB200_LIB=debug/libhtb200_tl.so python debug/tl4.py [B]
Per group j (warp 0, lane 0) and step t the kernel records (TLG in fwd_tc.cu):
  1 acc_full observed, 6 drain done, 8 slot re-init done, 2 group barrier
  passed, 3 a_full observed, 4 MMA batch issued, 5 end of step.
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib, synth  # noqa: E402
from paper_2304_12152_b200.imagecore import Rng  # noqa: E402
from paper_2304_12152_b200.nn import PolicyNetwork  # noqa: E402

lib = _lib.load()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
net = PolicyNetwork(32, 16)
net.init_params(Rng(0), std=0.01)
c = torch.from_numpy(synth.config_batch(B, 512, 512, seed=2)).cuda()
z = torch.randn(B, 512, 512, device='cuda')
h = torch.empty((B, 512, 512), dtype=torch.uint8, device='cuda')
for _ in range(2):
    net.halftone_device(c, z, h_out=h)
torch.cuda.synchronize()
buf = (C.c_longlong * (4 * 4 * 16384))()
lib.ht_debug_timeline(buf)
net.halftone_device(c, z, h_out=h)
torch.cuda.synchronize()
lib.ht_debug_timeline(buf)
a = np.frombuffer(buf, dtype=np.int64).reshape(4, 16384, 4)
np.save('gpurun_out/tl4.npy', a)

EV = {1: 'accf', 6: 'drain', 8: 'init', 2: 'bar', 3: 'afull', 9: 'desc', 4: 'issue', 5: 'end'}
rec = {}
for j in range(4):
    last = None
    for ev, t, jj, clk in a[j]:
        if clk == 0 or (last is not None and t < last - 5):   # first segment only
            break
        last = t
        rec[(j, int(t), int(ev))] = int(clk)
ts = sorted({t for (_, t, _) in rec})
mid = ts[len(ts) // 3: len(ts) // 3 + 6]
for t in mid:
    base = rec.get((0, t, 1)) or min(v for (j, tt, e), v in rec.items() if tt == t)
    print(f"t={t}")
    for j in range(4):
        row = ' '.join(f"{EV[e]}={rec[(j, t, e)] - base:+6d}" for e in (1, 6, 8, 2, 3, 9, 4, 5) if (j, t, e) in rec)
        print(f"   j{j}: {row}")
# period and per-phase medians over the middle third
lo, hi = ts[len(ts) // 3], ts[2 * len(ts) // 3]
for j in range(4):
    steps = [t for t in ts if lo <= t < hi and (j, t, 1) in rec and (j, t + 1, 1) in rec]
    per = np.median([rec[(j, t + 1, 1)] - rec[(j, t, 1)] for t in steps])
    ph = {}
    order = tuple(e for e in (1, 6, 8, 2, 3, 9, 4, 5) if any(k[2] == e for k in rec))
    for t in steps:
        for e0, e1 in zip(order, order[1:]):
            if (j, t, e0) in rec and (j, t, e1) in rec:
                ph.setdefault(f"{EV[e0]}->{EV[e1]}", []).append(rec[(j, t, e1)] - rec[(j, t, e0)])
        if (j, t, 5) in rec:
            ph.setdefault("end->next accf", []).append(rec[(j, t + 1, 1)] - rec[(j, t, 5)])
        if (j, t, 4) in rec:
            ph.setdefault("issue->next accf (MMA latency seen)", []).append(rec[(j, t + 1, 1)] - rec[(j, t, 4)])
    print(f"j{j}: period {per:.0f} clk;", ', '.join(f"{k} {np.median(v):.0f}" for k, v in ph.items()))
# issue order within a step: which layer's batch goes first
first = {}
for t in ts[len(ts) // 3: 2 * len(ts) // 3]:
    iss = [(rec[(j, t, 4)], j) for j in range(4) if (j, t, 4) in rec]
    if len(iss) == 4:
        order = ''.join(str(j) for _, j in sorted(iss))
        first[order] = first.get(order, 0) + 1
print('issue orders:', sorted(first.items(), key=lambda kv: -kv[1])[:6])
