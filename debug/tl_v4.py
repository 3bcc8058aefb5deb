"""Per-step timeline of the mid pass (CTA 0): HTB200_LIB=debug/libhtb200_tl.so
(built with -DHT_TIMELINE).  Events per group (warp 0 lane 0): 1 acc_full seen,
2 group barrier passed, 3 a_full seen (issue start), 4 MMAs committed, 5 step end."""
import ctypes as C, sys, numpy as np, torch
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
lib.ht_debug_timeline(buf)
net.halftone_device(c, z, h_out=h, workspace=ws); torch.cuda.synchronize()
lib.ht_debug_timeline(buf)
a = np.frombuffer(buf, dtype=np.int64).reshape(4, 16384, 4).copy()
np.save('gpurun_out/timeline_v4.npy', a)
ev = {}
for g in range(4):
    rec = a[g][a[g][:, 0] > 0]
    d = {}
    for e, t, r, clk in rec:
        d.setdefault(int(t), {})[int(e)] = int(clk)
    ev[g] = d
t0 = min(min(x.values()) for g in ev for x in ev[g].values())
def med(x): return int(np.median(x)) if len(x) else -1
for g in range(4):
    d = ev[g]; ts = sorted(d)
    per, lat, drain, afw, iss, ho = [], [], [], [], [], []
    sub = {k: [] for k in ("ld", "act", "init", "tobar")}
    for t in ts[5:-5]:
        x, y = d[t], d.get(t + 1, {})
        if 1 in x and 1 in y: per.append(y[1] - x[1])
        if 4 in x and 1 in y: lat.append(y[1] - x[4])
        if 1 in x and 2 in x: drain.append(x[2] - x[1])
        if 2 in x and 3 in x: afw.append(x[3] - x[2])
        if 3 in x and 4 in x: iss.append(x[4] - x[3])
        if 4 in x and 5 in x: ho.append(x[5] - x[4])
        if 1 in x and 6 in x: sub["ld"].append(x[6] - x[1])
        if 6 in x and 7 in x: sub["act"].append(x[7] - x[6])
        if 7 in x and 8 in x: sub["init"].append(x[8] - x[7])
        if 8 in x and 2 in x: sub["tobar"].append(x[2] - x[8])
    print(f"group {g}: steps {len(ts)} period {med(per)} | mma issue->seen {med(lat)} | seen->bar {med(drain)} "
          f"| a_full wait {med(afw)} | issue {med(iss)} | handoff {med(ho)}  [" + " ".join(f"{k} {med(v)}" for k, v in sub.items()) + "]")
# tensor-pipe view: intervals [issue start, completion seen] per group, first 40 steps
rows = []
for g in range(4):
    for t, x in ev[g].items():
        if 3 in x: rows.append((x[3] - t0, g, t, 'I'))
        if 1 in x: rows.append((x[1] - t0, g, t, 'C'))
rows.sort()
mid = len(rows) // 2
if len(sys.argv) > 2:
    for r in rows[mid:mid + 48]:
        print(r)
