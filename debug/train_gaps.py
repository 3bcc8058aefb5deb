"""GPU idle gaps inside config-5 train steps (torch profiler kernel events):
total idle per step and the largest gaps with the kernels around them."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import rl, synth
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import Adam, PolicyNetwork
from torch.profiler import profile, ProfilerActivity
cfg = rl.TrainConfig(iterations=1000, batch_size=16, crop_size=256, anisotropy_batch_size=4, hvs_model="gaussian")
ds = [synth.contone(384, 384, seed=100 + i).astype(np.float64) for i in range(8)]
rng = Rng(0); net = PolicyNetwork(32, 16); net.init_params(rng); adam = Adam(net.params())
import gc, os
if os.environ.get("NOGC"): gc.disable()
for t in range(4): rl.train_step(net, adam, ds, cfg, rng, t)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for t in range(3): rl.train_step(net, adam, ds, cfg, rng, 4 + t)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name[:50]) for e in ev)
# merge intervals across streams
busy, gaps = [], []
cur_s, cur_e, last_name = iv[0][0], iv[0][1], iv[0][2]
for s, e, n in iv[1:]:
    if s > cur_e:
        gaps.append((s - cur_e, last_name, n))
        busy.append((cur_s, cur_e)); cur_s = s
    if e >= cur_e:
        cur_e, last_name = e, n
busy.append((cur_s, cur_e))
span = iv[-1][1] - iv[0][0]
idle = sum(g[0] for g in gaps)
print(f"span {span / 3 / 1e3:.2f} ms/step, busy {(span - idle) / 3 / 1e3:.2f}, idle {idle / 3 / 1e3:.2f} ms/step, gaps>20us: {sum(1 for g in gaps if g[0] > 20) / 3:.0f}/step")
for g in sorted(gaps, reverse=True)[:12]:
    print(f"{g[0]:8.1f} us after {g[1]!r} before {g[2]!r}")
import collections
tot = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    tot[e.name[:70]][0] += 1; tot[e.name[:70]][1] += e.time_range.end - e.time_range.start
for k, (n, tt) in sorted(tot.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{tt / 3 / 1e3:7.3f} ms/step {n / 3:6.1f}  {k}")
