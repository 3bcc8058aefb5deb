"""Per-kernel GPU time of one config-5 rl.train_step (torch profiler / CUPTI, 3 steps averaged)."""
import sys, collections, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import rl, synth
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import Adam, PolicyNetwork
cfg = rl.TrainConfig(iterations=1000, batch_size=16, crop_size=256, anisotropy_batch_size=4, hvs_model="gaussian")
ds = [synth.contone(384, 384, seed=100 + i).astype(np.float64) for i in range(8)]
rng = Rng(0); net = PolicyNetwork(32, 16); net.init_params(rng); adam = Adam(net.params())
for t in range(3): rl.train_step(net, adam, ds, cfg, rng, t)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for t in range(3): rl.train_step(net, adam, ds, cfg, rng, 3 + t)
    torch.cuda.synchronize()
tot = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name[:70]
        tot[k][0] += 1; tot[k][1] += e.device_time_total if hasattr(e, 'device_time_total') else e.cuda_time_total
s = sum(v[1] for v in tot.values())
print(f"GPU time per step: {s / 3 / 1e3:.2f} ms")
for k, (n, t) in sorted(tot.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{t / 3 / 1e3:8.3f} ms/step {n // 3:5d} launches  {k}")
