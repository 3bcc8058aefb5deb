"""reward_le kernel time inside a config-5 step (torch profiler, 3 steps)."""
import sys, collections, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import rl, synth
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import Adam, PolicyNetwork
from torch.profiler import profile, ProfilerActivity
cfg = rl.TrainConfig(iterations=1000, batch_size=16, crop_size=256, anisotropy_batch_size=4, hvs_model="gaussian")
ds = [synth.contone(384, 384, seed=100 + i).astype(np.float64) for i in range(8)]
rng = Rng(0); net = PolicyNetwork(32, 16); net.init_params(rng); adam = Adam(net.params())
for t in range(3): rl.train_step(net, adam, ds, cfg, rng, t)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for t in range(3): rl.train_step(net, adam, ds, cfg, rng, 3 + t)
    torch.cuda.synchronize()
tot = collections.defaultdict(float)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and 'reward' in e.name:
        tot[e.name[:40]] += (e.time_range.end - e.time_range.start) / 3
print({k: round(v, 1) for k, v in tot.items()})
