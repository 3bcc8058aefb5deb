"""Config-5 train_step wall time with and without next-step prefetch (same process)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import rl, synth
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import Adam, PolicyNetwork
cfg = rl.TrainConfig(iterations=1000, batch_size=16, crop_size=256, anisotropy_batch_size=4, hvs_model="gaussian")
ds = [synth.contone(384, 384, seed=100 + i).astype(np.float64) for i in range(8)]
rng = Rng(0); net = PolicyNetwork(32, 16); net.init_params(rng); adam = Adam(net.params())
hits = [0]
orig = rl._prepare_step
def counting(*a, **k):
    hits[0] += 1
    return orig(*a, **k)
rl._prepare_step = counting
for pf in (False, True, False, True):
    for t in range(3): rl.train_step(net, adam, ds, cfg, rng, t, prefetch=pf)
    torch.cuda.synchronize()
    hits[0] = 0
    t0 = time.perf_counter()
    for t in range(10): rl.train_step(net, adam, ds, cfg, rng, 3 + t, prefetch=pf)
    torch.cuda.synchronize()
    print(f"prefetch={pf}: {(time.perf_counter() - t0) / 10 * 1e3:.2f} ms/step, prepares {hits[0]} for 10 steps")
