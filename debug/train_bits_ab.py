"""Config-5 train step time with the training ReLU bits on (1, default) vs
off (0: fp32 mask / residual epilogue inputs), interleaved, wall clock around
synchronised steps; plus per-kernel GPU time of one step per setting."""
import sys, time, collections
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2304_12152_b200 import rl, synth, _lib
from paper_2304_12152_b200.imagecore import Rng

cfg = rl.TrainConfig(iterations=1000, batch_size=16, crop_size=256, anisotropy_batch_size=4, hvs_model="gaussian")
ds = [synth.contone(384, 384, seed=100 + i).astype(np.float64) for i in range(8)]
rng = Rng(0); net = rl.PolicyNetwork(32, 16); net.init_params(rng); adam = rl.Adam(net.params())
t = 0
def steps(n):
    global t
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        rl.train_step(net, adam, ds, cfg, rng, t); t += 1
        torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    return ts
res = collections.defaultdict(list)
for rep in range(4):
    for impl in (1, 0):
        _lib.call("ht_set_train_bits", impl)
        steps(2)
        res[impl] += steps(5)
for impl, v in res.items():
    print(f"impl {impl}: median {np.median(v):.2f} ms  min {min(v):.2f} ms")
from torch.profiler import profile, ProfilerActivity
for impl in (1, 0):
    _lib.call("ht_set_train_bits", impl)
    steps(2)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        steps(3)
        torch.cuda.synchronize()
    tot = collections.defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot[e.name[:60]][0] += 1; tot[e.name[:60]][1] += e.device_time_total
    s = sum(v[1] for v in tot.values())
    print(f"impl {impl}: GPU time per step {s / 3 / 1e3:.2f} ms")
    for k, (n, tt) in sorted(tot.items(), key=lambda x: -x[1][1])[:6]:
        print(f"   {tt / 3 / 1e3:7.3f} ms/step {n // 3:4d} launches  {k}")
