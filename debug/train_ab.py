"""A/B the config-5 train step: current rl vs a saved older rl module source.
    python debug/train_ab.py debug/rl_old.py.txt"""
import importlib.util, sys, time, types
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2304_12152_b200 as pkg
from paper_2304_12152_b200 import rl as rl_new, synth
from paper_2304_12152_b200.imagecore import Rng

src = open(sys.argv[1]).read()
rl_old = types.ModuleType('paper_2304_12152_b200.rl_old')
rl_old.__package__ = 'paper_2304_12152_b200'
exec(compile(src, 'rl_old', 'exec'), rl_old.__dict__)

def run(rl, steps=6, warm=3):
    cfg = rl.TrainConfig(iterations=1000, batch_size=16, crop_size=256, anisotropy_batch_size=4)
    ds = [synth.config_batch(1, 512, 512, seed=s)[0].astype(np.float64) for s in range(4)]
    rng = Rng(0)
    net = rl.PolicyNetwork(32, 16); net.init_params(rng)
    adam = rl.Adam(net.params())
    for t in range(warm): rl.train_step(net, adam, ds, cfg, rng, t)
    ts = []
    for t in range(steps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        rl.train_step(net, adam, ds, cfg, rng, warm + t)
        torch.cuda.synchronize(); ts.append(round((time.perf_counter() - t0) * 1e3, 1))
    return ts

for rep in range(3):
    print("old", run(rl_old), "\nnew", run(rl_new))
