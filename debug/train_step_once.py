"""Three config-5 train steps after warm-up (for an ncu launch list)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import rl, synth
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import Adam, PolicyNetwork
cfg = rl.TrainConfig(iterations=1000, batch_size=16, crop_size=256, anisotropy_batch_size=4, hvs_model="gaussian")
ds = [synth.contone(384, 384, seed=100 + i).astype(np.float64) for i in range(8)]
rng = Rng(0); net = PolicyNetwork(32, 16); net.init_params(rng); adam = Adam(net.params())
for t in range(6): rl.train_step(net, adam, ds, cfg, rng, t)
torch.cuda.synchronize()
