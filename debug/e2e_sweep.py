"""e2e throughput of rl.HalftoneEngine at config 2 (64 x 512^2): per-call vs
streamed submit/wait, for several chunk counts (wall clock, pinned host)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import rl, synth
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import PolicyNetwork
B, H, W = 64, 512, 512
net = PolicyNetwork(32, 16); net.init_params(Rng(0), std=0.01)
ch = torch.from_numpy(synth.config_batch(B, H, W, seed=2)).pin_memory()
zh = torch.randn(B, H, W).pin_memory()
steps = 12
for chunks in (1, 2, 4):
    eng = rl.HalftoneEngine(net, B, H, W, chunks=chunks, output="h")
    outs = [torch.empty(eng.out_shape(), dtype=torch.uint8).pin_memory() for _ in range(2)]
    def streamed(n):
        t = []
        for i in range(n):
            if i >= 2: eng.wait(t[i - 2])
            t.append(eng.submit(ch, zh, outs[i % 2]))
        for x in t[-2:]: eng.wait(x)
    def percall(n):
        for i in range(n): eng(ch, zh, outs[0])
    for name, f in (("per-call", percall), ("streamed", streamed)):
        f(3); torch.cuda.synchronize()
        t0 = time.perf_counter(); f(steps); el = time.perf_counter() - t0
        print(f"chunks={chunks} {name}: {B * H * W * steps / el / 1e6:.1f} Mpx/s")
