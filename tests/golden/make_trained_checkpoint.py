"""Trained-weights fixture for K1 parity beyond random init (GPU box).

    python tests/golden/make_trained_checkpoint.py

Trains the paper network (C=32, 16 blocks) with this package's own
rl.train_loop for 2000 iterations on 64x64 crops (batch 8, anisotropy batch
4, LE estimator, Nasanen HVS -- the reference's TrainConfig defaults apart
from the sizes) of 8 seeded synthetic contones, and writes the bare HTNN
checkpoint tests/golden/trained_c32b16_2k.htnn (byte format of nn.py:205-
300).  The forward parity test (tests/test_gpu_forward.py) checks K1 with
these weights against the oracle; the weights themselves are not a golden
(training is only reproducible to the GPU's atomic-sum order).
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from paper_2304_12152_b200 import rl, synth  # noqa: E402
from paper_2304_12152_b200.checkpoint import save_checkpoint  # noqa: E402


def main(iterations=2000):
    cfg = rl.TrainConfig(iterations=iterations, batch_size=8, crop_size=64, anisotropy_batch_size=4)
    ds = [synth.contone(128, 128, seed=500 + i).astype(np.float64) for i in range(8)]
    t0 = time.time()
    rows = []
    net, adam, rng = rl.train_loop(cfg, ds, on_iteration=lambda t, d, *a: rows.append(d))
    path = os.path.join(HERE, "trained_c32b16_2k.htnn")
    save_checkpoint(path, net)
    w = np.concatenate([p.value.ravel() for p in net.params()])
    print(f"trained {iterations} iterations in {time.time() - t0:.1f}s; reward "
          f"{rows[0]['reward']:.5f} -> {rows[-1]['reward']:.5f}, bin_gap {rows[0]['bin_gap']:.4f} -> "
          f"{rows[-1]['bin_gap']:.4f}; weight std {w.std():.4f}; wrote {path}")


if __name__ == "__main__":
    main()
