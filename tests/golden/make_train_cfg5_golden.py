"""Golden fixture for BASELINE config 5 at full size, from the REAL reference.

    python tests/golden/make_train_cfg5_golden.py [gaussian|nasanen ...]

One `htlab.rl.train_step` (rl.py:232-278) with
TrainConfig(batch_size=16, crop_size=256, anisotropy_batch_size=4) -- the
paper architecture (C=32, 16 blocks), 16 MARL crops of 256x256 from 8 seeded
384x384 synthetic contones plus 4 flat-gray images -- once per HVS model.
About 6 minutes and 9 GB of cached activations per model on one core.

Runs in the build container only (imports /root/reference/pkg/src read-only).
The dataset is regenerated on the GPU box from `synth` (its SHA-256 is stored
and checked).  Stored per model (`{hvs}_...`): RNG states before/after, the
diagnostics row, the full flat parameter gradient and the post-Adam parameter
delta (float32: their rounding is 6e-8 relative, far below the 1e-4 bar),
the sampled action maps (bit-packed) and LE-signal / probability probes, so a
GPU step can be compared normwise per tensor and its sampled actions counted.
"""

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from htlab import nn, rl  # noqa: E402
from htlab.imagecore import Rng  # noqa: E402

from paper_2304_12152_b200 import synth  # noqa: E402

SUB = (slice(3, None, 37), slice(5, None, 41))      # fixed probe grid of a 256x256 map


def dataset():
    return [synth.contone(384, 384, seed=100 + i).astype(np.float64) for i in range(8)]


def dataset_sha(ds):
    h = hashlib.sha256()
    for a in ds:
        h.update(np.ascontiguousarray(a, dtype="<f8").tobytes())
    return np.frombuffer(h.digest(), dtype=np.uint8)


def run(hvs):
    t0 = time.time()
    cfg = rl.TrainConfig(iterations=1000, batch_size=16, crop_size=256,
                         anisotropy_batch_size=4, hvs_model=hvs)
    ds = dataset()
    rng = Rng(cfg.seed)
    net = nn.PolicyNetwork(channels=cfg.channels, blocks=cfg.blocks)
    adam = nn.Adam(net.params())
    net.init_params(rng)
    p0 = np.concatenate([q.value.ravel() for q in net.params()])
    state0 = rng.state_words()

    # record the samples and signals the step builds (read-only wrappers
    # around the reference functions; the step itself is unmodified)
    seen = {"m": [], "p": [], "sig": []}
    orig_make, orig_sig = rl.make_sample, rl._signals_for_batch

    def make_sample(p, c, z, r, mcfg=None, level_count=2):
        s = orig_make(p, c, z, r, mcfg, level_count)
        seen["m"].append(s.m.copy())
        seen["p"].append(s.p.copy())
        return s

    def signals(samples, est):
        out = orig_sig(samples, est)
        seen["sig"].extend([np.array(a) for a in out])
        return out

    rl.make_sample, rl._signals_for_batch = make_sample, signals
    try:
        diag = rl.train_step(net, adam, ds, cfg, rng, 0)
    finally:
        rl.make_sample, rl._signals_for_batch = orig_make, orig_sig
    g = np.concatenate([q.grad.ravel() for q in net.params()])
    p1 = np.concatenate([q.value.ravel() for q in net.params()])
    m = np.stack(seen["m"]).astype(np.uint8)
    p = np.stack(seen["p"])
    sig = np.stack(seen["sig"])
    out = {
        f"{hvs}_state0": np.array(state0, dtype=np.uint64),
        f"{hvs}_state1": np.array(rng.state_words(), dtype=np.uint64),
        f"{hvs}_diag": np.array([diag["reward"], diag["l_as"], diag["bin_gap"], diag["lr"]]),
        f"{hvs}_grad": g.astype(np.float32),
        f"{hvs}_grad_norms": np.array([np.linalg.norm(q.grad) for q in net.params()]),
        f"{hvs}_dparam": (p1 - p0).astype(np.float32),
        f"{hvs}_m_bits": np.packbits(m, axis=-1),
        f"{hvs}_p_sum": p.reshape(16, -1).sum(axis=1),
        f"{hvs}_p_sub": p[:, SUB[0], SUB[1]],
        f"{hvs}_sig_sum": sig.reshape(16, -1).sum(axis=1),
        f"{hvs}_sig_absum": np.abs(sig).reshape(16, -1).sum(axis=1),
        f"{hvs}_sig_sub": sig[:, SUB[0], SUB[1]],
        f"{hvs}_seconds": np.array([time.time() - t0]),
    }
    return out


if __name__ == "__main__":
    models = sys.argv[1:] or ["gaussian", "nasanen"]
    for hvs in models:
        out = run(hvs)
        out["dataset_sha"] = dataset_sha(dataset())
        path = os.path.join(HERE, f"train_cfg5_{hvs}.npz")
        np.savez_compressed(path, **out)
        print(f"wrote {path} ({os.path.getsize(path) / 1e3:.1f} kB) in "
              f"{float(out[f'{hvs}_seconds'][0]):.0f}s")
