"""Golden vectors for the estimators and multitone path,
computed by the REAL reference.  Run in the build container only:

    python tests/golden/make_estimators_golden.py

Writes tests/golden/estimators.npz:
  binary (L=2, 40x36, gaussian HVS): p, c, m sampled by rl.make_sample with
    Rng(21), the reward, le / coma / reinforce / reinforce(baseline) signals;
  multitone (L=4 and L=3, 32x28): v (with exact on-lattice values), c, the
    sample's m / floor / ceil / p_ceil, reward and le_signal;
  quantize: quantize_multitone of values incl. exact half-steps for L=2..7.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from htlab import hvs, metrics, multitone, rl  # noqa: E402
from htlab.imagecore import Rng  # noqa: E402

from paper_2304_12152_b200 import synth  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    out = {}
    cfg = metrics.MetricConfig(hvs=hvs.HvsConfig(model="gaussian"))
    # ---- binary estimators
    hh, ww = 40, 36
    c = f32(synth.contone(hh, ww, seed=31))
    p = f32(np.clip(Rng(32).uniforms(hh * ww).reshape(hh, ww), 0.0, 1.0))
    p[0, :4] = f32([0.0, 1.0, 1e-9, 1.0 - 2.0 ** -24])   # collapsed support / clip floor (fp32-exact)
    s = rl.make_sample(p, c, None, Rng(21), cfg)
    out.update(bin_c=c, bin_p=p, bin_m=s.m, bin_reward=np.array([s.ctx.reward]),
               bin_le=rl.le_signal(s), bin_coma=rl.coma_signal(s),
               bin_reinforce=rl.reinforce_signal(s),
               bin_reinforce_b=rl.reinforce_signal(s, baseline=0.0123))
    # ---- multitone samples + LE
    for L in (4, 3):
        hh, ww = 32, 28
        c = f32(synth.contone(hh, ww, seed=40 + L))
        v = f32(Rng(50 + L).uniforms(hh * ww).reshape(hh, ww))
        v[0, :L] = f32(np.arange(L) / (L - 1))           # on / next to the lattice (fp32-exact)
        lv = multitone.LevelSet(L)
        s = multitone.make_multitone_sample(v, c, None, lv, Rng(60 + L), cfg)
        out.update({f"mt{L}_c": c, f"mt{L}_v": v, f"mt{L}_m": s.m, f"mt{L}_floor": s.floor_vals,
                    f"mt{L}_ceil": s.ceil_vals, f"mt{L}_pceil": s.p_ceil,
                    f"mt{L}_reward": np.array([s.ctx.reward]),
                    f"mt{L}_le": multitone.le_signal_multitone(s)})
    # ---- quantize
    vals = [0.0, 1.0, 0.5, 0.25, 0.75, 1.0 / 3.0, 2.0 / 3.0, 1.0 / 6.0, 0.1, 0.9, 0.4999999, 0.5000001]
    q = np.array(vals + list(Rng(70).uniforms(40)))
    out["q_v"] = q
    for L in range(2, 8):
        out[f"q_L{L}"] = multitone.quantize_multitone(q, multitone.LevelSet(L))
    np.savez_compressed(os.path.join(HERE, "estimators.npz"), **out)
    print("wrote estimators.npz:", ", ".join(sorted(out)))


if __name__ == "__main__":
    main()
