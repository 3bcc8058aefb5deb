"""Golden vectors for the exhaustive expected-reward gradient (rl.py:139-164,
`exact_gradient_oracle`), computed by the REAL reference.  Run in the build
container only:

    python tests/golden/make_exact_grad_golden.py

Writes tests/golden/exact_grad.npz: for each case the (fp32-exact) policy p
(probabilities, or the value map for L > 2), the contone c, the metric
configuration as (w_s, hvs_size, hvs_sigma, ssim_window, levels) and the
reference's d E[R] / d p.  The configurations are the reference tests'
IDENTITY (1x1 filter, no SSIM: R = -(h-c)^2) and SMALL (3x3 HVS and SSIM
windows, tests/test_rl.py:26-29)."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from htlab import hvs, metrics, rl  # noqa: E402
from htlab.imagecore import Rng  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def cfg_of(w_s, hsize, hsigma, win):
    return metrics.MetricConfig(w_s=w_s, ssim_window=win,
                                hvs=hvs.HvsConfig(model="gaussian", size=hsize, sigma=hsigma))


def main():
    out = {}
    cases = [
        # name, shape, (w_s, hvs size, hvs sigma, ssim window), levels, seed
        ("identity_1x1", (1, 1), (0.0, 1, 1.0, 3), 2, None),
        ("small_2x2", (2, 2), (0.06, 3, 1.0, 3), 2, 31),
        ("small_2x3", (2, 3), (0.06, 3, 1.0, 3), 2, 33),
        ("small_3x3", (3, 3), (0.06, 3, 1.0, 3), 2, 35),
        ("small_ws0_3x3", (3, 3), (0.0, 3, 1.0, 3), 2, 37),
        ("mt3_2x3", (2, 3), (0.06, 3, 1.0, 3), 3, 39),
        ("mt4_2x2", (2, 2), (0.06, 3, 1.0, 3), 4, 41),
    ]
    names = []
    for name, shape, (w_s, hs, hsg, win), L, seed in cases:
        if seed is None:
            p, c = f32([[0.55]]), f32([[0.3]])
        else:
            r = Rng(seed)
            n = shape[0] * shape[1]
            p = f32(0.1 + 0.8 * r.uniforms(n).reshape(shape))
            c = f32(r.uniforms(n).reshape(shape))
        g = rl.exact_gradient_oracle(p, c, cfg_of(w_s, hs, hsg, win), level_count=L)
        out[f"{name}_p"] = p
        out[f"{name}_c"] = c
        out[f"{name}_cfg"] = np.array([w_s, hs, hsg, win, L], dtype=np.float64)
        out[f"{name}_grad"] = g
        names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "exact_grad.npz"), **out)
    print("wrote exact_grad.npz:", names)


if __name__ == "__main__":
    main()
