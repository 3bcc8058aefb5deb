"""Golden fixture for the drop-in RewardContext / delta_map in float64.

    python tests/golden/make_context_golden.py

Runs the REAL reference (htlab.metrics, /root/reference/pkg/src, read-only)
on float64 inputs that are NOT float32-representable, so a float32 round trip
on the device path would show: every map of RewardContext (metrics.py:
165-204) and delta_map (metrics.py:333-392) for a binary and a 4-level
action map, both HVS models.  Writes tests/golden/context.npz.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from htlab import hvs, metrics  # noqa: E402

MAPS = ("f_c", "mu_c", "scc", "sigma_c", "f_h", "e", "sq_err", "mu_h", "shh", "shc",
        "cssim_map", "reward_map")


def main():
    rng = np.random.default_rng(2024)
    H, W = 29, 37
    c = np.clip(0.5 + 0.3 * rng.standard_normal((H, W)), 0.0, 1.0)
    c = c + 1e-9 * rng.standard_normal((H, W))          # float64-only digits
    h2 = (rng.uniform(size=(H, W)) < c).astype(np.float64)
    h4 = np.round(np.clip(c + 0.2 * rng.standard_normal((H, W)), 0, 1) * 3) / 3
    other4 = np.round(rng.uniform(size=(H, W)) * 3) / 3
    out = {"c": c, "h2": h2, "h4": h4, "other4": other4}
    for model in ("nasanen", "gaussian"):
        cfg = metrics.MetricConfig(hvs=hvs.HvsConfig(model=model))
        for tag, h, other in (("h2", h2, 1.0 - h2), ("h4", h4, other4)):
            ctx = metrics.reward(h, c, cfg, region="full")
            key = f"{model}_{tag}"
            for m in MAPS:
                out[f"{key}_{m}"] = getattr(ctx, m)
            out[f"{key}_ssim"] = ctx.ssim_maps.ssim
            out[f"{key}_lum"] = ctx.ssim_maps.luminance
            out[f"{key}_con"] = ctx.ssim_maps.contrast
            out[f"{key}_str"] = ctx.ssim_maps.structure
            out[f"{key}_scalars"] = np.array([ctx.mse, ctx.cssim_scalar, ctx.reward])
            out[f"{key}_delta"] = metrics.delta_map(ctx, other)
    path = os.path.join(HERE, "context.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.1f} kB)")


if __name__ == "__main__":
    main()
