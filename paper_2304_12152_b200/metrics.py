"""Reward machinery on the GPU -- htlab.metrics drop-in for the training path.

Mirrors MetricConfig (metrics.py:31-39), reward()/RewardContext
(metrics.py:158-209, region="full") and delta_map (metrics.py:333-392) for
binary halftones.  All maps are computed by the K3/K4 CUDA kernels
(csrc/reward.cu) in float64.  The 'valid' evaluation region and non-binary
edits (multitone) are reporting paths outside the hot path (SURVEY.md §2
rows 13, 16) and raise NotImplementedError.
"""

import functools
from dataclasses import dataclass, field

import numpy as np

from . import _lib, hvs
from .hvs import HvsConfig


@dataclass(frozen=True)
class MetricConfig:
    """metrics.py:31-39."""
    w_s: float = 0.06
    ssim_window: int = 11
    ssim_sigma: float = 1.5
    c1: float = 0.01 ** 2
    c2: float = 0.03 ** 2
    contrast_gain: float = 2.0
    hvs: HvsConfig = field(default_factory=HvsConfig)


@functools.lru_cache(maxsize=32)
def _kernel_np(hvs_cfg):
    return hvs.build_kernel(hvs_cfg).weights


@functools.lru_cache(maxsize=32)
def _window_np(size, sigma):
    return hvs.build_gaussian_kernel(size, sigma).weights


_dev_cache = {}


def stencils_device(cfg, device):
    """(k_hvs, w_ssim) float64 device tensors for a MetricConfig (cached)."""
    import torch
    key = (cfg.hvs, cfg.ssim_window, cfg.ssim_sigma, str(device))
    if key not in _dev_cache:
        k = torch.from_numpy(np.ascontiguousarray(_kernel_np(cfg.hvs))).to(device)
        w = torch.from_numpy(np.ascontiguousarray(_window_np(cfg.ssim_window, cfg.ssim_sigma))).to(device)
        _dev_cache[key] = (k, w)
    return _dev_cache[key]


ESTIMATOR_CODES = {"local_expectation": 0, "coma": 1, "delta": 2}


def reward_signal_device(p, u, c, cfg, scale=1.0, want_signal=True, levels=2,
                         estimator="local_expectation", other=None):
    """Batched K3+K4 on device tensors (ht_reward_signal).

    p, c: (B, H, W) float32; u: (B, H, W) float64 uniforms, or None when p is
    already the action map; other: (B, H, W) float32 substitutes for
    estimator="delta".  Returns (m float32, signal float32 * scale or None,
    reward float64 (B,))."""
    import torch
    B, H, W = p.shape
    dev = p.device
    k, w = stencils_device(cfg, dev)
    m = torch.empty((B, H, W), dtype=torch.float32, device=dev)
    sig = torch.empty((B, H, W), dtype=torch.float32, device=dev) if want_signal else None
    rew = torch.empty(B, dtype=torch.float64, device=dev)
    nbytes = _lib.out_i64("ht_reward_workspace_bytes", B, H, W)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    _lib.call("ht_reward_signal", _lib.ptr(p.contiguous()),
              _lib.ptr(u.contiguous()) if u is not None else None,
              _lib.ptr(other.contiguous()) if other is not None else None,
              _lib.ptr(c.contiguous()), B, H, W, _lib.ptr(k), k.shape[0], _lib.ptr(w),
              w.shape[0], float(cfg.w_s), float(cfg.c1), float(cfg.c2), float(cfg.contrast_gain),
              int(levels), ESTIMATOR_CODES[estimator], float(scale), _lib.ptr(m), _lib.ptr(sig),
              _lib.ptr(rew), _lib.ptr(ws), nbytes, _lib.stream_ptr())
    return m, sig, rew


def reward_le_device(p, u, c, cfg, scale=1.0, want_signal=True):
    """Binary local-expectation form of reward_signal_device (ht_reward_le)."""
    return reward_signal_device(p, u, c, cfg, scale, want_signal)


def reinforce_signal_device(p, m, reward_b, baseline, scale=1.0):
    """REINFORCE signal on device tensors (ht_reinforce_signal): p, m (B,H,W)
    float32, reward_b (B,) float64."""
    import torch
    B = p.shape[0]
    out = torch.empty_like(p)
    _lib.call("ht_reinforce_signal", _lib.ptr(p.contiguous()), _lib.ptr(m.contiguous()), B,
              p[0].numel(), _lib.ptr(reward_b.contiguous()), float(baseline), float(scale),
              _lib.ptr(out), _lib.stream_ptr())
    return out


class RewardContext:
    """metrics.RewardContext for region='full' (metrics.py:165-204).

    h is any action map (binary or on an L-level lattice).  .reward is the
    scalar R = -HVS-MSE + w_s * CSSIM (metrics.py:201-203); delta_map()
    evaluates substitutions on the GPU (K3 maps + K4 deltas)."""

    def __init__(self, h, c, cfg, region="full"):
        if region != "full":
            if region == "valid":
                raise NotImplementedError("region='valid' is an evaluation metric outside the "
                                          "GPU hot path (use region='full')")
            raise ValueError(f"unknown region {region!r}")
        self.cfg, self.region = cfg, region
        self.h = np.asarray(h, dtype=np.float64).copy()
        self.c = np.asarray(c, dtype=np.float64)
        if self.c.shape != self.h.shape:
            raise ValueError("halftone and contone shapes differ")
        hh, ww = self.h.shape
        self.n_region = hh * ww
        _, _, rew = reward_signal_device(*self._dev(), self.cfg, want_signal=False)
        self.reward = float(rew[0].item())
        self.eval_count = 1

    def _dev(self):
        import torch
        _lib.require_cuda()
        dev = torch.device("cuda", torch.cuda.current_device())
        hd = torch.from_numpy(self.h.astype(np.float32))[None].to(dev)
        cd = torch.from_numpy(self.c.astype(np.float32))[None].to(dev)
        return hd, None, cd

    def delta(self, other):
        import torch
        hd, _, cd = self._dev()
        od = torch.from_numpy(np.asarray(other, dtype=np.float32))[None].to(hd.device)
        _, d, _ = reward_signal_device(hd, None, cd, self.cfg, estimator="delta", other=od)
        return d[0].double().cpu().numpy()


def reward(h, c, cfg=None, region="full"):
    """metrics.py:207-209."""
    return RewardContext(h, c, cfg or MetricConfig(), region)


def delta_map(ctx, other_values):
    """metrics.py:333-358: R(pixel a -> other[a]) - R(h) for every pixel a
    (0 where other == h)."""
    other = np.asarray(other_values, dtype=np.float64)
    if other.shape != ctx.h.shape:
        raise ValueError("other_values shape mismatch")
    hgt, wid = ctx.h.shape
    ctx.eval_count += hgt * wid
    return ctx.delta(other)