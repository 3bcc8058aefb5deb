"""Reward machinery on the GPU -- htlab.metrics drop-in for the training path.

Mirrors MetricConfig (metrics.py:31-39), SsimMaps (metrics.py:110-115),
reward()/RewardContext (metrics.py:158-209, region="full") and delta_map
(metrics.py:333-392).  All maps are computed by the K3/K4 CUDA kernels
(csrc/reward.cu) in float64 from the caller's float64 arrays; the training
path (reward_signal_device) feeds float32 action / contone maps.  The
'valid' evaluation region is a reporting path outside the hot path (SURVEY.md
§2 row 13) and raises NotImplementedError.
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


@dataclass
class SsimMaps:
    """metrics.py:110-115."""
    ssim: np.ndarray
    luminance: np.ndarray
    contrast: np.ndarray
    structure: np.ndarray


class RewardContext:
    """metrics.RewardContext for region='full' (metrics.py:165-204).

    h is any action map (binary or on an L-level lattice), c the contone,
    both kept float64.  Every map of the reference context is computed on
    the GPU in float64 (ht_reward_context_f64): f_c, mu_c, scc, sigma_c
    (contone side), f_h, e, sq_err, mu_h, shh, shc, ssim_maps, cssim_map,
    reward_map, and the scalars mse, cssim_scalar and reward = -mse + w_s *
    cssim_scalar (metrics.py:201-203).  delta() evaluates substitutions on
    the GPU in float64 (K3 maps + K4 deltas)."""

    def __init__(self, h, c, cfg, region="full"):
        if region != "full":
            if region == "valid":
                raise NotImplementedError("region='valid' is an evaluation metric outside the "
                                          "GPU hot path (use region='full')")
            raise ValueError(f"unknown region {region!r}")
        self.cfg, self.region = cfg, region
        self.c = np.asarray(c, dtype=np.float64)
        self.h = np.asarray(h, dtype=np.float64).copy()
        if self.c.shape != self.h.shape:
            raise ValueError("halftone and contone shapes differ")
        if self.h.ndim != 2 or self.h.size == 0:
            raise ValueError("expects non-empty 2-D maps")
        self.kernel = hvs.build_kernel(cfg.hvs)
        self.kf = self.kernel.weights[::-1, ::-1].copy()   # _corr_stencil (metrics.py:52-55)
        self.w = _window_np(cfg.ssim_window, cfg.ssim_sigma)
        self.mask = np.ones(self.h.shape, dtype=bool)
        self.n_region = self.h.size
        self.eval_count = 0
        self._rebuild()

    def _rebuild(self):
        """metrics.py:188-204, on the GPU in float64."""
        import torch
        _lib.require_cuda()
        dev = torch.device("cuda", torch.cuda.current_device())
        H, W = self.h.shape
        k, w = stencils_device(self.cfg, dev)
        hd = torch.from_numpy(self.h)[None].to(dev)
        cd = torch.from_numpy(self.c)[None].to(dev)
        maps = torch.empty((1, 8, H, W), dtype=torch.float64, device=dev)
        extra = torch.empty((1, 7, H, W), dtype=torch.float64, device=dev)
        sums = torch.empty((1, 2), dtype=torch.float64, device=dev)
        scratch = torch.empty((1, H, W), dtype=torch.float64, device=dev)
        cfg = self.cfg
        _lib.call("ht_reward_context_f64", _lib.ptr(hd), _lib.ptr(cd), 1, H, W, _lib.ptr(k), k.shape[0],
                  _lib.ptr(w), w.shape[0], float(cfg.w_s), float(cfg.c1), float(cfg.c2),
                  float(cfg.contrast_gain), _lib.ptr(maps), _lib.ptr(extra), _lib.ptr(sums),
                  _lib.ptr(scratch), _lib.stream_ptr())
        m, x, s = maps[0].cpu().numpy(), extra[0].cpu().numpy(), sums[0].cpu().numpy()
        self.e, self.mu_h, self.shc, self.mu_c, self.scc, self.sigma_c, ssim, self.shh = m
        self.f_h, self.f_c, lum, con, struct, self.cssim_map, self.reward_map = x
        self.sq_err = self.e * self.e
        self.ssim_maps = SsimMaps(ssim, lum, con, struct)
        self.mse = float(s[0] / self.n_region)
        self.cssim_scalar = float(s[1] / self.n_region)
        self.reward = -self.mse + cfg.w_s * self.cssim_scalar
        self.eval_count += 1

    def delta(self, other):
        """R(h with pixel a -> other[a]) - R(h) for every pixel a (float64)."""
        import torch
        dev = torch.device("cuda", torch.cuda.current_device())
        H, W = self.h.shape
        k, w = stencils_device(self.cfg, dev)
        hd = torch.from_numpy(self.h)[None].to(dev)
        cd = torch.from_numpy(self.c)[None].to(dev)
        od = torch.from_numpy(np.ascontiguousarray(other, dtype=np.float64))[None].to(dev)
        out = torch.empty((1, H, W), dtype=torch.float64, device=dev)
        nbytes = _lib.out_i64("ht_reward_workspace_bytes", 1, H, W) + 8 * H * W
        ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        cfg = self.cfg
        _lib.call("ht_reward_delta_f64", _lib.ptr(hd), _lib.ptr(od), _lib.ptr(cd), 1, H, W, _lib.ptr(k),
                  k.shape[0], _lib.ptr(w), w.shape[0], float(cfg.w_s), float(cfg.c1), float(cfg.c2),
                  float(cfg.contrast_gain), _lib.ptr(out), _lib.ptr(ws), nbytes, _lib.stream_ptr())
        return out[0].cpu().numpy()


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