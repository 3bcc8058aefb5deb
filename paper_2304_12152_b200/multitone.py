"""Multitone halftoning on a uniform lattice of L output levels (htlab
multitone.py).

Inference runs the fused forward with a level epilogue (K1, ht_multitone):
the nearest lattice level of the policy output, half-steps rounding up; L=2
is the binary threshold rule.  Training shares the binary path's device
kernels: the two-point cast of the value map onto the lattice, sampling, and
the local-expectation signal scaled by 1/delta (ht_reward_signal).
"""

from dataclasses import dataclass

import numpy as np

from . import rl


@dataclass(frozen=True)
class LevelSet:
    """multitone.py:18-32: uniform output lattice i/(L-1), i = 0..L-1."""
    count: int

    def __post_init__(self):
        if self.count < 2:
            raise ValueError("a level set needs at least 2 levels")

    @property
    def delta(self):
        return 1.0 / (self.count - 1)

    @property
    def values(self):
        return np.arange(self.count) / (self.count - 1)


def cast_probabilities(v, levels):
    """multitone.py:35-41: (floor_vals, ceil_vals, p_ceil) per value."""
    return rl._cast_two_point(v, levels.count)


def sample_multitone(v, levels, rng):
    """multitone.py:44-47: one lattice level per pixel from the cast."""
    floor_vals, ceil_vals, p_ceil = cast_probabilities(v, levels)
    return rl._sample_two_point(floor_vals, ceil_vals, p_ceil, rng)


def make_multitone_sample(v, c, z, levels, rng, cfg=None):
    """multitone.py:50-51."""
    return rl.make_sample(v, c, z, rng, cfg, level_count=levels.count)


def le_signal_multitone(sample):
    """multitone.py:54-57: two-point reward difference scaled by 1/delta."""
    return rl.le_signal(sample)


def quantize_multitone(v, levels):
    """multitone.py:60-67: nearest lattice level, half-steps round up."""
    v = np.asarray(v, dtype=np.float64)
    steps = levels.count - 1
    return np.clip(np.floor(v * steps + 0.5), 0, steps) / steps


def multitone(net, contone, noise, levels, impl=None):
    """Noise-explicit multitone inference on the GPU: returns (m, v) with m
    on the lattice (float64) and v the policy output."""
    torch = rl._torch()
    from . import _lib
    _lib.require_cuda()
    count = levels.count if isinstance(levels, LevelSet) else int(levels)
    dev = net.device
    cd = torch.from_numpy(np.ascontiguousarray(contone, dtype=np.float32)).to(dev) \
        if not isinstance(contone, torch.Tensor) else contone.to(dev, torch.float32)
    zd = torch.from_numpy(np.ascontiguousarray(noise, dtype=np.float32)).to(dev) \
        if not isinstance(noise, torch.Tensor) else noise.to(dev, torch.float32)
    if cd.shape != zd.shape or cd.dim() != 2 or cd.numel() == 0:
        raise ValueError("contone and noise must be non-empty (H, W) maps of the same shape")
    v = torch.empty(cd.shape, dtype=torch.float32, device=dev)
    q = torch.empty(cd.shape, dtype=torch.uint8, device=dev)
    net.halftone_device(cd, zd, p_out=v, h_out=q, impl=impl, check=True, levels=count)
    return q.double().cpu().numpy() / (count - 1), v.double().cpu().numpy()


def infer_multitone(net, c, levels, rng, impl=None):
    """multitone.py:70-76: draw z = gaussian_noise_map(rng, W, H) (on the
    GPU, same stream), run the policy once, round to the lattice.  Returns
    (m, v)."""
    from .imagecore import gaussian_noise_map_device
    c = np.asarray(c, dtype=np.float64)
    if c.ndim != 2 or c.size == 0:
        raise ValueError("contone must be a non-empty (H, W) array")
    z = gaussian_noise_map_device(rng, c.shape[1], c.shape[0], device=net.device)
    return multitone(net, c, z, levels, impl=impl)
