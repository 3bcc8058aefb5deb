"""HVS stencils (host constants), mirroring htlab.hvs (hvs.py:37-103).

The kernels are 11x11 unit-sum float64 arrays built once on the host and
passed to the CUDA reward kernels as data.
"""

from dataclasses import dataclass, field

import numpy as np

NASANEN_CONSTANTS = {"a": 131.6, "b": 0.3188, "c": 0.525, "d": 3.91, "luminance": 11.0}


@dataclass(frozen=True)
class HvsKernel:
    """Odd square spatial kernel with unit coefficient sum (hvs.py:22-34)."""
    size: int
    weights: np.ndarray = field(repr=False)

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=np.float64)
        if w.shape != (self.size, self.size):
            raise ValueError("kernel weights must be size x size")
        if self.size % 2 != 1 or self.size < 1:
            raise ValueError("kernel size must be odd and positive")
        object.__setattr__(self, "weights", w)


@dataclass(frozen=True)
class HvsConfig:
    """hvs.py:37-43: 'nasanen' (scale S) or 'gaussian' (sigma)."""
    model: str = "nasanen"
    size: int = 11
    scale: float = 2000.0
    sigma: float = 2.0


def build_gaussian_kernel(size, sigma):
    """hvs.py:54-64: sampled isotropic Gaussian, unit sum."""
    if size % 2 != 1 or size < 1:
        raise ValueError("kernel size must be odd and positive")
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    half = size // 2
    ax = np.arange(-half, half + 1, dtype=np.float64)
    g = np.exp(-(ax * ax) / (2.0 * sigma * sigma))
    k = np.outer(g, g)
    return HvsKernel(size, k / k.sum())


def nasanen_frequency_response(f_cpd, constants=None):
    """hvs.py:67-73."""
    c = constants or NASANEN_CONSTANTS
    lum = c["luminance"]
    return c["a"] * lum ** c["b"] * np.exp(
        -np.asarray(f_cpd, dtype=np.float64) / (c["c"] * np.log(lum) + c["d"]))


def build_nasanen_kernel(size, scale, dense_size=128):
    """hvs.py:83-103: CSF sampled on a dense DFT grid, inverse DFT, centre
    crop, renormalise."""
    if size % 2 != 1 or size < 1:
        raise ValueError("kernel size must be odd and positive")
    if scale <= 0:
        raise ValueError("scale must be positive")
    if dense_size < size:
        raise ValueError("dense grid smaller than requested kernel")
    f = np.fft.fftfreq(dense_size)
    rho = np.sqrt(f[:, None] ** 2 + f[None, :] ** 2) * np.pi * scale / 180.0
    spatial = np.fft.fftshift(np.fft.ifft2(nasanen_frequency_response(rho)).real)
    half, mid = size // 2, dense_size // 2
    k = spatial[mid - half:mid + half + 1, mid - half:mid + half + 1].copy()
    return HvsKernel(size, k / k.sum())


def build_kernel(cfg):
    """hvs.py:46-51."""
    if cfg.model == "nasanen":
        return build_nasanen_kernel(cfg.size, cfg.scale)
    if cfg.model == "gaussian":
        return build_gaussian_kernel(cfg.size, cfg.sigma)
    raise ValueError(f"unknown HVS model {cfg.model!r}")
