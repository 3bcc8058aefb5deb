"""Blue-noise spectral statistics on the GPU -- htlab.spectral drop-in.

ring_partition (spectral.py:39-55) is host-side integer set-up (cached, like
the reference's _part_cache, rl.py:266-268).  The periodogram, the anisotropy
loss, its gradient (spectral.py:17-24, 100-133) and the RAPSD / anisotropy of
halftones (spectral.py:74-97) run in csrc/spectral.cu in float64 (batched
cuFFT transforms + ring-reduction kernels).  The drop-in functions take the
reference's float64 arrays and compute on them in float64; the training path
feeds float32 probability maps (anisotropy_device).
"""

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib


@dataclass(frozen=True)
class RingPartition:
    """spectral.py:27-32."""
    shape: tuple
    ring_index: np.ndarray = field(repr=False)   # -1 marks the DC bin
    radii: np.ndarray = field(repr=False)
    counts: np.ndarray = field(repr=False)


def _signed_freqs(n):
    return ((np.arange(n) + n // 2) % n) - n // 2


def ring_partition(shape):
    """spectral.py:39-55: ring = rint(|f|) on the signed DFT lattice, DC -> -1,
    densely re-indexed."""
    hgt, wid = shape
    if hgt < 1 or wid < 1:
        raise ValueError("shape must be positive")
    fy, fx = _signed_freqs(hgt), _signed_freqs(wid)
    ring = np.rint(np.sqrt(fy[:, None] ** 2.0 + fx[None, :] ** 2.0)).astype(np.int64)
    ring[0, 0] = -1
    radii, inv = np.unique(ring[ring > 0], return_inverse=True)
    dense = np.full(ring.shape, -1, dtype=np.int64)
    dense[ring > 0] = inv
    counts = np.bincount(inv, minlength=len(radii)).astype(np.int64)
    return RingPartition((hgt, wid), dense, radii, counts)


def ring_count(shape):
    return len(ring_partition(shape).radii)


_dev_parts = {}


def _part_device(part, device):
    import torch
    key = (part.shape, str(device))
    if key not in _dev_parts:
        ring = torch.from_numpy(part.ring_index.astype(np.int32).ravel()).to(device)
        counts = torch.from_numpy(part.counts.astype(np.int32)).to(device)
        _dev_parts[key] = (ring, counts)
    return _dev_parts[key]


def anisotropy_device(x, part=None, scale=1.0, want_grad=True):
    """Batched K5 on a device tensor x (B, H, W) float32.
    Returns (loss float64 (B,), grad float32 (B,H,W) * scale or None)."""
    import torch
    B, H, W = x.shape
    part = part or ring_partition((H, W))
    if part.shape != (H, W):
        raise ValueError("partition shape mismatch")
    ring, counts = _part_device(part, x.device)
    nr = len(part.radii)
    loss = torch.empty(B, dtype=torch.float64, device=x.device)
    grad = torch.empty((B, H, W), dtype=torch.float32, device=x.device) if want_grad else None
    nbytes = _lib.out_i64("ht_spectral_workspace_bytes", B, H, W, nr)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    _lib.call("ht_anisotropy", _lib.ptr(x.contiguous()), B, H, W, _lib.ptr(ring),
              _lib.ptr(counts), nr, float(scale), _lib.ptr(loss), _lib.ptr(grad), _lib.ptr(ws),
              nbytes, _lib.stream_ptr())
    return loss, grad


def _to_device(x, what="expects"):
    """float64 (1, H, W) CUDA tensor of a non-empty 2-D array (no downcast)."""
    import torch
    _lib.require_cuda()
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2 or x.size == 0:
        raise ValueError(f"{what} a non-empty 2-D array")
    return torch.from_numpy(np.ascontiguousarray(x))[None].cuda()


def _aniso_f64(xd, part, want_grad):
    import torch
    B, H, W = xd.shape
    part = part or ring_partition((H, W))
    if part.shape != (H, W):
        raise ValueError("partition shape mismatch")
    ring, counts = _part_device(part, xd.device)
    nr = len(part.radii)
    loss = torch.empty(B, dtype=torch.float64, device=xd.device)
    grad = torch.empty((B, H, W), dtype=torch.float64, device=xd.device) if want_grad else None
    nbytes = _lib.out_i64("ht_spectral_workspace_bytes", B, H, W, nr)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=xd.device)
    _lib.call("ht_anisotropy_f64", _lib.ptr(xd), B, H, W, _lib.ptr(ring), _lib.ptr(counts), nr, 1.0,
              _lib.ptr(loss), _lib.ptr(grad), _lib.ptr(ws), nbytes, _lib.stream_ptr())
    return loss, grad


def anisotropy_loss(x, part=None):
    """spectral.py:117-121 (float64 throughout)."""
    loss, _ = _aniso_f64(_to_device(x), part, want_grad=False)
    return float(loss[0].item())


def anisotropy_loss_backward(x, part=None):
    """spectral.py:124-133: analytic gradient (float64 array)."""
    _, grad = _aniso_f64(_to_device(x), part, want_grad=True)
    return grad[0].cpu().numpy()


def periodogram(x):
    """spectral.py:17-24: P(f) = |DFT(x)|^2 / N, float64 (H, W)."""
    import torch
    xd = _to_device(x, "periodogram expects")
    _, H, W = xd.shape
    P = torch.empty((1, H, W), dtype=torch.float64, device=xd.device)
    nbytes = _lib.out_i64("ht_spectral_workspace_bytes", 1, H, W, 1)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=xd.device)
    _lib.call("ht_periodogram_f64", _lib.ptr(xd), 1, H, W, _lib.ptr(P), _lib.ptr(ws), nbytes,
              _lib.stream_ptr())
    return P[0].cpu().numpy()


@dataclass
class RapsdCurve:
    """spectral.py:58-64."""
    radii: np.ndarray
    power: np.ndarray
    anisotropy: np.ndarray
    counts: np.ndarray
    dc_power: float


def rapsd_device(x, part=None):
    """K7: rapsd(periodogram(x_b)) for B images x (B,H,W) float32 on device.
    Returns (power (B,R), anis (B,R), dc (B,)) float64 device tensors."""
    import torch
    B, H, W = x.shape
    part = part or ring_partition((H, W))
    ring, counts = _part_device(part, x.device)
    nr = len(part.radii)
    power = torch.empty((B, nr), dtype=torch.float64, device=x.device)
    anis = torch.empty((B, nr), dtype=torch.float64, device=x.device)
    dc = torch.empty(B, dtype=torch.float64, device=x.device)
    nbytes = _lib.out_i64("ht_spectral_workspace_bytes", B, H, W, nr)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    _lib.call("ht_rapsd", _lib.ptr(x.contiguous()), B, H, W, _lib.ptr(ring), _lib.ptr(counts), nr,
              _lib.ptr(power), _lib.ptr(anis), _lib.ptr(dc), _lib.ptr(ws), nbytes,
              _lib.stream_ptr())
    return power, anis, dc


def rapsd(p_hat, part=None):
    """spectral.py:74-88: radially averaged power and per-ring anisotropy of
    a periodogram p_hat (H, W) -> RapsdCurve."""
    import torch
    _lib.require_cuda()
    p_hat = np.asarray(p_hat, dtype=np.float64)
    if p_hat.ndim != 2 or p_hat.size == 0:
        raise ValueError("rapsd expects a non-empty 2-D periodogram")
    part = part or ring_partition(p_hat.shape)
    if part.shape != p_hat.shape:
        raise ValueError("partition shape mismatch")
    H, W = p_hat.shape
    Pd = torch.from_numpy(np.ascontiguousarray(p_hat))[None].cuda()
    ring, counts = _part_device(part, Pd.device)
    nr = len(part.radii)
    power = torch.empty((1, nr), dtype=torch.float64, device=Pd.device)
    anis = torch.empty((1, nr), dtype=torch.float64, device=Pd.device)
    dc = torch.empty(1, dtype=torch.float64, device=Pd.device)
    nbytes = _lib.out_i64("ht_spectral_workspace_bytes", 1, H, W, nr)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=Pd.device)
    _lib.call("ht_rapsd_power_f64", _lib.ptr(Pd), 1, H, W, _lib.ptr(ring), _lib.ptr(counts), nr,
              _lib.ptr(power), _lib.ptr(anis), _lib.ptr(dc), _lib.ptr(ws), nbytes, _lib.stream_ptr())
    return RapsdCurve(part.radii.copy(), power[0].cpu().numpy(), anis[0].cpu().numpy(),
                      part.counts.copy(), float(dc[0].item()))


def image_rapsd(x, part=None):
    """rapsd(periodogram(x)) (spectral.py:17-24, 74-88) for one image, in one
    pass on the device (float64)."""
    import torch
    xd = _to_device(x)
    _, H, W = xd.shape
    part = part or ring_partition((H, W))
    ring, counts = _part_device(part, xd.device)
    nr = len(part.radii)
    power = torch.empty((1, nr), dtype=torch.float64, device=xd.device)
    anis = torch.empty((1, nr), dtype=torch.float64, device=xd.device)
    dc = torch.empty(1, dtype=torch.float64, device=xd.device)
    nbytes = _lib.out_i64("ht_spectral_workspace_bytes", 1, H, W, nr)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=xd.device)
    _lib.call("ht_rapsd_f64", _lib.ptr(xd), 1, H, W, _lib.ptr(ring), _lib.ptr(counts), nr,
              _lib.ptr(power), _lib.ptr(anis), _lib.ptr(dc), _lib.ptr(ws), nbytes, _lib.stream_ptr())
    return RapsdCurve(part.radii.copy(), power[0].cpu().numpy(), anis[0].cpu().numpy(),
                      part.counts.copy(), float(dc[0].item()))


def anisotropy_db(anis):
    """spectral.py:91-97 (post-processing of a few hundred numbers)."""
    anis = np.asarray(anis, dtype=np.float64)
    out = np.full(anis.shape, math.nan)
    ok = np.isfinite(anis) & (anis > 0)
    out[ok] = 10.0 * np.log10(anis[ok])
    return out
