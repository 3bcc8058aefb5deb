"""Host-side input preparation: the reference RNG and image helpers.

Mirrors htlab.imagecore (imagecore.py:14-171).  The xoshiro256++ stream and
the Box-Muller gaussians run in C inside libhtb200.so (ht_rng_*), bit-exact
with the reference's pure-Python loop (uniforms exactly; gaussians to libm
rounding), so noise maps for print pages take ~0.3 s instead of ~45 s.
This is input preparation, never part of a timed region.
"""

import ctypes as C

import numpy as np

from . import _lib

_M64 = (1 << 64) - 1


def splitmix64(state):
    """imagecore.py:14-21: returns (new_state, output)."""
    state = (state + 0x9E3779B97F4A7C15) & _M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return state, z ^ (z >> 31)


def derive_seed(seed, index):
    """imagecore.py:24-32."""
    if index < 0:
        raise ValueError("index must be non-negative")
    s, z = seed & _M64, 0
    for _ in range(index + 1):
        s, z = splitmix64(s)
    return z


class Rng:
    """xoshiro256++ seeded through splitmix64 (imagecore.py:35-120)."""

    def __init__(self, seed):
        self.seed = int(seed) & _M64
        self._s = (C.c_uint64 * 4)()
        _lib.call("ht_rng_seed", C.c_uint64(self.seed), self._s)

    def next_uint64(self):
        s0, s1, s2, s3 = (int(v) for v in self._s)
        x = (s0 + s3) & _M64
        r = ((((x << 23) | (x >> 41)) & _M64) + s0) & _M64
        t = (s1 << 17) & _M64
        s2 ^= s0
        s3 ^= s1
        s1 ^= s2
        s0 ^= s3
        s2 ^= t
        s3 = ((s3 << 45) | (s3 >> 19)) & _M64
        self._s[:] = [s0, s1, s2, s3]
        return r

    def uniform(self):
        return float(self.uniforms(1)[0])

    def uniforms(self, n):
        out = np.empty(int(n), dtype=np.float64)
        _lib.call("ht_rng_uniforms", self._s, C.c_int64(int(n)), out.ctypes.data_as(C.c_void_p))
        return out

    def gaussians(self, n):
        out = np.empty(int(n), dtype=np.float64)
        _lib.call("ht_rng_gaussians", self._s, C.c_int64(int(n)), out.ctypes.data_as(C.c_void_p))
        return out

    def gaussians_f32(self, n):
        out = np.empty(int(n), dtype=np.float32)
        _lib.call("ht_rng_gaussians_f32", self._s, C.c_int64(int(n)),
                  out.ctypes.data_as(C.c_void_p))
        return out

    def gaussian(self):
        return float(self.gaussians(1)[0])

    def jump(self, n):
        """Advance the stream by n draws without producing them."""
        _lib.call("ht_rng_jump", self._s, C.c_uint64(int(n)))

    def _device_out(self, n, out, dtype, device):
        import torch
        if out is None:
            dev = torch.device(device) if device is not None else torch.device(
                "cuda", torch.cuda.current_device())
            out = torch.empty(int(n), dtype=dtype, device=dev)
        if not out.is_cuda or not out.is_contiguous() or out.numel() != int(n) or out.dtype not in (
                torch.float32, torch.float64):
            raise ValueError("out must be a contiguous CUDA float32/float64 tensor of n elements")
        return out

    def gaussians_device(self, n, out=None, dtype=None, device=None):
        """Rng.gaussians(n) generated on the GPU (same stream; the host state
        advances identically).  Returns a CUDA tensor (float32 by default)."""
        import torch
        _lib.require_cuda()
        out = self._device_out(n, out, dtype or torch.float32, device)
        with torch.cuda.device(out.device):
            _lib.call("ht_rng_gaussians_device", self._s, C.c_int64(int(n)), _lib.ptr(out),
                      int(out.dtype == torch.float64), _lib.stream_ptr())
        return out

    def uniforms_device(self, n, out=None, dtype=None, device=None):
        """Rng.uniforms(n) generated on the GPU (bit-exact; the host state
        advances identically).  Returns a CUDA tensor (float64 by default)."""
        import torch
        _lib.require_cuda()
        out = self._device_out(n, out, dtype or torch.float64, device)
        with torch.cuda.device(out.device):
            _lib.call("ht_rng_uniforms_device", self._s, C.c_int64(int(n)), _lib.ptr(out),
                      int(out.dtype == torch.float64), _lib.stream_ptr())
        return out

    def randint(self, n):
        """imagecore.py:104-108."""
        if n <= 0:
            raise ValueError("n must be positive")
        return int(self.uniform() * n)

    def spawn(self, index):
        return Rng(derive_seed(self.seed, index))

    def state_words(self):
        return tuple(int(v) for v in self._s)

    def set_state_words(self, words):
        if len(words) != 4:
            raise ValueError("xoshiro256++ state is four 64-bit words")
        self._s[:] = [int(w) & _M64 for w in words]


def gaussian_noise_map(rng, width, height):
    """imagecore.py:155-159: standard-normal map, row-major draw order."""
    if width <= 0 or height <= 0:
        raise ValueError("noise map dimensions must be positive")
    return rng.gaussians(width * height).reshape(height, width)


def gaussian_noise_map_f32(rng, width, height):
    """Same draws as gaussian_noise_map, rounded once to float32."""
    if width <= 0 or height <= 0:
        raise ValueError("noise map dimensions must be positive")
    return rng.gaussians_f32(width * height).reshape(height, width)


def gaussian_noise_map_device(rng, width, height, dtype=None, device=None):
    """gaussian_noise_map drawn on the GPU: (height, width) CUDA tensor
    (float32 by default, the fused kernel's input type)."""
    if width <= 0 or height <= 0:
        raise ValueError("noise map dimensions must be positive")
    return rng.gaussians_device(width * height, dtype=dtype, device=device).view(height, width)


def gaussian_maps_device(states, width, height, dtype=None, device=None):
    """Noise maps drawn on the GPU in one launch, map m from the stream state
    states[m] (4 words, as recorded with Rng.state_words() before the map's
    draws).  Returns a (len(states), height, width) CUDA tensor."""
    import torch
    _lib.require_cuda()
    n_maps = len(states)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    out = torch.empty((n_maps, height, width), dtype=dtype or torch.float32, device=dev)
    if n_maps:
        words = np.ascontiguousarray(np.array(states, dtype=np.uint64).reshape(n_maps, 4))
        with torch.cuda.device(dev):
            _lib.call("ht_rng_gaussian_maps_device", words.ctypes.data_as(C.c_void_p), n_maps,
                      C.c_int64(width * height), _lib.ptr(out), int(out.dtype == torch.float64),
                      _lib.stream_ptr())
    return out


def constant_image(gray, width, height):
    """imagecore.py:146-152."""
    if not 0.0 <= gray <= 1.0:
        raise ValueError("gray level outside [0, 1]")
    if width <= 0 or height <= 0:
        raise ValueError("image dimensions must be positive")
    return np.full((height, width), float(gray), dtype=np.float64)


def random_crop(rng, img, size):
    """imagecore.py:162-171: offsets drawn y then x."""
    h, w = img.shape
    if size <= 0:
        raise ValueError("crop size must be positive")
    if size > h or size > w:
        raise ValueError("crop larger than image")
    y = rng.randint(h - size + 1)
    x = rng.randint(w - size + 1)
    return img[y:y + size, x:x + size].copy()


def validate_contone(img):
    """imagecore.py:126-134."""
    img = np.asarray(img, dtype=np.float64)
    if img.ndim != 2:
        raise ValueError("contone image must be 2-D")
    if img.size == 0:
        raise ValueError("contone image must be non-empty")
    if not np.all(np.isfinite(img)) or img.min() < 0.0 or img.max() > 1.0:
        raise ValueError("contone values must lie in [0, 1]")
    return img
