"""Policy network, Adam and the cosine schedule -- htlab.nn drop-in (nn.py:28-199).

The object model mirrors the reference: `PolicyNetwork(channels, blocks,
in_channels)` with `.conv_in`, `.res[i].conv1/.conv2`, `.conv_out`, and
`params()` returning `Parameter`s whose `.value` / `.grad` are float64 numpy
arrays in the reference order (nn.py:118-122).  Those host arrays stay the
API surface; the network keeps a device copy (flat float64 + the packed
kernel layouts of ht_pack_params) that is re-synchronised whenever the host
values change, and device-side updates (GPU Adam in rl.train_step) are
written back to the host arrays.

Compute:
  forward / backward   training kernels (tcgen05 split-bf16 32->32 convs,
                       fp32 edge convs), activations kept on the device
                       between the two calls (nn.py:138-160)
  halftone_device      the fused tcgen05 kernel K1 (inference hot path)
  Conv2d / ResidualBlock .forward / .backward, and PolicyNetwork with
  in_channels != 2: the reference's layer-level API, float64 device convs
  (csrc/conv_f64.cu) chained on the device
"""

import math

import numpy as np

from . import _lib

PRESET_PAPER = (32, 16)
PRESET_MINI = (8, 2)


class Parameter:
    """nn.py:28-33."""
    __slots__ = ("value", "grad")

    def __init__(self, value):
        self.value = np.asarray(value, dtype=np.float64)
        self.grad = np.zeros_like(self.value)


def _torch():
    import torch
    return torch


_libc = None


def _memcmp(a, b, n):
    global _libc
    if _libc is None:
        import ctypes
        _libc = ctypes.CDLL(None)
        _libc.memcmp.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
        _libc.memcmp.restype = ctypes.c_int
    return _libc.memcmp(a, b, n)


def _dev64(a):
    """numpy -> float64 CUDA tensor (CUDA tensors pass through as float64)."""
    torch = _torch()
    _lib.require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


class Conv2d:
    """3x3, stride 1, zero-pad 1 cross-correlation (nn.py:36-80).  forward
    caches its input (on the device) for backward, which accumulates
    .weight.grad / .bias.grad and returns dL/dx; both run in float64 on the
    device (ht_conv3x3_f64, ht_conv3x3_f64_backward)."""

    def __init__(self, c_in, c_out):
        self.c_in, self.c_out = c_in, c_out
        self.weight = Parameter(np.zeros((c_out, c_in, 3, 3)))
        self.bias = Parameter(np.zeros(c_out))
        self._x = None

    def params(self):
        return [self.weight, self.bias]

    def forward(self, x):
        return self._fwd(_dev64(x)).cpu().numpy()

    def backward(self, dout):
        return self._bwd(_dev64(dout)).cpu().numpy()

    def _fwd(self, xd):
        torch = _torch()
        if xd.dim() != 4:
            raise ValueError("input must be (batch, channels, height, width)")
        b, c, hgt, wid = xd.shape
        if c != self.c_in:
            raise ValueError(f"expected {self.c_in} input channels, got {c}")
        w, bias = _dev64(self.weight.value), _dev64(self.bias.value)
        out = torch.empty((b, self.c_out, hgt, wid), dtype=torch.float64, device=xd.device)
        if out.numel():
            _lib.call("ht_conv3x3_f64", _lib.ptr(xd), b, c, self.c_out, hgt, wid, _lib.ptr(w),
                      _lib.ptr(bias), _lib.ptr(out), _lib.stream_ptr())
        self._x, self._w = xd, w
        return out

    def _bwd(self, dd):
        torch = _torch()
        if self._x is None:
            raise RuntimeError("backward() needs a preceding forward()")
        xd, w = self._x, self._w
        b, c, hgt, wid = xd.shape
        if tuple(dd.shape) != (b, self.c_out, hgt, wid):
            raise ValueError("dout shape does not match the last forward")
        dw = torch.zeros_like(w)
        db = torch.zeros(self.c_out, dtype=torch.float64, device=xd.device)
        dx = torch.empty_like(xd)
        if dx.numel():
            _lib.call("ht_conv3x3_f64_backward", _lib.ptr(xd), _lib.ptr(dd), b, c, self.c_out, hgt, wid,
                      _lib.ptr(w), _lib.ptr(dw), _lib.ptr(db), _lib.ptr(dx), _lib.stream_ptr())
        self.weight.grad += dw.cpu().numpy()
        self.bias.grad += db.cpu().numpy()
        return dx


class ResidualBlock:
    """x + conv2(relu(conv1(x))) (nn.py:83-103)."""

    def __init__(self, channels):
        self.conv1 = Conv2d(channels, channels)
        self.conv2 = Conv2d(channels, channels)
        self._mask = None

    def params(self):
        return self.conv1.params() + self.conv2.params()

    def forward(self, x):
        return self._fwd(_dev64(x)).cpu().numpy()

    def backward(self, dout):
        return self._bwd(_dev64(dout)).cpu().numpy()

    def _fwd(self, xd):
        y = self.conv1._fwd(xd)
        self._mask = y > 0
        return xd + self.conv2._fwd(y * self._mask)

    def _bwd(self, dd):
        dy = self.conv2._bwd(dd) * self._mask
        return dd + self.conv1._bwd(dy)


class PolicyNetwork:
    """Input conv (2 -> C), B residual blocks, output conv (C -> 1), sigmoid."""

    def __init__(self, channels=32, blocks=16, in_channels=2):
        if channels < 1 or blocks < 0 or in_channels < 1:
            raise ValueError("channels / in_channels must be positive and blocks non-negative")
        self.channels, self.blocks, self.in_channels = channels, blocks, in_channels
        self.conv_in = Conv2d(in_channels, channels)
        self.res = [ResidualBlock(channels) for _ in range(blocks)]
        self.conv_out = Conv2d(channels, 1)
        self._params = self.params()
        # the host .value arrays are views into one contiguous buffer, so the
        # per-use "did the host values change?" check is one memory compare
        # (a caller that rebinds a .value array gets the per-tensor check)
        self._host = np.zeros(sum(p.value.size for p in self._params))
        at = 0
        for p in self._params:
            n = p.value.size
            p.value = self._host[at:at + n].reshape(p.value.shape)
            at += n
        self._dev = None            # torch.device
        self._flat = None           # float64 device params
        self._packed = None         # uint8 device packed weights
        self._uploaded = None       # host flat copy matching the device
        self._cache = None          # training forward state (x, act, p, B, H, W)

    # ------------------------------------------------------------------ host API
    def params(self):
        out = self.conv_in.params()
        for blk in self.res:
            out += blk.params()
        return out + self.conv_out.params()

    def num_params(self):
        return sum(p.value.size for p in self._params)

    def init_params(self, rng, std=0.01):
        """nn.py:124-132: weights N(0, std^2) drawn in params() order, biases 0."""
        for p in self._params:
            if p.value.ndim > 1:
                p.value[...] = rng.gaussians(p.value.size).reshape(p.value.shape) * std
            else:
                p.value[...] = 0.0
            p.grad[...] = 0.0

    def zero_grad(self):
        for p in self._params:
            p.grad[...] = 0.0

    def _host_views_intact(self):
        base = self._host
        return all(p.value.base is base for p in self._params)

    def flat_values(self):
        if self._host_views_intact():
            return self._host.copy()
        return np.concatenate([p.value.ravel() for p in self._params])

    def set_flat_values(self, flat):
        at = 0
        for p in self._params:
            n = p.value.size
            p.value[...] = np.asarray(flat[at:at + n]).reshape(p.value.shape)
            at += n

    # ------------------------------------------------------------------ device state
    def to(self, device):
        torch = _torch()
        self._dev = torch.device(device)
        self._flat = None
        self._uploaded = None
        return self

    @property
    def device(self):
        if self._dev is None:
            _lib.require_cuda()
            torch = _torch()
            self._dev = torch.device("cuda", torch.cuda.current_device())
        return self._dev

    def _host_matches_upload(self):
        """Host .value arrays still equal the last uploaded / pulled values
        (one compare of the contiguous host buffer; per tensor, stopping at
        the first difference, if a caller rebound a .value array)."""
        up = self._uploaded
        if self._host_views_intact() and up.size == self._host.size:
            return _memcmp(self._host.ctypes.data, up.ctypes.data, self._host.nbytes) == 0
        at = 0
        for p in self._params:
            n = p.value.size
            if not np.array_equal(p.value.ravel(), up[at:at + n]):
                return False
            at += n
        return True

    def sync(self, force=False):
        """Upload + repack if the host parameter values changed; True if it
        uploaded."""
        torch = _torch()
        if self.in_channels != 2:
            raise ValueError("the fused / training kernels take the (contone, noise) pair: "
                             "in_channels must be 2 (other networks run forward/backward "
                             "layer by layer)")
        if (not force and self._flat is not None and self._uploaded is not None
                and self._host_matches_upload()):
            return False
        flat = self.flat_values()
        dev = self.device
        with torch.cuda.device(dev):
            if self._flat is None:
                self._flat = torch.empty(flat.size, dtype=torch.float64, device=dev)
                nbytes = _lib.out_i64("ht_packed_bytes", self.channels, self.blocks)
                self._packed = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            self._flat.copy_(torch.from_numpy(flat))
            self._repack()
        self._uploaded = flat
        return True

    def _repack(self):
        _lib.call("ht_pack_params", _lib.ptr(self._flat), self.channels, self.blocks,
                  _lib.ptr(self._packed), _lib.stream_ptr())
        # counts repacks (host uploads and device updates alike): captured
        # CUDA graphs that baked in the biases compare it (rl.HalftoneEngine)
        self.upload_generation = getattr(self, "upload_generation", 0) + 1

    def device_flat(self):
        self.sync()
        return self._flat

    def packed(self):
        self.sync()
        return self._packed

    def pull_from_device(self):
        """Device params (after a device-side update) -> host arrays (through
        a pinned staging buffer)."""
        self._pull_start()
        self._pull_finish()

    def _pull_start(self):
        """Repack the updated device parameters and start their copy to the
        pinned staging buffer (stream-ordered, no wait)."""
        torch = _torch()
        self._repack()
        if getattr(self, "_pin", None) is None or self._pin.numel() != self._flat.numel():
            self._pin = torch.empty(self._flat.numel(), dtype=torch.float64, pin_memory=True)
        self._pin.copy_(self._flat, non_blocking=True)
        self._pin_done = torch.cuda.Event()
        self._pin_done.record(torch.cuda.current_stream(self._flat.device))

    def _pull_finish(self):
        """Wait for the copy only (not for work queued after it) and update
        the host arrays."""
        self._pin_done.synchronize()
        flat = self._pin.numpy().copy()   # (the next pull rewrites the pinned buffer early)
        self.set_flat_values(flat)
        self._uploaded = flat

    # ------------------------------------------------------------------ compute
    def forward(self, x):
        """nn.py:138-150: probabilities (B, 1, H, W) float64; keeps the
        activations on the device for backward()."""
        torch = _torch()
        x = np.asarray(x, dtype=np.float64)
        if x.ndim != 4:
            raise ValueError("input must be (batch, channels, height, width)")
        if x.shape[1] != self.in_channels:
            raise ValueError(f"expected {self.in_channels} input channels, got {x.shape[1]}")
        if self.in_channels != 2:
            return self._module_forward(x)
        xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(self.device)
        p = self.forward_device(xd)
        return p.double().cpu().numpy()[:, None]

    def forward_device(self, x, flag=None, _sync=True):
        """Training forward on a device tensor x (B, 2, H, W) float32 ->
        p (B, H, W) float32 device tensor; activations cached.  Raises
        FloatingPointError on non-finite logits (nn.py:147-148) -- or, with
        flag (an int32 device tensor of B entries), ORs sample b's condition
        into flag[b] without waiting for the GPU, for the caller to check
        later."""
        torch = _torch()
        _lib.require_cuda()
        if _sync:
            self.sync()
        if x.dim() != 4 or x.shape[1] != self.in_channels:
            raise ValueError("input must be (batch, 2, height, width)")
        B, _, H, W = x.shape
        if B == 0 or H == 0 or W == 0:
            raise ValueError("input must be non-empty")
        x = x.contiguous().float()
        nbytes = _lib.out_i64("ht_train_act_bytes", self.channels, self.blocks, B, H, W)
        act = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
        p = torch.empty((B, H, W), dtype=torch.float32, device=x.device)
        self._cache = None
        if flag is None:
            _lib.call("ht_policy_forward_train", _lib.ptr(self._packed), self.channels, self.blocks,
                      _lib.ptr(x), B, H, W, _lib.ptr(act), _lib.ptr(p), _lib.stream_ptr())
        else:
            _lib.call("ht_policy_forward_train_async", _lib.ptr(self._packed), self.channels, self.blocks,
                      _lib.ptr(x), B, H, W, _lib.ptr(act), _lib.ptr(p), _lib.ptr(flag), _lib.stream_ptr())
        self._cache = (x, act, p, B, H, W)
        return p

    def _module_forward(self, x):
        """nn.py:138-150 layer by layer (float64 device convs): the path for
        networks whose input is not the (contone, noise) pair."""
        torch = _torch()
        y = self.conv_in._fwd(_dev64(x))
        for blk in self.res:
            y = blk._fwd(y)
        logits = self.conv_out._fwd(y)
        if not bool(torch.isfinite(logits).all()):
            raise FloatingPointError("non-finite logits")
        p = 1.0 / (1.0 + torch.exp(-logits))
        self._cache = ("module", p)
        return p.cpu().numpy()

    def _module_backward(self, dp):
        p = self._cache[1]
        dy = self.conv_out._bwd(_dev64(dp).reshape(p.shape) * p * (1.0 - p))
        for blk in reversed(self.res):
            dy = blk._bwd(dy)
        return self.conv_in._bwd(dy).cpu().numpy()

    def backward(self, dp):
        """nn.py:152-160: accumulate parameter grads into .grad, return dL/dx."""
        torch = _torch()
        if self._cache is not None and isinstance(self._cache[0], str):
            return self._module_backward(dp)
        if self._cache is None:
            raise RuntimeError("backward() needs a preceding forward()")
        x, act, p, B, H, W = self._cache
        dp = np.asarray(dp, dtype=np.float64).reshape(B, H, W)
        dpd = torch.from_numpy(np.ascontiguousarray(dp, dtype=np.float32)).to(x.device)
        grad = torch.zeros(self.num_params(), dtype=torch.float64, device=x.device)
        dx = torch.empty((B, 2, H, W), dtype=torch.float32, device=x.device)
        self.backward_device(dpd, grad, dx)
        g = grad.cpu().numpy()
        at = 0
        for prm in self._params:
            n = prm.value.size
            prm.grad += g[at:at + n].reshape(prm.value.shape)
            at += n
        return dx.double().cpu().numpy()

    def backward_device(self, dp, grad, dx=None):
        """Device backward: dp (B,H,W) fp32; grad (flat fp64) accumulated."""
        if self._cache is None:
            raise RuntimeError("backward() needs a preceding forward()")
        x, act, p, B, H, W = self._cache
        _lib.call("ht_policy_backward", _lib.ptr(self._packed), self.channels, self.blocks,
                  _lib.ptr(x), B, H, W, _lib.ptr(act), _lib.ptr(p), _lib.ptr(dp.contiguous()),
                  _lib.ptr(grad), _lib.ptr(dx), _lib.stream_ptr())

    def halftone_device(self, c, z, p_out=None, h_out=None, pbm_out=None, impl=None,
                        rows=None, workspace=None, check=False, stream=None, levels=2):
        """Fused inference forward + threshold (K1) on device tensors.

        c, z: (B, in_rows, W) float32 contone / noise (rows [in_row0,
        in_row0+in_rows) of images of height H: rows=(H, in_row0, out_row0,
        out_rows), default the whole image).  Outputs (B, out_rows, W):
        p_out float32, h_out uint8 (1 = white), pbm_out PBM P4 payload
        (B, out_rows, ceil(W/8)).  impl 0 = tcgen05 fused kernel (default for
        the paper architecture), 1 = fp32 SIMT cross-check path.  levels > 2:
        h_out receives the multitone level index (multitone.py:61-76)."""
        torch = _torch()
        self.sync()
        if c.dim() == 2:
            c, z = c[None], z[None]
        B, in_rows, W = c.shape
        if z.shape != c.shape:
            raise ValueError("contone and noise shapes differ")
        if rows is None:
            rows = (in_rows, 0, 0, in_rows)
        H, in_row0, out_row0, out_rows = rows
        if impl is None:
            impl = 0 if self.channels == 32 else 1
        nbytes = _lib.out_i64("ht_halftone_workspace_bytes", self.channels, self.blocks, B, H, W,
                              in_rows, out_rows, impl)
        if workspace is None or workspace.numel() < nbytes:
            workspace = torch.empty(nbytes, dtype=torch.uint8, device=c.device)
        sp = _lib.stream_ptr(stream)
        if levels == 2:
            _lib.call("ht_halftone", _lib.ptr(self._packed), self.channels, self.blocks,
                      _lib.ptr(c.contiguous()), _lib.ptr(z.contiguous()), B, H, W, in_row0,
                      in_rows, out_row0, out_rows, _lib.ptr(p_out), _lib.ptr(h_out),
                      _lib.ptr(pbm_out), _lib.ptr(workspace), nbytes, impl, sp)
        else:
            if pbm_out is not None:
                raise ValueError("the PBM payload is binary (levels = 2)")
            _lib.call("ht_multitone", _lib.ptr(self._packed), self.channels, self.blocks,
                      _lib.ptr(c.contiguous()), _lib.ptr(z.contiguous()), B, H, W, in_row0,
                      in_rows, out_row0, out_rows, int(levels), _lib.ptr(p_out), _lib.ptr(h_out),
                      _lib.ptr(workspace), nbytes, impl, sp)
        if check:
            try:
                _lib.call("ht_halftone_check", _lib.ptr(workspace), sp)
            except FloatingPointError:
                # K1 carries activations as fp16 MMA operands: a network whose
                # activations leave fp16's range (|x| > 65504, e.g. std-0.1
                # random init: ~1e5 after 16 blocks) overflows there while the
                # reference (fp64) stays finite -- and at that scale fp32 no
                # longer resolves p near the logit's zero crossings either.
                # Redo the batch in float64 on the device (the reference's
                # precision); it raises only if the logits are non-finite in
                # float64 too, exactly where the reference raises.
                self._halftone_f64(c, z, p_out, h_out, pbm_out, rows, levels, stream)
        return workspace

    def _halftone_f64(self, c, z, p_out, h_out, pbm_out, rows, levels, stream):
        """Float64 device forward + threshold epilogue, image by image, layer
        by layer (ht_conv3x3_f64; nothing cached for backward)."""
        torch = _torch()
        H, in_row0, out_row0, out_rows = rows
        lo = out_row0 - in_row0
        W = c.shape[-1]
        with torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.current_stream()):
            sp = _lib.stream_ptr()
            convs = [self.conv_in]
            for blk in self.res:
                convs += [blk.conv1, blk.conv2]
            convs.append(self.conv_out)
            wb = [(_dev64(cv.weight.value), _dev64(cv.bias.value)) for cv in convs]

            def conv(x, k):
                w, b = wb[k]
                out = torch.empty((1, w.shape[0], x.shape[2], W), dtype=torch.float64, device=x.device)
                _lib.call("ht_conv3x3_f64", _lib.ptr(x), 1, x.shape[1], w.shape[0], x.shape[2], W, _lib.ptr(w),
                          _lib.ptr(b), _lib.ptr(out), sp)
                return out

            for i in range(c.shape[0]):
                y = conv(torch.stack((c[i], z[i]))[None].double().contiguous(), 0)
                for k in range(self.blocks):
                    y = y + conv(torch.relu(conv(y, 1 + 2 * k)), 2 + 2 * k)
                logit = conv(y, len(convs) - 1)[0, 0, lo:lo + out_rows]
                if not bool(torch.isfinite(logit).all()):
                    raise FloatingPointError("non-finite logits")
                p = 1.0 / (1.0 + torch.exp(-logit))
                if p_out is not None:
                    p_out[i].copy_(p)
                if levels == 2:
                    h = (p >= 0.5).to(torch.uint8)
                else:   # multitone.quantize_multitone (multitone.py:61-67)
                    s = levels - 1
                    h = torch.clamp(torch.floor(p * s + 0.5), 0, s).to(torch.uint8)
                if h_out is not None:
                    h_out[i].copy_(h)
                if pbm_out is not None:   # PBM P4: bit 1 = black, MSB first (imagecore.py:289-297)
                    nb = (W + 7) // 8
                    bits = torch.zeros((out_rows, nb * 8), dtype=torch.uint8, device=p.device)
                    bits[:, :W] = 1 - h
                    wts = torch.tensor([128, 64, 32, 16, 8, 4, 2, 1], dtype=torch.uint8, device=p.device)
                    pbm_out[i].copy_((bits.view(out_rows, nb, 8) * wts).sum(-1).to(torch.uint8))


class Adam:
    """Bias-corrected Adam (nn.py:163-186), run on the device (K6)."""

    def __init__(self, params, beta1=0.9, beta2=0.999, eps=1e-8):
        self.params = list(params)
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.t = 0
        self.m = [np.zeros_like(p.value) for p in self.params]
        self.v = [np.zeros_like(p.value) for p in self.params]
        self._dm = self._dv = None

    def _device_state(self, dev):
        torch = _torch()
        if self._dm is None:
            self._dm = torch.from_numpy(np.concatenate([m.ravel() for m in self.m])).to(dev)
            self._dv = torch.from_numpy(np.concatenate([v.ravel() for v in self.v])).to(dev)
        return self._dm, self._dv

    def step_device(self, flat, grad, lr):
        """One Adam step on device tensors (flat params, flat grads, fp64)."""
        m, v = self._device_state(flat.device)
        self.t += 1
        _lib.call("ht_adam_step", _lib.ptr(flat), _lib.ptr(grad), _lib.ptr(m), _lib.ptr(v),
                  flat.numel(), self.t, float(lr), self.beta1, self.beta2, self.eps,
                  _lib.stream_ptr())

    def invalidate_device_state(self):
        """Host m/v were rewritten (checkpoint load): re-upload on next step."""
        self._dm = self._dv = None

    def pull_state(self):
        """Device moments -> the host lists (checkpointing / inspection)."""
        if self._dm is None:
            return
        mh, vh = self._dm.cpu().numpy(), self._dv.cpu().numpy()
        at = 0
        for m, v in zip(self.m, self.v):
            n = m.size
            m[...] = mh[at:at + n].reshape(m.shape)
            v[...] = vh[at:at + n].reshape(v.shape)
            at += n

    def step(self, lr):
        """nn.py:175-186 on the parameters' host .value/.grad (uploads, runs
        the device kernel, writes back)."""
        torch = _torch()
        _lib.require_cuda()
        dev = torch.device("cuda", torch.cuda.current_device())
        flat = torch.from_numpy(np.concatenate([p.value.ravel() for p in self.params])).to(dev)
        grad = torch.from_numpy(np.concatenate([p.grad.ravel() for p in self.params])).to(dev)
        self.step_device(flat, grad, lr)
        fh = flat.cpu().numpy()
        at = 0
        for p in self.params:
            n = p.value.size
            p.value[...] = fh[at:at + n].reshape(p.value.shape)
            at += n
        self.pull_state()


def cosine_lr(t, total, lr_start=3e-4, lr_end=1e-5):
    """nn.py:189-199."""
    if total <= 0:
        raise ValueError("total steps must be positive")
    if t >= total:
        return lr_end
    if t < 0:
        raise ValueError("step must be non-negative")
    return float(lr_end + 0.5 * (lr_start - lr_end) * (1.0 + math.cos(math.pi * t / total)))


# checkpoint format (nn.py:200-300), re-exported so `from ...nn import
# load_checkpoint` works as it does for the reference
from .checkpoint import (CheckpointError, load_checkpoint, network_from_checkpoint,  # noqa: E402
                         read_checkpoint, save_checkpoint)
