"""Inference and training entry points -- htlab.rl drop-in (rl.py:40-311).

infer_halftone / halftone run the fused tensor-core forward K1.  train_step
follows the reference's Algorithm-1 step (rl.py:232-278) with the same host
RNG draw order, running the forward, the LE estimator (K3/K4), the
anisotropy loss (K5), the backward and Adam (K6) on the GPU.  With
torch.distributed initialised it is data parallel: every rank consumes the
full host RNG stream, computes its shard of the batch, and the gradient and
diagnostics are all-reduced once per step (signals are pre-scaled by the
GLOBAL 1/batch_size and w_a/ba, rl.py:253, 272).
"""

import math
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .hvs import HvsConfig
from .imagecore import (Rng, gaussian_maps_device, gaussian_noise_map, gaussian_noise_map_device,
                        random_crop)
from .metrics import MetricConfig, reinforce_signal_device, reward, reward_signal_device
from .nn import Adam, PolicyNetwork, cosine_lr, load_checkpoint
from .spectral import anisotropy_device, ring_partition

ESTIMATORS = ("reinforce", "reinforce_meanbaseline", "coma", "local_expectation")


def _torch():
    import torch
    return torch


# ---------------------------------------------------------------------------
# inference

def halftone(net, contone, noise, impl=None):
    """Noise-explicit factoring of rl.infer_halftone (rl.py:309-311):
    returns (h, p) float64 arrays; h = (p >= 0.5) with ties -> 1 (white).
    contone/noise: (H, W) or batched (B, H, W).  Host batches of >= 4
    images are pipelined in chunks (_halftone_host_batch)."""
    _lib.require_cuda()
    net.device
    if _host_batch(contone) and _host_batch(noise) and np.shape(contone) == np.shape(noise) \
            and len(np.shape(contone)) == 3 and np.shape(contone)[0] >= _PIPE_MIN_BATCH \
            and math.prod(np.shape(contone)) > 0:
        with _pipe_lock:
            return _halftone_host_batch(net, contone, noise, impl)
    return _halftone_oneshot(net, contone, noise, impl)


def _halftone_oneshot(net, contone, noise, impl):
    torch = _torch()
    dev = net.device

    def as_dev(a):        # numpy / host -> device float32 (CUDA tensors pass through)
        if isinstance(a, torch.Tensor):
            return a.to(device=dev, dtype=torch.float32).contiguous()
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)

    cd, zd = as_dev(contone), as_dev(noise)
    if cd.shape != zd.shape:
        raise ValueError("contone and noise shapes differ")
    if cd.dim() not in (2, 3) or cd.numel() == 0:
        raise ValueError("contone must be a non-empty (H, W) or (B, H, W) array")
    single = cd.dim() == 2
    if single:
        cd, zd = cd[None], zd[None]
    p = torch.empty(cd.shape, dtype=torch.float32, device=dev)
    h = torch.empty(cd.shape, dtype=torch.uint8, device=dev)
    net.halftone_device(cd, zd, p_out=p, h_out=h, impl=impl, check=True)
    # float64 results (the reference's types) widened on the device and read
    # back into page-locked host arrays (torch's host allocator caches the
    # blocks; each call returns fresh arrays)
    hp = torch.empty(h.shape, dtype=torch.float64, pin_memory=True)
    pp = torch.empty(p.shape, dtype=torch.float64, pin_memory=True)
    hp.copy_(h.double(), non_blocking=True)
    pp.copy_(p.double(), non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    hp, pp = hp.numpy(), pp.numpy()
    return (hp[0], pp[0]) if single else (hp, pp)


_PIPE_MIN_BATCH = 4      # host batches of at least this many images are pipelined
_PIPE_CHUNKS = 8
_pipe_cache = {}
_pipe_lock = threading.Lock()      # the cached staging buffers serve one call at a time


def _host_batch(a):
    if isinstance(a, np.ndarray):
        return a.dtype.kind in "fiub"
    torch = _torch()
    return isinstance(a, torch.Tensor) and a.device.type == "cpu"


def _halftone_host_batch(net, contone, noise, impl):
    """halftone() for a host batch: the images flow in chunks through
    host staging (float32, page-locked) -> H2D -> fused K1 -> float64 widening
    -> D2H into the page-locked result arrays, on two alternating streams, so
    one chunk's copies and host-side conversion overlap another chunk's
    kernel.  Same results as the one-shot path (K1 is bitwise batch
    invariant); a chunk whose fp16 operands overflowed is redone in float64
    like halftone_device(check=True)."""
    torch = _torch()
    dev = net.device
    B, H, W = (int(x) for x in np.shape(contone))
    m = -(-B // _PIPE_CHUNKS)
    bounds = list(range(0, B, m)) + [B]
    groups = list(zip(bounds[:-1], bounds[1:]))
    key = (str(dev), m, H, W)
    res = _pipe_cache.get(key)
    if res is None:
        _pipe_cache.clear()              # one shape's buffers at a time
        res = {
            "streams": [torch.cuda.Stream(dev, priority=-1) for _ in range(2)],
            "stage": [torch.empty((2, m, H, W), dtype=torch.float32, pin_memory=True) for _ in range(2)],
            "inp": [torch.empty((2, m, H, W), dtype=torch.float32, device=dev) for _ in range(2)],
            "p": [torch.empty((m, H, W), dtype=torch.float32, device=dev) for _ in range(2)],
            "h": [torch.empty((m, H, W), dtype=torch.uint8, device=dev) for _ in range(2)],
            "p64": [torch.empty((m, H, W), dtype=torch.float64, device=dev) for _ in range(2)],
            "h64": [torch.empty((m, H, W), dtype=torch.float64, device=dev) for _ in range(2)],
            "ws": [None, None],
            "done": [None, None],
        }
        _pipe_cache[key] = res
    hp = torch.empty((B, H, W), dtype=torch.float64, pin_memory=True)
    pp = torch.empty((B, H, W), dtype=torch.float64, pin_memory=True)

    def host(a, lo, hi):
        if isinstance(a, np.ndarray):
            a = a[lo:hi]
            if any(s < 0 for s in a.strides) or a.dtype.kind != "f":
                a = a.astype(a.dtype if a.dtype.kind == "f" else np.float64, order="C", copy=True)
            return torch.from_numpy(a)
        return a[lo:hi]

    cur = torch.cuda.current_stream(dev)
    owner = [None, None]                 # chunk index last run on each slot
    redo = []

    def retire(s):
        """Wait for slot s's chunk and check its non-finite flag."""
        if res["done"][s] is None:
            return
        res["done"][s].synchronize()
        k = owner[s]
        try:
            _lib.call("ht_halftone_check", _lib.ptr(res["ws"][s]), _lib.stream_ptr(res["streams"][s]))
        except FloatingPointError:
            redo.append(groups[k])
        res["done"][s] = None

    for k, (a, b) in enumerate(groups):
        s, n = k % 2, b - a
        retire(s)                        # staging / device buffers of chunk k-2 are free
        st = res["stage"][s]
        st[0, :n].copy_(host(contone, a, b))
        st[1, :n].copy_(host(noise, a, b))
        S = res["streams"][s]
        S.wait_stream(cur)
        with torch.cuda.stream(S):
            inp = res["inp"][s]
            inp[:, :n].copy_(st[:, :n], non_blocking=True)
            res["ws"][s] = net.halftone_device(inp[0, :n], inp[1, :n], p_out=res["p"][s][:n],
                                               h_out=res["h"][s][:n], impl=impl, workspace=res["ws"][s],
                                               stream=S)
            res["p64"][s][:n].copy_(res["p"][s][:n])
            res["h64"][s][:n].copy_(res["h"][s][:n])
            pp[a:b].copy_(res["p64"][s][:n], non_blocking=True)
            hp[a:b].copy_(res["h64"][s][:n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(S)
        res["done"][s], owner[s] = ev, k
    for s in range(2):
        retire(s)
    for s in range(2):
        cur.wait_stream(res["streams"][s])
    hp, pp = hp.numpy(), pp.numpy()
    for a, b in redo:                    # rare: fp16 overflow -> float64 redo
        h1, p1 = _halftone_oneshot(net, host(contone, a, b), host(noise, a, b), impl)
        hp[a:b], pp[a:b] = h1, p1
    return hp, pp


def infer_halftone(net, c, rng, impl=None):
    """rl.py:306-311: draw z = gaussian_noise_map(rng, W, H), run the policy,
    threshold at 0.5 (ties go white).  Returns (h, p).  The noise map is the
    same Rng stream drawn on the GPU (imagecore.gaussian_noise_map_device)."""
    c = np.asarray(c, dtype=np.float64)
    if c.ndim != 2 or c.size == 0:
        raise ValueError("contone must be a non-empty (H, W) array")
    net.device                                   # CUDA required before drawing
    z = gaussian_noise_map_device(rng, c.shape[1], c.shape[0], device=net.device)
    return halftone(net, c, z, impl=impl)


# ---------------------------------------------------------------------------
# sampling / estimators (host API of the reference; rewards on the GPU)

PROB_FLOOR = 1e-7   # rl.py:34, clamp before the log-derivative division


def _cast_two_point(values, level_count):
    """rl.py:40-57: the two lattice levels around each value (levels
    i/(L-1)) and the upper-level mass; on-lattice values collapse."""
    v = np.asarray(values, dtype=np.float64)
    if np.any(v < 0.0) or np.any(v > 1.0):
        raise ValueError("values outside [0, 1]")
    steps = level_count - 1
    scaled = v * steps
    idx = np.floor(scaled)
    frac = scaled - idx
    floor_vals = idx / steps
    ceil_vals = np.where(frac == 0.0, floor_vals, np.minimum(idx + 1.0, steps) / steps)
    return floor_vals, ceil_vals, frac


def sample_actions(p, rng):
    """rl.py:60-64: independent Bernoulli(p), one uniform per pixel, row-major."""
    p = np.asarray(p, dtype=np.float64)
    return (rng.uniforms(p.size).reshape(p.shape) < p).astype(np.float64)


def _sample_two_point(floor_vals, ceil_vals, p_ceil, rng):
    """rl.py:67-69."""
    u = rng.uniforms(p_ceil.size).reshape(p_ceil.shape)
    return np.where(u < p_ceil, ceil_vals, floor_vals)


@dataclass
class EpisodeSample:
    """rl.py:72-82."""
    c: np.ndarray
    z: np.ndarray
    p: np.ndarray
    m: np.ndarray
    floor_vals: np.ndarray
    ceil_vals: np.ndarray
    p_ceil: np.ndarray
    level_count: int
    ctx: object


def make_sample(p, c, z, rng, cfg=None, level_count=2):
    """rl.py:85-93: sample the cast policy, reward context built on the GPU."""
    floor_vals, ceil_vals, p_ceil = _cast_two_point(p, level_count)
    m = _sample_two_point(floor_vals, ceil_vals, p_ceil, rng)
    ctx = reward(m, c, cfg or MetricConfig(), region="full")
    return EpisodeSample(c=c, z=z, p=np.asarray(p, dtype=np.float64), m=m, floor_vals=floor_vals,
                         ceil_vals=ceil_vals, p_ceil=p_ceil, level_count=level_count, ctx=ctx)


def exact_gradient_oracle(p, c, cfg=None, region="full", level_count=2):
    """rl.py:139-164: d E[R] / d p by enumerating every joint action map
    (each pixel at the lower or upper point of its two-point cast), at most 20
    pixels.  The 2^n rewards are evaluated on the GPU in batched launches of
    the reward kernel (maps passed as given action maps); the weighting is
    host arithmetic.  For L > 2, p is the value map and upper-level mass moves
    at (L - 1) per unit value."""
    torch = _torch()
    _lib.require_cuda()
    p = np.asarray(p, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    n = p.size
    if n > 20:
        raise ValueError("oracle enumeration limited to 20 pixels")
    if c.shape != p.shape:
        raise ValueError("p and c must have the same shape")
    if region != "full":
        if region == "valid":
            raise NotImplementedError("region='valid' is an evaluation metric outside the GPU hot "
                                      "path (use region='full')")
        raise ValueError(f"unknown region {region!r}")
    cfg = cfg or MetricConfig()
    floor_vals, ceil_vals, p_ceil = _cast_two_point(p, level_count)
    fv, cv, q = floor_vals.ravel(), ceil_vals.ravel(), p_ceil.ravel()
    dev = torch.device("cuda", torch.cuda.current_device())
    total = 1 << n
    grad = np.zeros(n)
    chunk = 1 << 16
    cd = None
    for b0 in range(0, total, chunk):
        b1 = min(total, b0 + chunk)
        up = ((np.arange(b0, b1)[:, None] >> np.arange(n)[None, :]) & 1).astype(bool)
        m = np.where(up, cv[None], fv[None]).reshape((b1 - b0,) + p.shape)
        if cd is None or cd.shape[0] != b1 - b0:
            cd = torch.from_numpy(np.broadcast_to(c, m.shape).astype(np.float32).copy()).to(dev)
        md = torch.from_numpy(m.astype(np.float32)).to(dev)
        _, _, rew = reward_signal_device(md, None, cd, cfg, want_signal=False, levels=level_count)
        r = rew.cpu().numpy()
        prob_each = np.where(up, q[None], 1.0 - q[None])
        sign = np.where(up, 1.0, -1.0)
        for a in range(n):
            rest = np.prod(np.delete(prob_each, a, axis=1), axis=1)
            grad[a] += float(np.sum(r * sign[:, a] * rest))
    return (grad * (level_count - 1)).reshape(p.shape)


def _two_point_diff(sample):
    """rl.py:96-103: R(upper) - R(lower) per pixel (0 where collapsed)."""
    from .metrics import delta_map
    at_ceil = sample.m == sample.ceil_vals
    other = np.where(at_ceil, sample.floor_vals, sample.ceil_vals)
    return np.where(at_ceil, -1.0, 1.0) * delta_map(sample.ctx, other)


def le_signal(sample):
    """rl.py:106-109: dL/dp_a = -(R(up) - R(down)) / delta."""
    return -_two_point_diff(sample) * (sample.level_count - 1)


def _dlogpi(p, h):
    p = np.clip(p, PROB_FLOOR, 1.0 - PROB_FLOOR)
    return np.where(h == 1.0, 1.0 / p, -1.0 / (1.0 - p))


def coma_signal(sample):
    """rl.py:117-129: counterfactual-baseline gradient (binary only)."""
    from .metrics import delta_map
    if sample.level_count != 2:
        raise ValueError("coma_signal requires a binary policy")
    h = sample.m
    r_cur = sample.ctx.reward
    r_flip = r_cur + delta_map(sample.ctx, 1.0 - h)
    r_up = np.where(h == 1.0, r_cur, r_flip)
    r_down = np.where(h == 0.0, r_cur, r_flip)
    p = np.clip(sample.p, PROB_FLOOR, 1.0 - PROB_FLOOR)
    return -_dlogpi(sample.p, h) * (r_cur - (p * r_up + (1.0 - p) * r_down))


def reinforce_signal(sample, baseline=0.0):
    """rl.py:132-136: score-function gradient, optional scalar baseline."""
    if sample.level_count != 2:
        raise ValueError("reinforce_signal requires a binary policy")
    return -_dlogpi(sample.p, sample.m) * (sample.ctx.reward - baseline)


def _signals_for_batch(samples, estimator):
    """rl.py:219-229 (host API; train_step runs the device kernels)."""
    if estimator == "local_expectation":
        return [le_signal(s) for s in samples]
    if estimator == "coma":
        return [coma_signal(s) for s in samples]
    if estimator == "reinforce":
        return [reinforce_signal(s) for s in samples]
    if estimator == "reinforce_meanbaseline":
        mean_r = float(np.mean([s.ctx.reward for s in samples]))
        return [reinforce_signal(s, baseline=mean_r) for s in samples]
    raise ValueError(f"unknown estimator {estimator!r}")


# ---------------------------------------------------------------------------
# training

@dataclass(frozen=True)
class TrainConfig:
    """rl.py:170-216."""
    dataset_dir: str = ""
    out_dir: str = ""
    iterations: int = 200000
    batch_size: int = 64
    crop_size: int = 64
    channels: int = 32
    blocks: int = 16
    w_s: float = 0.06
    w_a: float = 0.002
    lr_start: float = 3e-4
    lr_end: float = 1e-5
    estimator: str = "local_expectation"
    seed: int = 0
    levels: int = 2
    anisotropy_batch_size: int = 0
    multitone_anisotropy: bool = False
    log_every: int = 100
    checkpoint_every: int = 0
    hvs_model: str = "nasanen"
    hvs_size: int = 11
    hvs_scale: float = 2000.0
    hvs_sigma: float = 2.0

    def metric_config(self):
        return MetricConfig(w_s=self.w_s, hvs=HvsConfig(
            model=self.hvs_model, size=self.hvs_size, scale=self.hvs_scale,
            sigma=self.hvs_sigma))

    def validate(self):
        if self.estimator not in ESTIMATORS:
            raise ValueError(f"unknown estimator {self.estimator!r}")
        if self.levels < 2:
            raise ValueError("levels must be at least 2")
        if self.levels > 2 and self.estimator != "local_expectation":
            raise ValueError("multitone training supports only local_expectation")
        if self.batch_size < 1 or self.crop_size < 1 or self.iterations < 1:
            raise ValueError("batch size, crop size and iterations must be positive")
        if self.channels < 1 or self.blocks < 0:
            raise ValueError("channels must be positive and blocks non-negative")
        if self.log_every < 1 or self.checkpoint_every < 0:
            raise ValueError("log_every must be positive and checkpoint_every non-negative")


from .parallel import allreduce_sum_, shard_range  # noqa: E402
from .parallel import dist_info as _dist_info  # noqa: E402


def draw_batch(dataset, cfg, rng, device=None, keep=None):
    """RNG draws of rl.py:242-245 in reference order (image pick, crop y,
    crop x, noise map).  Host mode returns (crops, noise maps).  With
    `device`, the noise maps of the samples in `keep` (a range: this rank's
    shard) are drawn on the GPU in one launch from the stream states they
    start at, the others only advance the stream (jump-ahead); returns
    (crops, (len(keep), size, size) float32 CUDA tensor)."""
    size = cfg.crop_size
    draws = 2 * ((size * size + 1) // 2)          # one gaussian_noise_map
    crops, noises, starts = [], [], []
    for i in range(cfg.batch_size):
        img = dataset[rng.randint(len(dataset))]
        crops.append(random_crop(rng, img, size))
        if device is None:
            noises.append(gaussian_noise_map(rng, size, size))
        else:
            if keep is None or i in keep:
                starts.append(rng.state_words())
            rng.jump(draws)
    if device is None:
        return crops, noises
    return crops, gaussian_maps_device(starts, size, size, device=device)


def _prepare_step(dataset, cfg, rng, dev, rank, world):
    """Every RNG draw of one train_step, in the reference's order (crops and
    noise maps, action uniforms, gray levels and their noise maps), and this
    rank's inputs on the device.  Nothing here depends on the network."""
    torch = _torch()
    size, bs = cfg.crop_size, cfg.batch_size
    lo, hi = shard_range(bs, rank, world)
    start = rng.state_words()
    crops, noises = draw_batch(dataset, cfg, rng, device=dev, keep=range(lo, hi))
    # RNG states at the reference's two forwards: a non-finite logit is
    # detected once per step (no wait per forward) and raised with the
    # stream where the reference's forward (nn.py:147-148) would have raised
    rng_at_fwd = [rng.state_words(), None]
    # action uniforms for every sample, in order (rl.py:249 -> rl.py:68): this
    # rank's shard is one contiguous stretch of the stream, drawn on the GPU
    # in one launch; the other ranks' stretches are skipped (jump-ahead).  No
    # draw depends on the forward, so all of the step's draws come first.
    n = size * size
    rng.jump(lo * n)
    ud = rng.uniforms_device((hi - lo) * n, device=dev).view(hi - lo, size, size) if hi > lo else None
    rng.jump((bs - hi) * n)
    run_aniso = cfg.w_a != 0.0 and (cfg.levels == 2 or cfg.multitone_anisotropy)
    nm, ng, ba = hi - lo, 0, cfg.anisotropy_batch_size or bs
    inputs, cd, ready = [], None, None
    if nm:
        # the crops' H2D on a copy stream: a prefetch enqueued mid-step must
        # not sit in the compute stream between this step's kernels; users
        # of the batch wait for it (_materialize)
        host = torch.from_numpy(np.stack(crops[lo:hi]).astype(np.float32)).pin_memory()
        cs = _copy_stream(dev)
        with torch.cuda.stream(cs):
            cd = host.to(dev, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(cs)
        cd.record_stream(torch.cuda.current_stream(dev))
        inputs.append((cd, noises))
    if run_aniso:
        grays = [rng.uniform() for _ in range(ba)]
        glo, ghi = shard_range(ba, rank, world)
        # the gray images' noise maps follow each other in the stream: this
        # rank's maps in one launch from their start states, the rest skipped
        draws = 2 * ((size * size + 1) // 2)
        starts = []
        for i in range(ba):
            if glo <= i < ghi:
                starts.append(rng.state_words())
            rng.jump(draws)
        rng_at_fwd[1] = rng.state_words()
        ng = ghi - glo
        if ng:
            znoise = gaussian_maps_device(starts, size, size, device=dev)
            gd = torch.tensor([grays[i] for i in range(glo, ghi)], dtype=torch.float32)
            gd = gd.pin_memory().to(dev, non_blocking=True)[:, None, None].expand(-1, size, size)
            inputs.append(torch.stack((gd, znoise), dim=1))
    return {"start": start, "end": rng.state_words(), "rng_at_fwd": rng_at_fwd, "lo": lo, "hi": hi,
            "nm": nm, "ng": ng, "ba": ba, "cd": cd, "ud": ud, "inputs": inputs, "ready": ready}


_copy_streams = {}


def _copy_stream(dev):
    torch = _torch()
    key = str(dev)
    if key not in _copy_streams:
        _copy_streams[key] = torch.cuda.Stream(dev)
    return _copy_streams[key]


def _materialize(prep):
    """Order the current stream after the prepared batch's H2D and build the
    MARL input planes (contone, noise) on it (once)."""
    torch = _torch()
    if prep.get("ready") is not None:
        torch.cuda.current_stream(prep["cd"].device).wait_event(prep["ready"])
        prep["ready"] = None
    if prep["inputs"] and isinstance(prep["inputs"][0], tuple):
        cd, noises = prep["inputs"][0]
        prep["inputs"][0] = torch.stack((cd, noises), dim=1)
    return prep


# the next step's draws and inputs, prepared while the GPU runs this step
# (one entry; used only if the caller's RNG is where this step left it)
_next_step = {}


def _dataset_key(dataset):
    # identity of the image list and of each array's buffer (an image
    # replaced between steps invalidates the prefetched batch)
    return (id(dataset), len(dataset),
            tuple((id(a), a.__array_interface__["data"][0] if hasattr(a, "__array_interface__") else 0)
                  for a in dataset))


def reset_prefetch():
    """Drop the prefetched next-step batch and any queued speculative forward
    (frees their device buffers; the next train_step draws afresh)."""
    _next_step.clear()


def _take_prepared(dataset, cfg, rng, dev, rank, world):
    key = (_dataset_key(dataset), cfg, str(dev), rank, world)
    prep = _next_step.pop("prep", None)
    if prep is not None and _next_step.pop("key", None) == key and prep["start"] == rng.state_words():
        rng.set_state_words(prep["end"])
        return prep
    _next_step.clear()
    return _prepare_step(dataset, cfg, rng, dev, rank, world)


def _speculate_forward(net, dev):
    """Queue the next step's forward (its prepared inputs, the parameters
    Adam just produced) behind this step's work, so the GPU does not idle
    while the host finishes this step and starts the next; the next step uses
    it only if it takes the same prepared batch and uploads no parameters."""
    torch = _torch()
    prep = _next_step.get("prep")
    if prep is None or not prep["inputs"]:
        return
    _materialize(prep)
    # this step's backward has consumed the training cache: free it before the
    # speculative forward allocates its own (no doubled activation memory)
    net._cache = None
    ins = prep["inputs"]
    x = ins[0] if len(ins) == 1 else torch.cat(ins)
    flag = torch.zeros(max(prep["nm"] + prep["ng"], 1), dtype=torch.int32, device=dev)
    # (no host-parameter check: this step changed none; the device copy is
    # Adam's update, which the pull now under way brings to the host)
    p = net.forward_device(x.contiguous(), flag=flag, _sync=False)
    _next_step["spec"] = {"prep": prep, "net": net, "p": p, "flag": flag, "cache": net._cache}
    net._cache = None


def _prefetch_next(dataset, cfg, rng, dev, rank, world):
    ahead = Rng(0)
    ahead.set_state_words(rng.state_words())
    _next_step["prep"] = _prepare_step(dataset, cfg, ahead, dev, rank, world)
    _next_step["key"] = (_dataset_key(dataset), cfg, str(dev), rank, world)


def train_step(net, adam, dataset, cfg, rng, t, group=None, signal_override=None, prefetch=True):
    """One optimisation step (rl.py:232-278); returns the diagnostics row.

    group: torch.distributed process group for data parallelism (default:
    the world group when initialised).  signal_override: test hook -- a
    callable(sample_index, m) -> LE signal (float64 (H,W)) replacing the GPU
    estimator, used by staged parity tests.  prefetch: draw the next step's
    batch (from a copy of the RNG stream) while the GPU runs this one; the
    next call uses it only if its RNG is exactly where this step left it and
    the dataset holds the same arrays (pass prefetch=False if image contents
    are edited in place between steps: the batch is then always drawn
    afresh, and nothing is prepared ahead)."""
    torch = _torch()
    _lib.require_cuda()
    if not prefetch:
        _next_step.clear()
    rank, world = _dist_info(group)
    dev = net.device
    bs = cfg.batch_size
    mcfg = cfg.metric_config()
    prep = _materialize(_take_prepared(dataset, cfg, rng, dev, rank, world))
    spec = _next_step.pop("spec", None)
    lo, nm, ng, ba = prep["lo"], prep["nm"], prep["ng"], prep["ba"]
    cd, ud, inputs, rng_at_fwd = prep["cd"], prep["ud"], prep["inputs"], prep["rng_at_fwd"]
    size = cfg.crop_size
    run_aniso = cfg.w_a != 0.0 and (cfg.levels == 2 or cfg.multitone_anisotropy)
    grad = torch.zeros(net.num_params(), dtype=torch.float64, device=dev)
    # reward, bin_gap, l_as sums, non-finite flags of the MARL and of the
    # gray forward (one all-reduce, one read-back per step)
    stats = torch.zeros(5, dtype=torch.float64, device=dev)
    # one forward + one backward over this rank's MARL crops and gray images
    # (the reference's two forwards, batched: samples are independent and the
    # parameters do not change in between); sample b's non-finite flag
    nonfinite = torch.zeros(max(nm + ng, 1), dtype=torch.int32, device=dev)
    if nm + ng:
        # the previous step may already have run this forward (same prepared
        # inputs, same parameters: nothing was uploaded since)
        uploaded = net.sync()
        if spec is not None and spec["prep"] is prep and spec["net"] is net and not uploaded:
            p_all, nonfinite, net._cache = spec["p"], spec["flag"], spec["cache"]
        else:
            x = inputs[0] if len(inputs) == 1 else torch.cat(inputs)
            p_all = net.forward_device(x.contiguous(), flag=nonfinite, _sync=False)
    dps = []
    reinforce = cfg.estimator in ("reinforce", "reinforce_meanbaseline")
    if nm:
        p = p_all[:nm]
        if not reinforce:
            m, sig, rew = reward_signal_device(p, ud, cd, mcfg, scale=1.0 / bs, levels=cfg.levels,
                                               estimator=cfg.estimator)
        else:
            m, _, rew = reward_signal_device(p, ud, cd, mcfg, want_signal=False)
    if cfg.estimator == "reinforce_meanbaseline":
        # baseline = mean reward of the GLOBAL batch: one extra scalar
        # all-reduce, joined by every rank (also those without samples)
        rsum = rew.sum().reshape(1) if nm else torch.zeros(1, dtype=torch.float64, device=dev)
        allreduce_sum_(rsum, group=group)
        baseline = float(rsum.item()) / bs
    else:
        baseline = 0.0
    if nm:
        if reinforce:
            sig = reinforce_signal_device(p, m, rew, baseline, scale=1.0 / bs)
        if signal_override is not None:
            mh = m.double().cpu().numpy()
            sig = torch.from_numpy(np.stack([signal_override(lo + i, mh[i]) / bs
                                             for i in range(nm)]).astype(np.float32)).to(dev)
        dps.append(sig)
        stats[0] += rew.sum()
        _lib.call("ht_bin_gap_sum", _lib.ptr(p), p.numel(), _lib.ptr(stats[1:2]),
                  _lib.stream_ptr())
    if ng:
        part = _part_cache(size)
        loss, dpg = anisotropy_device(p_all[nm:], part, scale=cfg.w_a / ba)
        dps.append(dpg)
        stats[2] += loss.sum()
    if dps:
        net.backward_device(dps[0] if len(dps) == 1 else torch.cat(dps), grad)
    if prefetch:
        _prefetch_next(dataset, cfg, rng, dev, rank, world)
    if nm:
        stats[3] = nonfinite[:nm].amax().double()
    if ng:
        stats[4] = nonfinite[nm:nm + ng].amax().double()
    # the step's one exchange: gradients in fp32 (1.19 MB),
    # the five statistics in fp64
    g_ex = grad.float() if world > 1 else grad
    allreduce_sum_(g_ex, stats, group=group)
    if g_ex is not grad:
        grad.copy_(g_ex)
    st = stats.cpu().numpy()
    if st[3] != 0.0 or st[4] != 0.0:
        # first forward with a non-finite logit on any rank (the MARL forward
        # comes first); parameters and Adam state untouched, RNG as the
        # reference leaves it when it raises
        which = 0 if st[3] != 0.0 else 1
        rng.set_state_words(rng_at_fwd[which])
        raise FloatingPointError("non-finite logits")
    mean_reward = float(st[0] / bs)
    bin_gap = float(st[1] / (bs * size * size))
    l_as = float(st[2] / (cfg.anisotropy_batch_size or bs)) if run_aniso else math.nan
    lr = cosine_lr(t, cfg.iterations, cfg.lr_start, cfg.lr_end)
    # (the device parameters are current: forward_device synced them and no
    # host code of this step changes them)
    adam.step_device(net._flat, grad, lr)
    net._pull_start()
    if prefetch:
        _speculate_forward(net, dev)
    net._pull_finish()
    net._last_grad = grad
    return {"iteration": t, "reward": mean_reward, "l_as": l_as, "bin_gap": bin_gap, "lr": lr}


_parts = {}


def _part_cache(size):
    if size not in _parts:
        _parts[size] = ring_partition((size, size))
    return _parts[size]


def train_loop(cfg, dataset, resume_path=None, on_iteration=None, group=None, prefetch=True):
    """rl.py:281-303.  resume_path restores parameters, Adam state, the
    iteration counter and the RNG state words, so a split run reproduces an
    unsplit one.  prefetch=False: every step draws its batch afresh (for
    on_iteration callbacks that edit dataset arrays in place)."""
    cfg.validate()
    if not dataset:
        raise ValueError("dataset is empty")
    rng = Rng(cfg.seed)
    net = PolicyNetwork(channels=cfg.channels, blocks=cfg.blocks)
    adam = Adam(net.params())
    net.init_params(rng)
    start = 0
    if resume_path is not None:
        meta = load_checkpoint(resume_path, net, adam)
        start = meta["iteration"]
        rng.set_state_words(meta["rng_state"])
    try:
        for t in range(start, cfg.iterations):
            diag = train_step(net, adam, dataset, cfg, rng, t, group=group, prefetch=prefetch)
            if on_iteration is not None:
                on_iteration(t, diag, net, adam, rng)
    finally:
        reset_prefetch()
    adam.pull_state()
    return net, adam, rng


# ---------------------------------------------------------------------------
# batched end-to-end engine (host buffers in, halftones out)

class HalftoneEngine:
    """Reusable batched halftoner for a fixed (B, H, W): host contone/noise
    (float32, ideally pinned) in, uint8 halftones (1 = white) or PBM P4
    payloads out.  A call (or submit) performs the full host->device->host
    round trip of one batch.  Within a batch, `chunks` groups of images flow
    through H2D -> fused K1 kernel -> D2H on alternating CUDA streams, so
    copies of one chunk overlap the kernel of another (lowest latency for a
    single call).  For throughput, submit()/wait() stream batches through
    `depth` sets of device buffers: batch i+1's copies overlap batch i's
    kernels, and one chunk per batch keeps the launches few."""

    def __init__(self, net, B, H, W, chunks=4, output="h", impl=None, depth=2, graph=False):
        torch = _torch()
        _lib.require_cuda()
        if output not in ("h", "pbm", "p"):
            raise ValueError("output must be 'h', 'pbm' or 'p'")
        self.net, self.B, self.H, self.W = net, B, H, W
        self.output = output
        self.impl = impl
        chunks = max(1, min(chunks, B))
        # a small first chunk (its H2D is the one copy nothing overlaps), the
        # rest split evenly so the fused kernel keeps long strips per CTA
        first = max(1, -(-B // 16)) if chunks > 1 else B
        rest = np.linspace(first, B, chunks).round().astype(int)
        bounds = [0] + [int(x) for x in rest]
        self.groups = [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        dev = net.device
        self.dev = dev
        if depth < 1:
            raise ValueError("depth must be >= 1")
        # `depth` sets of device buffers + streams: submitted batches rotate
        # through them, so batch i+1's copies and kernels run beside batch i's
        # (a set is reused, in its streams' order, by batch i+depth).  The
        # forward/copy streams run at high priority: the block scheduler then
        # prefers the fused kernel's CTAs over the side stream's noise blocks
        self._sets = []
        for _ in range(depth):
            if output == "pbm":
                out = torch.empty((B, H, (W + 7) // 8), dtype=torch.uint8, device=dev)
            elif output == "h":
                out = torch.empty((B, H, W), dtype=torch.uint8, device=dev)
            else:
                out = torch.empty((B, H, W), dtype=torch.float32, device=dev)
            self._sets.append({
                "streams": [torch.cuda.Stream(dev, priority=-1) for _ in range(2)],
                "noise": torch.cuda.Stream(dev, priority=0),
                "c": torch.empty((B, H, W), dtype=torch.float32, device=dev),
                "z": torch.empty((B, H, W), dtype=torch.float32, device=dev),
                "out": out, "ws": [None, None]})
        self._next = 0
        self.out = self._sets[0]["out"]
        # graph=True (latency mode): a call with pinned host tensors replays
        # one CUDA graph of H2D -> fused forward -> D2H (+ the non-finite
        # flag's 4 bytes), captured per (host buffers, parameter upload)
        self.graph = graph
        self._graph = None
        self._graph_key = None
        self._flag_host = torch.zeros(1, dtype=torch.int32, pin_memory=True) if graph else None
        net.sync()

    def out_shape(self):
        return tuple(self.out.shape)

    def h2d_bytes(self, device_noise=False):
        return (1 if device_noise else 2) * self.B * self.H * self.W * 4

    def d2h_bytes(self):
        return self.out.numel() * self.out.element_size()

    def __call__(self, c_host, z_host, out_host):
        """c_host: (B,H,W) float32 CPU tensor (pinned for async copies);
        z_host: the (B,H,W) float32 noise as a CPU tensor, or an Rng -- then
        image i's noise map is gaussian_noise_map(rng, W, H) drawn on the GPU
        in image order, as B calls of rl.infer_halftone would draw it
        (rl.py:306-311); out_host: CPU tensor shaped out_shape().  Returns
        out_host once it holds the result."""
        if (self.graph and not isinstance(z_host, Rng) and c_host.is_pinned()
                and z_host.is_pinned() and out_host.is_pinned()):
            return self._graph_call(c_host, z_host, out_host)
        self.wait(self.submit(c_host, z_host, out_host))
        return out_host

    def _graph_call(self, c_host, z_host, out_host):
        """One batch as a single CUDA-graph replay on the current stream (the
        nine K1 passes keep their programmatic-dependent edges inside the
        graph); the host waits once and reads the flag copied by the graph."""
        torch = _torch()
        self.net.sync()
        # the graph bakes in the host buffers and the per-pass biases (kernel
        # parameters): any other buffer or a newer parameter upload recaptures
        key = (c_host.data_ptr(), z_host.data_ptr(), out_host.data_ptr(),
               getattr(self.net, "upload_generation", 0))
        if self._graph is None or self._graph_key != key:
            self._capture(c_host, z_host, out_host, key)
        cur = torch.cuda.current_stream(self.dev)
        self._graph.replay()
        cur.synchronize()
        if int(self._flag_host[0]) != 0:
            raise FloatingPointError("non-finite logits in the fused forward (use impl=1 or "
                                     "rl.halftone for networks that leave fp16's range)")
        return out_host

    def _capture(self, c_host, z_host, out_host, key):
        torch = _torch()
        st = self._sets[0]
        cbuf, zbuf, obuf = st["c"], st["z"], st["out"]
        kw = {"h_out" if self.output == "h" else
              ("pbm_out" if self.output == "pbm" else "p_out"): obuf}
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        # uncaptured run first: allocates the workspace, sets the kernels'
        # shared-memory attributes and refreshes the library's host bias copy
        with torch.cuda.stream(s):
            cbuf.copy_(c_host, non_blocking=True)
            zbuf.copy_(z_host, non_blocking=True)
            ws = self.net.halftone_device(cbuf, zbuf, impl=self.impl, workspace=st["ws"][0],
                                          stream=s, **kw)
        s.synchronize()
        st["ws"][0] = ws
        self._graph = None
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            cbuf.copy_(c_host, non_blocking=True)
            zbuf.copy_(z_host, non_blocking=True)
            self.net.halftone_device(cbuf, zbuf, impl=self.impl, workspace=ws, stream=s, **kw)
            out_host.copy_(obuf, non_blocking=True)
            self._flag_host.copy_(ws[:4].view(torch.int32), non_blocking=True)
        self._graph, self._graph_key = g, key

    def submit(self, c_host, z_host, out_host):
        """Enqueue one batch (H2D -> fused forward -> D2H) without waiting and
        return a ticket for wait().  Back-to-back submits pipeline: the next
        batch's first copies and kernel overlap this batch's tail (the device
        buffers are reused in stream order).  c_host / z_host must stay
        unchanged and out_host unread until the ticket is waited on; give
        batches in flight distinct out_host buffers."""
        torch = _torch()
        cur = torch.cuda.current_stream(self.dev)
        device_noise = isinstance(z_host, Rng)
        st = self._sets[self._next % len(self._sets)]
        self._next += 1
        streams, zbuf, cbuf, obuf, ws = st["streams"], st["z"], st["c"], st["out"], st["ws"]
        ready = [None] * len(self.groups)
        if device_noise:
            # every chunk's noise maps, drawn in image order from the stream;
            # chunk 0 on its own stream, the rest on a side stream so they
            # run beside chunk 0's forward (the fused kernel leaves the FP64
            # pipe and 1/8 of the register file free)
            n = self.H * self.W
            for k, (a, b) in enumerate(self.groups):
                ns = streams[0] if k == 0 else st["noise"]
                ns.wait_stream(cur)
                # the previous batch on this buffer set read this chunk's z
                ns.wait_stream(streams[k % 2])
                with torch.cuda.stream(ns):
                    if n % 2 == 0:     # maps of even size are back-to-back in the stream
                        z_host.gaussians_device((b - a) * n, out=zbuf[a:b].view(-1))
                    else:              # odd size: each map burns one draw
                        for i in range(a, b):
                            z_host.gaussians_device(n, out=zbuf[i].view(-1))
                    ready[k] = torch.cuda.Event()
                    ready[k].record(ns)
        for k, (a, b) in enumerate(self.groups):
            s = streams[k % 2]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                cbuf[a:b].copy_(c_host[a:b], non_blocking=True)
                if device_noise:
                    s.wait_event(ready[k])
                else:
                    zbuf[a:b].copy_(z_host[a:b], non_blocking=True)
                kw = {"h_out" if self.output == "h" else
                      ("pbm_out" if self.output == "pbm" else "p_out"): obuf[a:b]}
                ws[k % 2] = self.net.halftone_device(
                    cbuf[a:b], zbuf[a:b], impl=self.impl, workspace=ws[k % 2],
                    stream=s, **kw)
                out_host[a:b].copy_(obuf[a:b], non_blocking=True)
        ticket = []
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            ticket.append(e)
        return (ticket, st)

    def wait(self, ticket):
        """Block until a submitted batch's result is in its out_host; later
        work on the current stream is ordered after it.  Raises
        FloatingPointError if the fused kernel saw a non-finite logit (for a
        network whose activations leave fp16's range, use impl=1 or
        rl.halftone, which redoes such batches on the fp32 path)."""
        torch = _torch()
        cur = torch.cuda.current_stream(self.dev)
        events, st = ticket
        for e in events:
            cur.wait_event(e)
            e.synchronize()
        for k, ws in enumerate(st["ws"]):
            if ws is not None:
                _lib.call("ht_halftone_check", _lib.ptr(ws), _lib.stream_ptr(st["streams"][k % 2]))


def halftone_batch(net, contones, noises, output="h", chunks=4):
    """Batched public entry: (B,H,W) contones + noise maps (numpy or CPU
    tensors) -> uint8 halftones (1 = white) or PBM payloads (numpy)."""
    torch = _torch()
    c = torch.as_tensor(np.ascontiguousarray(contones, dtype=np.float32)).pin_memory()
    z = torch.as_tensor(np.ascontiguousarray(noises, dtype=np.float32)).pin_memory()
    if c.dim() == 2:
        c, z = c[None], z[None]
    eng = HalftoneEngine(net, *c.shape, chunks=chunks, output=output)
    out = torch.empty(eng.out_shape(), dtype=eng.out.dtype).pin_memory()
    return eng(c, z, out).numpy()
