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
from dataclasses import dataclass

import numpy as np

from . import _lib
from .hvs import HvsConfig
from .imagecore import Rng, gaussian_noise_map, random_crop
from .metrics import MetricConfig, reward, reward_le_device
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
    contone/noise: (H, W) or batched (B, H, W)."""
    torch = _torch()
    _lib.require_cuda()
    c = np.asarray(contone)
    z = np.asarray(noise)
    if c.shape != z.shape:
        raise ValueError("contone and noise shapes differ")
    if c.ndim not in (2, 3) or c.size == 0:
        raise ValueError("contone must be a non-empty (H, W) or (B, H, W) array")
    single = c.ndim == 2
    if single:
        c, z = c[None], z[None]
    dev = net.device
    cd = torch.from_numpy(np.ascontiguousarray(c, dtype=np.float32)).to(dev)
    zd = torch.from_numpy(np.ascontiguousarray(z, dtype=np.float32)).to(dev)
    p = torch.empty(cd.shape, dtype=torch.float32, device=dev)
    h = torch.empty(cd.shape, dtype=torch.uint8, device=dev)
    net.halftone_device(cd, zd, p_out=p, h_out=h, impl=impl, check=True)
    hp, pp = h.cpu().numpy().astype(np.float64), p.cpu().numpy().astype(np.float64)
    return (hp[0], pp[0]) if single else (hp, pp)


def infer_halftone(net, c, rng, impl=None):
    """rl.py:306-311: draw z = gaussian_noise_map(rng, W, H), run the policy,
    threshold at 0.5 (ties go white).  Returns (h, p)."""
    c = np.asarray(c, dtype=np.float64)
    z = gaussian_noise_map(rng, c.shape[1], c.shape[0])
    return halftone(net, c, z, impl=impl)


# ---------------------------------------------------------------------------
# sampling / estimators (binary policy)

@dataclass
class EpisodeSample:
    """rl.py:72-82 (binary: floor 0, ceil 1, p_ceil = p)."""
    c: np.ndarray
    z: np.ndarray
    p: np.ndarray
    m: np.ndarray
    level_count: int
    ctx: object


def make_sample(p, c, z, rng, cfg=None, level_count=2):
    """rl.py:85-93 for L=2: m = (u < p) with row-major uniforms, reward
    context built on the GPU."""
    if level_count != 2:
        raise NotImplementedError("multitone (L>2) is outside the GPU hot path")
    p = np.asarray(p, dtype=np.float64)
    u = rng.uniforms(p.size).reshape(p.shape)
    m = (u < p).astype(np.float64)
    ctx = reward(m, c, cfg or MetricConfig(), region="full")
    return EpisodeSample(c=c, z=z, p=p, m=m, level_count=2, ctx=ctx)


def le_signal(sample):
    """rl.py:106-109: dL/dp_a = -(R(up) - R(down)) / delta, delta = 1."""
    from .metrics import delta_map
    d_other = delta_map(sample.ctx, 1.0 - sample.m)
    sign = np.where(sample.m == 1.0, -1.0, 1.0)
    return -(sign * d_other)


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
        if self.estimator != "local_expectation" or self.levels != 2:
            raise NotImplementedError("the GPU training path implements the binary "
                                      "local_expectation estimator (rl.py:106-109)")


from .parallel import allreduce_sum_, shard_range  # noqa: E402
from .parallel import dist_info as _dist_info  # noqa: E402


def draw_batch(dataset, cfg, rng):
    """Host RNG draws of rl.py:242-245 (image pick, crop y, crop x, noise)."""
    size = cfg.crop_size
    crops, noises = [], []
    for _ in range(cfg.batch_size):
        img = dataset[rng.randint(len(dataset))]
        crops.append(random_crop(rng, img, size))
        noises.append(gaussian_noise_map(rng, size, size))
    return crops, noises


def train_step(net, adam, dataset, cfg, rng, t, group=None, signal_override=None):
    """One optimisation step (rl.py:232-278); returns the diagnostics row.

    group: torch.distributed process group for data parallelism (default:
    the world group when initialised).  signal_override: test hook -- a
    callable(sample_index, m) -> LE signal (float64 (H,W)) replacing the GPU
    estimator, used by staged parity tests."""
    torch = _torch()
    _lib.require_cuda()
    rank, world = _dist_info(group)
    dev = net.device
    size, bs = cfg.crop_size, cfg.batch_size
    mcfg = cfg.metric_config()
    crops, noises = draw_batch(dataset, cfg, rng)
    lo, hi = shard_range(bs, rank, world)
    grad = torch.zeros(net.num_params(), dtype=torch.float64, device=dev)
    stats = torch.zeros(3, dtype=torch.float64, device=dev)  # reward, bin_gap, l_as sums
    p = None
    if hi > lo:
        x = np.stack([np.stack((crops[i], noises[i])) for i in range(lo, hi)])
        p = net.forward_device(torch.from_numpy(x.astype(np.float32)).to(dev))
    # action uniforms for every sample, in order (rl.py:249 -> rl.py:68)
    us = [rng.uniforms(size * size).reshape(size, size) for _ in range(bs)]
    if hi > lo:
        ud = torch.from_numpy(np.stack(us[lo:hi])).to(dev)
        cd = torch.from_numpy(np.stack(crops[lo:hi]).astype(np.float32)).to(dev)
        m, sig, rew = reward_le_device(p, ud, cd, mcfg, scale=1.0 / bs)
        if signal_override is not None:
            mh = m.double().cpu().numpy()
            sig = torch.from_numpy(np.stack([signal_override(lo + i, mh[i]) / bs
                                             for i in range(hi - lo)]).astype(np.float32)).to(dev)
        net.backward_device(sig, grad)
        stats[0] += rew.sum()
        _lib.call("ht_bin_gap_sum", _lib.ptr(p), p.numel(), _lib.ptr(stats[1:2]),
                  _lib.stream_ptr())
    run_aniso = cfg.w_a != 0.0 and (cfg.levels == 2 or cfg.multitone_anisotropy)
    if run_aniso:
        ba = cfg.anisotropy_batch_size or bs
        grays = [rng.uniform() for _ in range(ba)]
        znoise = [gaussian_noise_map(rng, size, size) for _ in range(ba)]
        glo, ghi = shard_range(ba, rank, world)
        if ghi > glo:
            xg = np.stack([np.stack((np.full((size, size), grays[i]), znoise[i]))
                           for i in range(glo, ghi)])
            pg = net.forward_device(torch.from_numpy(xg.astype(np.float32)).to(dev))
            part = _part_cache(size)
            loss, dpg = anisotropy_device(pg, part, scale=cfg.w_a / ba)
            net.backward_device(dpg, grad)
            stats[2] += loss.sum()
    allreduce_sum_(grad, stats, group=group)   # the step's one exchange
    st = stats.cpu().numpy()
    mean_reward = float(st[0] / bs)
    bin_gap = float(st[1] / (bs * size * size))
    l_as = float(st[2] / (cfg.anisotropy_batch_size or bs)) if run_aniso else math.nan
    lr = cosine_lr(t, cfg.iterations, cfg.lr_start, cfg.lr_end)
    net.sync()
    adam.step_device(net._flat, grad, lr)
    net.pull_from_device()
    net._last_grad = grad
    return {"iteration": t, "reward": mean_reward, "l_as": l_as, "bin_gap": bin_gap, "lr": lr}


_parts = {}


def _part_cache(size):
    if size not in _parts:
        _parts[size] = ring_partition((size, size))
    return _parts[size]


def train_loop(cfg, dataset, resume_path=None, on_iteration=None, group=None):
    """rl.py:281-303.  resume_path restores parameters, Adam state, the
    iteration counter and the RNG state words, so a split run reproduces an
    unsplit one."""
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
    for t in range(start, cfg.iterations):
        diag = train_step(net, adam, dataset, cfg, rng, t, group=group)
        if on_iteration is not None:
            on_iteration(t, diag, net, adam, rng)
    adam.pull_state()
    return net, adam, rng


# ---------------------------------------------------------------------------
# batched end-to-end engine (host buffers in, halftones out)

class HalftoneEngine:
    """Reusable batched halftoner for a fixed (B, H, W): host contone/noise
    (float32, ideally pinned) in, uint8 halftones (1 = white) or PBM P4
    payloads out.  The batch is split into `chunks` groups of images that
    flow through H2D -> fused K1 kernel -> D2H on alternating CUDA streams, so
    copies of one chunk overlap the kernel of another.  Every call performs
    the full host->device->host round trip."""

    def __init__(self, net, B, H, W, chunks=4, output="h", impl=None):
        torch = _torch()
        _lib.require_cuda()
        if output not in ("h", "pbm", "p"):
            raise ValueError("output must be 'h', 'pbm' or 'p'")
        self.net, self.B, self.H, self.W = net, B, H, W
        self.output = output
        self.impl = impl
        chunks = max(1, min(chunks, B))
        bounds = np.linspace(0, B, chunks + 1).round().astype(int)
        self.groups = [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        dev = net.device
        self.dev = dev
        self.streams = [torch.cuda.Stream(dev) for _ in range(2)]
        self.c = torch.empty((B, H, W), dtype=torch.float32, device=dev)
        self.z = torch.empty((B, H, W), dtype=torch.float32, device=dev)
        if output == "pbm":
            self.out = torch.empty((B, H, (W + 7) // 8), dtype=torch.uint8, device=dev)
        elif output == "h":
            self.out = torch.empty((B, H, W), dtype=torch.uint8, device=dev)
        else:
            self.out = torch.empty((B, H, W), dtype=torch.float32, device=dev)
        self.ws = [None, None]
        net.sync()

    def out_shape(self):
        return tuple(self.out.shape)

    def h2d_bytes(self):
        return 2 * self.B * self.H * self.W * 4

    def d2h_bytes(self):
        return self.out.numel() * self.out.element_size()

    def __call__(self, c_host, z_host, out_host):
        """c_host, z_host: (B,H,W) float32 CPU tensors (pinned for async
        copies); out_host: CPU tensor shaped out_shape()."""
        torch = _torch()
        cur = torch.cuda.current_stream(self.dev)
        for k, (a, b) in enumerate(self.groups):
            s = self.streams[k % 2]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                self.c[a:b].copy_(c_host[a:b], non_blocking=True)
                self.z[a:b].copy_(z_host[a:b], non_blocking=True)
                kw = {"h_out" if self.output == "h" else
                      ("pbm_out" if self.output == "pbm" else "p_out"): self.out[a:b]}
                self.ws[k % 2] = self.net.halftone_device(
                    self.c[a:b], self.z[a:b], impl=self.impl, workspace=self.ws[k % 2],
                    stream=s, **kw)
                out_host[a:b].copy_(self.out[a:b], non_blocking=True)
        for s in self.streams:
            cur.wait_stream(s)
        cur.synchronize()
        return out_host


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
