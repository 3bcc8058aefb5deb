"""Benchmark of the halftoning hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under `python -m torch.distributed.run --nproc-per-node N` (one rank per GPU,
NCCL, rendezvous on 127.0.0.1); under torchrun it checks WORLD_SIZE == N.

Headline workload = BASELINE config 2: 64 seeded synthetic 512x512 contones
(ramp + 8 Gaussian blobs + 2 rectangles, 10% with step edges) with N(0,1)
noise maps from the reference RNG; the reference's default policy CNN (C=32,
16 blocks, 296,833 params) with seeded random-init weights (std 0.01).  One
step = fused forward + sigmoid/threshold (K1) over the 64 images, sharded
64/N per rank (strong scaling, no collective on the data path).

value    = device-resident throughput (inputs in HBM), CUDA events on the
           launch stream, max over ranks.
e2e      = same metric through rl.HalftoneEngine (public API): pinned host
           contone+noise -> H2D -> K1 -> D2H uint8 halftones, every step,
           batches streamed two deep (submit/wait), max over ranks.
roofline = the dominant kernel (the 2-residual-block pass, 7 of 9 launches):
           algorithmic FLOPs per launch / its mean CUDA-event duration,
           against the measured burst bf16/fp16 dense peak (MEASURED_PEAKS).
cpu_baseline = the REAL reference (htlab installed under baseline/_ref:
           PolicyNetwork.forward + p >= 0.5, nn.py:138-150, rl.py:310-311) on
           all host cores, single-threaded BLAS per worker process, one
           256x256 tile of a config-2 image per core (bounded sample).
configs  = the other BASELINE configs, each with its own clocks: cfg1
           latency, cfg3 flat-gray sweep incl. spectra, cfg4 print page in
           row strips, cfg5 training step (data parallel at N > 1).

--impl reference: the reference arm (rank 0 only; other ranks exit 0): the
same htlab forward + threshold on the host cores, same metric / config.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_PATH = os.path.join(ROOT, "baseline", "_ref")

FLOP_PER_PX = 2 * 9 * (2 * 32 + 2 * 16 * 32 * 32 + 32)   # 591,552
FLOP_PER_PX_MIDPASS = 2 * 9 * 4 * 32 * 32               # 4 convs of 32->32 per pass
MID_TAG = 20                                             # pass tag: no conv_in, 2 blocks, no conv_out
METRIC = "halftone Mpixel/s (CNN inference+binarize) at 1/2/4/8 B200; % of roofline"
B2, S2 = 64, 512                                         # BASELINE config 2
REF_TILE = 256                                           # reference sample tile edge


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["bf16_tflops"], d["bf16_tflops_sustained"], d["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def headline_config(world):
    return {"workload": f"BASELINE config 2: {B2} x {S2}x{S2} contones, policy CNN C=32 B=16",
            "global_batch": B2, "image": [S2, S2],
            "parallelism": f"images sharded {B2}/{world} per rank, {world} rank(s), no collective",
            "l2": "inputs (134 MB) + pass buffers larger than L2 (126 MB)"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during a region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.15)          # first sample lands inside the region
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower() == "active":
                    reasons.add(nm)
        pw = [float(r[3]) for r in self.rows if len(r) > 3 and r[3].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "power_w": round(float(np.median(pw)), 1) if pw else None,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ inputs
def noise_seed(seed):
    return seed * 1_000_003


def make_inputs(lo, hi, H, W, seed, device):
    """Images [lo, hi) of the config-2 batch: contones from the BASELINE
    generator (image i uses seed (seed, i)); noise maps drawn in image order
    from one reference-RNG stream (as B calls of rl.infer_halftone would), on
    the GPU, starting at image lo (jump-ahead over the earlier maps)."""
    from paper_2304_12152_b200 import synth
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_device
    c = np.stack([synth.contone(H, W, seed=noise_seed(seed) + i, blobs=8, rects=2,
                                step_edge=i < round(0.1 * B2)) for i in range(lo, hi)])
    rng = Rng(noise_seed(seed))
    rng.jump(lo * 2 * ((H * W + 1) // 2))
    z = np.stack([gaussian_noise_map_device(rng, W, H, device=device).cpu().numpy()
                  for _ in range(lo, hi)])
    return c, z


def make_net(std=0.01):
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = PolicyNetwork(32, 16)
    net.init_params(Rng(0), std=std)
    return net


def l2_flush(dev, buf=[]):
    """Write 256 MB (> 126 MB L2) so the next kernel starts from cold L2."""
    import torch
    if not buf:
        buf.append(torch.empty(64 << 20, dtype=torch.float32, device=dev))
    buf[0].fill_(1.0)


# ------------------------------------------------------------------ reference (CPU)
def _ref_worker_init(ref_path):
    # single-threaded BLAS is already in the environment this process was
    # spawned with; the reference is imported from its install only
    sys.path.insert(0, ref_path)
    global _REF_NET
    from htlab import nn as hnn
    from htlab.imagecore import Rng as HRng
    _REF_NET = hnn.PolicyNetwork()              # PRESET_PAPER: C=32, 16 blocks
    _REF_NET.init_params(HRng(0), std=0.01)


def _ref_task(job):
    """One tile through the reference's own path: forward + threshold
    (nn.py:138-150, rl.py:310-311)."""
    c, z = job
    t0 = time.perf_counter()
    p = _REF_NET.forward(np.stack((c, z))[None])[0, 0]
    h = p >= 0.5
    return c.size, time.perf_counter() - t0, int(h.sum())


def _port_worker_init(_):
    global _REF_NET
    from oracle import htoracle as O
    _REF_NET = O.init_params(O.Rng(0), 32, 16, 2, 0.01)


def _port_task(job):
    from oracle import htoracle as O
    c, z = job
    t0 = time.perf_counter()
    _, p = O.halftone(_REF_NET, c, z)
    return c.size, time.perf_counter() - t0, int((p >= 0.5).sum())


_ref_images = {}


def ref_tiles(n, tile):
    """n tiles (tile x tile, float64 copies of the fp32 inputs) of the
    config-2 images: tile k is quadrant k % 4 of image k // 4 (images in
    batch order).  Noise maps come from the reference's own Rng stream (its
    gaussian_noise_map, imagecore.py:155-159) when the reference is
    installed, else the oracle port's (bit-identical, pinned by tests)."""
    from paper_2304_12152_b200 import synth
    if os.path.isdir(os.path.join(REF_PATH, "htlab")):
        sys.path.insert(0, REF_PATH)
        from htlab.imagecore import Rng as R, gaussian_noise_map as gmap
    else:
        from oracle.htoracle import Rng as R, gaussian_noise_map as gmap
    n_img = (n + 3) // 4
    if len(_ref_images) < n_img:
        rng = R(noise_seed(2))
        for i in range(n_img):
            c = synth.contone(S2, S2, seed=noise_seed(2) + i, blobs=8, rects=2,
                              step_edge=i < round(0.1 * B2))
            _ref_images[i] = (c, gmap(rng, S2, S2).astype(np.float32))
    jobs = []
    for i in range(n_img):
        c, z = _ref_images[i]
        for q in range(4):
            if len(jobs) == n:
                break
            y0, x0 = (q // 2) * (S2 - tile), (q % 2) * (S2 - tile)
            jobs.append((c[y0:y0 + tile, x0:x0 + tile].astype(np.float64),
                         z[y0:y0 + tile, x0:x0 + tile].astype(np.float64)))
    return jobs


class RefPool:
    """Worker processes running the reference forward, one BLAS thread each
    (the limits are exported before the workers are spawned, so OpenBLAS
    starts single-threaded in every worker)."""

    def __init__(self, cores):
        import multiprocessing as mp
        for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[k] = "1"
        self.kind = "reference" if os.path.isdir(os.path.join(REF_PATH, "htlab")) else "port"
        init, self.task = ((_ref_worker_init, _ref_task) if self.kind == "reference"
                           else (_port_worker_init, _port_task))
        self.cores = cores
        self.pool = mp.get_context("spawn").Pool(cores, initializer=init, initargs=(REF_PATH,))

    def run(self, jobs):
        t0 = time.perf_counter()
        res = self.pool.map(self.task, jobs, chunksize=1)
        return sum(r[0] for r in res), time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self, tile, n):
        what = ("htlab PolicyNetwork.forward + (p >= 0.5) from baseline/_ref (the unmodified "
                "reference)" if self.kind == "reference" else
                "oracle/htoracle.py port of nn.py:138-150 + rl.py:311 (reference not installed)")
        return (f"{n} tiles of {tile}x{tile} px per step (quadrants of config-2 images), one per "
                f"worker process, {self.cores} processes x 1 BLAS thread: {what}")


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ distributed
def dist_setup(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    return rank, world, local


def relaunch(args):
    """--gpus N > 1 outside torchrun: one rank per GPU under torch.distributed.run."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


class Dist:
    def __init__(self, rank, world, dev):
        self.rank, self.world, self.dev = rank, world, dev

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max(self, *vals):
        import torch
        t = torch.tensor(vals, dtype=torch.float64, device=self.dev)
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t.cpu()]


def timed(D, fn, steps, warmup, stream=None):
    """Device time of `steps` calls of fn (CUDA events on the launch stream,
    barrier + synchronize on both sides), max over ranks; returns ms/step."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    D.barrier()
    st = stream or torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    D.barrier()
    return D.max(e0.elapsed_time(e1) / steps)[0]


# ------------------------------------------------------------------ sub-configs
def bench_cfg1(D, net, reps):
    """Config 1: one 256x256 contone, batch 1 -- latency.  Device-resident
    (inputs in HBM, L2 flushed before each run) and end to end through
    rl.HalftoneEngine (pinned host in, uint8 out), median of `reps`."""
    import torch
    from paper_2304_12152_b200 import rl, synth
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_device
    dev = D.dev
    c = torch.from_numpy(synth.contone(256, 256, seed=0, blobs=8, rects=2)).to(dev)[None]
    z = gaussian_noise_map_device(Rng(0), 256, 256, device=dev)[None]
    h = torch.empty((1, 256, 256), dtype=torch.uint8, device=dev)
    ws = net.halftone_device(c, z, h_out=h, check=True)
    st = torch.cuda.current_stream()
    dev_ms = []
    with ClockSampler(dev.index) as clk:
        for _ in range(reps + 3):
            l2_flush(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            net.halftone_device(c, z, h_out=h, workspace=ws)
            e1.record(st)
            torch.cuda.synchronize()
            dev_ms.append(e0.elapsed_time(e1))
        ch, zh = c.cpu().pin_memory(), z.cpu().pin_memory()
        e2e = {}
        for mode in ("graph", "streams"):
            eng = rl.HalftoneEngine(net, 1, 256, 256, chunks=1, output="h", depth=1,
                                    graph=mode == "graph")
            oh = torch.empty(eng.out_shape(), dtype=torch.uint8).pin_memory()
            e2e[mode] = []
            for _ in range(reps + 3):
                l2_flush(dev)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                eng(ch, zh, oh)
                e2e[mode].append((time.perf_counter() - t0) * 1e3)
            assert torch.equal(oh, h.cpu()), f"cfg1: e2e ({mode}) output differs from the device path"
    e2e_ms = e2e["graph"]
    return {"workload": "BASELINE config 1: 1 x 256x256 contone (seed 0), batch 1",
            "latency_ms": round(float(np.median(dev_ms[3:])), 4),
            "latency_ms_e2e": round(float(np.median(e2e_ms[3:])), 4),
            "latency_ms_e2e_streams": round(float(np.median(e2e["streams"][3:])), 4),
            "unit": "ms (median, L2 flushed before each run)", "reps": reps,
            "e2e_api": "rl.HalftoneEngine(B=1, graph=True) pinned host fp32 in -> uint8 out, one CUDA-graph replay (H2D, 9 K1 passes, D2H, flag), wall clock; _streams = the same engine without the graph",
            "clocks": clk.summary()}


def bench_cfg3(D, net, steps, warmup):
    """Config 3: 256 flat-gray 256x256 images g = k/255 with their own noise
    maps -> forward + binarize, then per-level RAPSD + anisotropy of the
    halftone (K7) and the anisotropy loss of p (K5).  Levels sharded over the
    ranks; Mpx/s over all levels (max over ranks)."""
    import torch
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.parallel import shard_range
    from paper_2304_12152_b200.spectral import anisotropy_device, rapsd_device, ring_partition
    dev = D.dev
    n_lv, S = 256, 256
    lo, hi = shard_range(n_lv, D.rank, D.world)
    n = hi - lo
    g = torch.arange(lo, hi, dtype=torch.float32, device=dev) / 255.0
    c = g[:, None, None].expand(n, S, S).contiguous()
    rng = Rng(noise_seed(3))
    rng.jump(lo * S * S)
    z = rng.gaussians_device(n * S * S, device=dev).view(n, S, S)
    part = ring_partition((S, S))
    p = torch.empty((n, S, S), dtype=torch.float32, device=dev)
    h = torch.empty((n, S, S), dtype=torch.uint8, device=dev)
    ws = net.halftone_device(c, z, p_out=p, h_out=h, check=True)
    hf = torch.empty((n, S, S), dtype=torch.float32, device=dev)
    out = {}

    def step():
        net.halftone_device(c, z, p_out=p, h_out=h, workspace=ws)
        hf.copy_(h)
        out["spec"] = rapsd_device(hf, part)
        out["las"] = anisotropy_device(p, part, want_grad=False)[0]

    with ClockSampler(dev.index) as clk:
        ms = timed(D, step, steps, warmup)
    power, anis, dc = out["spec"]
    from paper_2304_12152_b200.spectral import anisotropy_db
    mean_db = float(np.nanmean(anisotropy_db(anis.cpu().numpy())))
    return {"workload": "BASELINE config 3: 256 flat-gray 256x256 levels g=k/255, forward + "
                        "binarize + RAPSD/anisotropy of each halftone + L_AS of each p",
            "value": round(n_lv * S * S / (ms * 1e-3) / 1e6, 2), "unit": "Mpixel/s",
            "ms_per_step": round(ms, 4), "steps": steps,
            "parallelism": f"levels sharded {n_lv}/{D.world} per rank",
            "mean_anisotropy_db_rank0": round(mean_db, 3),
            "l2": "inputs (134 MB) larger than L2", "clocks": clk.summary()}


def bench_cfg4(D, net, steps, warmup):
    """Config 4: one 7016x4960 page (64 blobs, 16 rects), row strips over the
    ranks with a 34-row input halo (no communication; stitched result equals
    the unsharded one, tests/test_gpu_forward.py).  Device-resident and end
    to end (the rank's strip of contone+noise from pinned host memory in,
    its uint8 rows out), max over ranks."""
    import torch
    from paper_2304_12152_b200 import synth
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.parallel import row_strip
    dev = D.dev
    H, W = 7016, 4960
    st = row_strip(H, D.rank, D.world)
    page = synth.contone(H, W, seed=4, blobs=64, rects=16)
    rng = Rng(noise_seed(4))
    rng.jump(st.in_row0 * W)                         # W even: rows are whole draw pairs
    z = rng.gaussians_device(st.in_rows * W, device=dev).view(1, st.in_rows, W)
    c = torch.from_numpy(page[st.in_row0:st.in_row0 + st.in_rows]).to(dev)[None]
    h = torch.empty((1, st.out_rows, W), dtype=torch.uint8, device=dev)
    rows = st.as_kernel_rows(H)
    ws = net.halftone_device(c, z, h_out=h, rows=rows, check=True)
    # end to end: whole host pages (pinned) streamed two deep through
    # parallel.PageEngine -- every page does its strip's H2D of contone +
    # noise and the D2H of its halftone rows; page i+1's copies overlap page
    # i's kernels
    from paper_2304_12152_b200.parallel import PageEngine
    eng = PageEngine(net, H, W, depth=2)
    ph = torch.from_numpy(page).pin_memory()
    zh = torch.zeros((H, W), dtype=torch.float32).pin_memory()
    zh[st.in_row0:st.in_row0 + st.in_rows] = z[0].cpu()
    outs = [torch.empty(eng.out_shape(), dtype=torch.uint8).pin_memory() for _ in range(2)]

    def stream_pages(n):
        tickets = []
        for i in range(n):
            if i >= 2:
                eng.wait(tickets[i - 2])
            tickets.append(eng.submit(ph, zh, outs[i % 2]))
        for t_ in tickets[-2:]:
            eng.wait(t_)
        return outs[(n - 1) % 2]

    def step_dev():
        net.halftone_device(c, z, h_out=h, rows=rows, workspace=ws)

    with ClockSampler(dev.index) as clk:
        ms = timed(D, step_dev, steps, warmup)
        stream_pages(warmup)
        D.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        last = stream_pages(steps)
        ms_e2e = D.max((time.perf_counter() - t0) * 1e3 / steps)[0]
    assert torch.equal(last, h[0].cpu()), "page e2e output differs from the device path"
    return {"workload": "BASELINE config 4: one 7016x4960 page (64 blobs, 16 rects), row strips "
                        "with 34-row halos",
            "value": round(H * W / (ms * 1e-3) / 1e6, 2), "unit": "Mpixel/s",
            "ms_per_page": round(ms, 4),
            "e2e": {"value": round(H * W / (ms_e2e * 1e-3) / 1e6, 2), "unit": "Mpixel/s",
                    "h2d_bytes_per_step": eng.h2d_bytes(), "d2h_bytes_per_step": eng.d2h_bytes(),
                    "api": "parallel.PageEngine.submit/wait (pinned host fp32 page + noise -> the strip's "
                           "uint8 rows, pages streamed two deep), per rank, wall clock"},
            "steps": steps, "parallelism": f"row strips over {D.world} rank(s), no collective",
            "l2": "inputs (278 MB) larger than L2", "clocks": clk.summary()}


def bench_cfg5(D, steps, warmup, burst):
    """Config 5: rl.train_step with 16 x 256x256 crops + 4 flat-gray images
    (LE estimator, Gaussian HVS, anisotropy loss, backward, Adam); data
    parallel over the ranks with one gradient all-reduce per step."""
    import torch
    from paper_2304_12152_b200 import rl, synth
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import Adam, PolicyNetwork
    group = None
    cfg = rl.TrainConfig(iterations=1000, batch_size=16, crop_size=256, anisotropy_batch_size=4,
                         hvs_model="gaussian")
    ds = [synth.contone(384, 384, seed=100 + i).astype(np.float64) for i in range(8)]
    rng = Rng(cfg.seed)
    net = PolicyNetwork(cfg.channels, cfg.blocks)
    adam = Adam(net.params())
    net.init_params(rng)
    t = [0]
    diag = {}

    def step():
        diag.update(rl.train_step(net, adam, ds, cfg, rng, t[0], group=group))
        t[0] += 1

    with ClockSampler(D.dev.index) as clk:
        ms = timed(D, step, steps, warmup)
    # tensor work the 32->32 convs execute per step (default kernels): the
    # 16 forward conv1s as three fp16-pair products (conv_tc2), the 16 forward
    # conv2s and the 32 input gradients as six split-bf16 products (conv_tc),
    # the 32 weight gradients as three two-part bf16 products (wgrad_tc)
    px = 20 * 256 * 256
    products = 16 * 3 + 16 * 6 + 32 * 6 + 32 * 3
    flop = px * 2 * 9 * 32 * 32 * products
    return {"workload": "BASELINE config 5: train_step, 16 x 256x256 crops + 4 flat-gray images, "
                        "LE estimator (Gaussian HVS), anisotropy loss, backward, Adam",
            "value": round(1e3 / ms, 3), "unit": "steps/s", "ms_per_step": round(ms, 3),
            "steps": steps, "parallelism": f"data parallel over {D.world} rank(s), one all-reduce per step",
            "roofline": {"bound": "tensor", "unit": "TFLOP/s",
                         "achieved": round(flop / (ms * 1e-3) / 1e12, 1), "peak": burst,
                         "frac": round(flop / (ms * 1e-3) / 1e12 / burst, 4),
                         "work": "executed MMA work of the 32->32 convs (fwd conv1 3 fp16-pair products, fwd conv2 and dgrad 6 split-bf16, wgrad 3 two-part bf16) over the whole step time"},
            "last_diag": {k: (round(v, 9) if isinstance(v, float) else v) for k, v in diag.items()},
            "clocks": clk.summary()}


# ------------------------------------------------------------------ main arms
def run_ours(args, rank, world, local):
    import ctypes as C

    import torch
    import torch.distributed as dist
    from paper_2304_12152_b200.parallel import shard_range
    # HT_BENCH_FUNCTIONAL=1: control-flow check of the N-rank path on fewer
    # GPUs (ranks share devices, gloo instead of NCCL); its numbers are not
    # measurements and the line says so
    functional = os.environ.get("HT_BENCH_FUNCTIONAL") == "1"
    if functional:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    from paper_2304_12152_b200 import _lib, rl
    D = Dist(rank, world, dev)
    burst, sustained, hbm, src = load_peaks()

    lo, hi = shard_range(B2, rank, world)
    B = hi - lo
    c_np, z_np = make_inputs(lo, hi, S2, S2, seed=2, device=dev)
    net = make_net()
    c = torch.from_numpy(c_np).to(dev)
    z = torch.from_numpy(z_np).to(dev)
    h = torch.empty((B, S2, S2), dtype=torch.uint8, device=dev)
    ws = net.halftone_device(c, z, h_out=h, check=True)       # correctness gate + workspace
    torch.cuda.synchronize()

    def step():
        net.halftone_device(c, z, h_out=h, workspace=ws)

    for _ in range(args.warmup):
        step()
    launches_per_step = _lib.launch_count()
    _lib.call("ht_timing_reserve", 16 * args.steps)
    _lib.call("ht_timing_enable", 1)
    with ClockSampler(local) as clk:
        ms_step = timed(D, step, args.steps, 0)
    _lib.call("ht_timing_enable", 0)
    nmax = 64 * args.steps
    tags, tms, cnt = (C.c_int * nmax)(), (C.c_float * nmax)(), C.c_int(0)
    _lib.call("ht_timing_read", tags, tms, nmax, C.byref(cnt))
    per_tag = {}
    for i in range(cnt.value):
        per_tag.setdefault(int(tags[i]), []).append(float(tms[i]))
    mid = per_tag.get(MID_TAG, [float("nan")])
    mid_ms = D.max(float(np.mean(mid)))[0]
    value = B2 * S2 * S2 / (ms_step * 1e-3) / 1e6

    # ---- end to end through the public API (pinned host in, uint8 out)
    e2e = None
    if not args.no_e2e:
        eng = rl.HalftoneEngine(net, B, S2, S2, chunks=1, output="h", depth=2)
        ch = torch.from_numpy(c_np).pin_memory()
        zh = torch.from_numpy(z_np).pin_memory()
        outs = [torch.empty(eng.out_shape(), dtype=torch.uint8).pin_memory() for _ in range(2)]

        def stream_batches(n):
            # batch i+1 is submitted while batch i finishes (its copies overlap
            # i's kernels); every batch does its own H2D of contone + noise and
            # D2H of the halftone; batch i is waited on before i+2 reuses its
            # output buffer
            tickets = []
            for i in range(n):
                if i >= 2:
                    eng.wait(tickets[i - 2])
                tickets.append(eng.submit(ch, zh, outs[i % 2]))
            for t_ in tickets[-2:]:
                eng.wait(t_)
            return outs[(n - 1) % 2]

        stream_batches(args.warmup)
        D.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        last = stream_batches(args.steps)
        el = D.max(time.perf_counter() - t0)[0]
        assert np.array_equal(last.numpy(), h.cpu().numpy()), "e2e output differs from device path"
        e2e = {"value": round(B2 * S2 * S2 * args.steps / el / 1e6, 3), "unit": "Mpixel/s",
               "h2d_bytes_per_step": eng.h2d_bytes(), "d2h_bytes_per_step": eng.d2h_bytes(),
               "api": "rl.HalftoneEngine.submit/wait (pinned host fp32 contone+noise -> uint8 "
                      "halftone, batches streamed two deep), per rank",
               "bytes_note": "per rank; summed over ranks the copies are the whole batch"}

    # ---- the reference-compatible drop-in call: rl.halftone(net, c, z) with
    #      numpy float32 (B, H, W) in and float64 (h, p) arrays out, as
    #      rl.infer_halftone returns them (rl.py:306-311), per rank's shard
    dropin = None
    if not args.no_e2e:
        hd, pd = rl.halftone(net, c_np, z_np)        # warm (allocations)
        assert np.array_equal(hd.astype(np.uint8), h.cpu().numpy())
        del hd, pd
        reps = 3
        D.barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            hd, pd = rl.halftone(net, c_np, z_np)
            del hd, pd
        el = D.max((time.perf_counter() - t0) / reps)[0]
        dropin = {"value": round(B2 * S2 * S2 / el / 1e6, 2), "unit": "Mpixel/s",
                  "api": "rl.halftone(net, contone, noise): numpy float32 (B,H,W) in, float64 (h, p) out "
                         "(the reference's return types), wall clock, mean of %d calls; host batches "
                         "flow in 8 chunks over two streams" % reps,
                  "h2d_bytes_per_step": 2 * B * S2 * S2 * 4, "d2h_bytes_per_step": B * S2 * S2 * 16}

    # ---- weak scaling (secondary): every rank halftones its own 64 images
    weak = None
    if world > 1:
        cw, zw = make_inputs(0, B2, S2, S2, seed=2 + 7919 * rank, device=dev)
        cw, zw = torch.from_numpy(cw).to(dev), torch.from_numpy(zw).to(dev)
        hw_ = torch.empty((B2, S2, S2), dtype=torch.uint8, device=dev)
        wsw = net.halftone_device(cw, zw, h_out=hw_, check=True)
        msw = timed(D, lambda: net.halftone_device(cw, zw, h_out=hw_, workspace=wsw), args.steps, 2)
        weak = {"value": round(B2 * world * S2 * S2 / (msw * 1e-3) / 1e6, 2), "unit": "Mpixel/s",
                "ms_per_step": round(msw, 4), "per_rank_images": B2}
        del cw, zw, hw_, wsw

    # ---- CPU baseline: the real reference on the host cores (rank 0, N=1)
    cpu = None
    if world == 1 and not args.no_cpu:
        cores = host_cores()
        pool = RefPool(cores)
        pool.run(ref_tiles(cores, 32))                 # worker start-up / imports
        jobs = ref_tiles(cores, REF_TILE)
        px, wall = pool.run(jobs)
        pool.close()
        cpu = {"value": round(px / wall / 1e6, 6), "unit": "Mpixel/s", "cores": cores,
               "kind": pool.kind, "sample": pool.describe(REF_TILE, len(jobs)) + f", {wall:.1f} s wall"}

    # ---- other BASELINE configs
    configs = {}
    if not args.no_configs:
        sub_steps = max(3, min(args.steps, 10))
        configs["cfg1"] = bench_cfg1(D, net, reps=20)
        configs["cfg3"] = bench_cfg3(D, net, sub_steps, 2)
        configs["cfg4"] = bench_cfg4(D, net, sub_steps, 2)
        configs["cfg5"] = bench_cfg5(D, sub_steps, 3, burst)

    if rank == 0:
        achieved = FLOP_PER_PX_MIDPASS * B * S2 * S2 / (mid_ms * 1e-3) / 1e12
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            try:   # measured DRAM bytes/pixel of this kernel (ncu) x pixels per launch
                traffic = round(json.load(open(tpath))[str(MID_TAG)]["bytes_per_px"] * B * S2 * S2)
            except Exception:
                traffic = None
        roofline = {"bound": "tensor", "achieved": round(achieved, 2), "peak": burst,
                    "unit": "TFLOP/s", "frac": round(achieved / burst, 4), "traffic": traffic,
                    "kernel": "tc_pass_kernel<false,2,false> (2 residual blocks = 4 convs 32->32)",
                    "traffic_unit": "bytes per launch (DRAM read+write, ncu)",
                    "algorithmic_flop_per_launch": FLOP_PER_PX_MIDPASS * B * S2 * S2,
                    "mean_launch_ms": round(mid_ms, 4), "launches_timed": len(mid),
                    "peak_kind": f"burst bf16/fp16 dense ({src}); sustained {sustained}",
                    "frac_of_sustained": round(achieved / sustained, 4),
                    "step_frac_of_peak": round(FLOP_PER_PX * B2 * S2 * S2 / world / (ms_step * 1e-3) / 1e12 / burst, 4),
                    "pass_ms": {str(k): round(float(np.mean(v)), 4) for k, v in sorted(per_tag.items())}}
        out = {"metric": METRIC, "value": round(value, 3), "unit": "Mpixel/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "f16xf16->f32 (fp32 residual)",
               "data": "synthetic (seeded ramp+blob+rect contones, reference-RNG noise), random-init weights std 0.01",
               "config": headline_config(world),
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": launches_per_step * args.steps,
               "clocks": clk.summary()}
        if weak is not None:
            out["weak_scaling"] = weak
        if dropin is not None:
            out["e2e_dropin"] = dropin
        if configs:
            out["configs"] = configs
        if functional:
            out["functional_check_only"] = "ranks shared GPUs over gloo: not a measurement"
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, rank, world):
    """Reference arm: the unmodified reference (htlab from baseline/_ref)
    forward + threshold on the host cores; rank 0 only."""
    if rank != 0:
        return
    cores = host_cores()
    pool = RefPool(cores)
    warm = ref_tiles(cores, 32)
    jobs = ref_tiles(cores, REF_TILE)
    for _ in range(args.warmup):                 # worker start-up, imports, BLAS init
        pool.run(warm)
    times, px = [], 0
    for _ in range(args.steps):
        px, wall = pool.run(jobs)
        times.append(wall)
    pool.close()
    ms = float(np.mean(times)) * 1e3
    value = px / (ms * 1e-3) / 1e6
    sample = pool.describe(REF_TILE, len(jobs)) + "; warm-up steps use 32x32 tiles"
    out = {"metric": METRIC, "value": round(value, 6), "unit": "Mpixel/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (same generator, noise stream and weights as the GPU arm)",
           "config": headline_config(world),
           "impl": "reference",
           "cpu_baseline": {"value": round(value, 6), "unit": "Mpixel/s", "cores": cores,
                            "kind": pool.kind, "sample": sample},
           "e2e": {"value": round(value, 6), "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="headline config 2 only")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import torch
        if torch.cuda.device_count() < args.gpus and os.environ.get("HT_BENCH_FUNCTIONAL") != "1":
            raise SystemExit(f"bench.py: --gpus {args.gpus} but {torch.cuda.device_count()} GPU(s) visible")
        sys.exit(relaunch(args))
    rank, world, local = dist_setup(args)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
