"""Benchmark of the halftoning hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU)

Workload (config 2 of BASELINE.json, the largest single-GPU config the metric
is quoted on): 64 seeded synthetic 512x512 contones (ramp + 8 Gaussian blobs
+ 2 rectangles, 10% with step edges) with N(0,1) noise maps from the
reference RNG; the reference's default policy CNN (C=32, 16 blocks, 296,833
params) with seeded random-init weights (std 0.01).  One step = fused
forward + sigmoid/threshold (K1) over the rank's 64 images.  Multi-GPU is
weak scaling: every rank halftones its own 64-image batch (independent
images, no collective on the data path).

value  = device-resident throughput (inputs in HBM), CUDA events, max over ranks.
e2e    = same metric through rl.HalftoneEngine (public API): pinned host
         contone+noise -> H2D -> K1 -> D2H uint8 halftones, every step;
         batches streamed two deep (submit/wait), wall clock.
roofline = the dominant kernel (the 2-residual-block pass, 7 of 9 launches),
         algorithmic FLOPs per launch / its mean CUDA-event duration, against
         the measured sustained bf16/fp16 dense peak (MEASURED_PEAKS.json).
cpu_baseline = the CPU oracle (NumPy port of the reference forward) on the
         host's cores over a bounded sample of the same images.
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

FLOP_PER_PX = 2 * 9 * (2 * 32 + 2 * 16 * 32 * 32 + 32)   # 591,552
FLOP_PER_PX_MIDPASS = 2 * 9 * 4 * 32 * 32               # 4 convs of 32->32 per pass
MID_TAG = 20                                             # pass tag: no conv_in, 2 blocks, no conv_out
METRIC = "halftone Mpixel/s (CNN inference+binarize) at 1/2/4/8 B200; % of roofline"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["bf16_tflops"], d["bf16_tflops_sustained"], d["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


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
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
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
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ------------------------------------------------------------------ inputs
def noise_seed(seed):
    return seed * 1_000_003


def make_inputs(B, H, W, seed, device=None):
    """Contones from the BASELINE generator; noise maps drawn in image order
    from one reference-RNG stream (as B calls of rl.infer_halftone would),
    on the GPU when `device` is given (the same stream the e2e engine draws)."""
    from paper_2304_12152_b200 import synth
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_device, gaussian_noise_map_f32
    c = synth.config_batch(B, H, W, seed=seed, blobs=8, rects=2, step_frac=0.1)
    rng = Rng(noise_seed(seed))
    if device is not None:
        z = np.stack([gaussian_noise_map_device(rng, W, H, device=device).cpu().numpy()
                      for _ in range(B)])
    else:
        z = np.stack([gaussian_noise_map_f32(rng, W, H) for _ in range(B)])
    return c, z


def make_net():
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = PolicyNetwork(32, 16)
    net.init_params(Rng(0), std=0.01)
    return net


# ------------------------------------------------------------------ CPU baseline
def _cpu_init():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"


def _cpu_worker(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    c, z = args
    from oracle import htoracle as O
    params = O.init_params(O.Rng(0), 32, 16, 2, 0.01)
    t0 = time.perf_counter()
    O.halftone(params, c.astype(np.float64), z.astype(np.float64))
    return c.size, time.perf_counter() - t0


def cpu_sample(c, z, tile, cores):
    """Oracle (NumPy port of nn.py:138-150 + rl.py:311) on `cores` worker
    processes, one tile x tile crop of a distinct image each."""
    import multiprocessing as mp
    jobs = []
    for k in range(cores):
        i = k % c.shape[0]
        y0 = (k * 37) % (c.shape[1] - tile + 1)
        x0 = (k * 53) % (c.shape[2] - tile + 1)
        jobs.append((c[i, y0:y0 + tile, x0:x0 + tile].copy(), z[i, y0:y0 + tile, x0:x0 + tile].copy()))
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores, initializer=_cpu_init) as pool:
        pool.map(_cpu_worker, jobs[:cores])        # warm the workers (imports)
        t0 = time.perf_counter()
        res = pool.map(_cpu_worker, jobs)
        wall = time.perf_counter() - t0
    px = sum(r[0] for r in res)
    return px / wall / 1e6, wall, px


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-tile", type=int, default=64)
    ap.add_argument("--workload", default="halftone", choices=["halftone", "train"],
                    help="halftone = BASELINE config 2 (headline); train = config 5 train_step")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    B, H, W = args.batch, args.size, args.size

    if args.impl == "reference":
        return run_reference(args, rank, world, B, H, W)
    if args.workload == "train":
        return run_train(args, rank, world, local)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2304_12152_b200 import _lib, rl

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    seed = 2 + 7919 * rank
    c_np, z_np = make_inputs(B, H, W, seed=seed, device=dev)
    net = make_net()
    c = torch.from_numpy(c_np).to(dev)
    z = torch.from_numpy(z_np).to(dev)
    h = torch.empty((B, H, W), dtype=torch.uint8, device=dev)
    ws = net.halftone_device(c, z, h_out=h, check=True)       # correctness gate + workspace
    torch.cuda.synchronize()

    def step():
        net.halftone_device(c, z, h_out=h, workspace=ws)

    for _ in range(args.warmup):
        step()
    launches_per_step = _lib.launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    _lib.call("ht_timing_reserve", 16 * args.steps)
    _lib.call("ht_timing_enable", 1)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(args.steps):
            step()
        e1.record(st)
        torch.cuda.synchronize()
    _lib.call("ht_timing_enable", 0)
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    import ctypes as C
    nmax = 64 * args.steps
    tags = (C.c_int * nmax)()
    tms = (C.c_float * nmax)()
    cnt = C.c_int(0)
    _lib.call("ht_timing_read", tags, tms, nmax, C.byref(cnt))
    per_tag = {}
    for i in range(cnt.value):
        per_tag.setdefault(int(tags[i]), []).append(float(tms[i]))
    mid = per_tag.get(MID_TAG, [float("nan")])
    mid_ms = float(np.mean(mid))
    t = torch.tensor([ms, mid_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, mid_ms = float(t[0]), float(t[1])
    ms_step = ms / args.steps
    px_rank = B * H * W
    value = px_rank * world / (ms_step * 1e-3) / 1e6

    # ---- end-to-end through the public API (pinned host in, uint8 out)
    e2e = None
    if not args.no_e2e:
        # streamed batches, one chunk each: batch i+1's copies run under batch
        # i's kernels (measured: 1222 Mpx/s streamed vs 1178 for the best
        # per-call chunking, debug/e2e_sweep.py)
        eng = rl.HalftoneEngine(net, B, H, W, chunks=1, output="h", depth=2)
        ch = torch.from_numpy(c_np).pin_memory()
        zh = torch.from_numpy(z_np).pin_memory()
        oh = torch.empty(eng.out_shape(), dtype=torch.uint8).pin_memory()
        # contones + noise maps from pinned host memory.  (The engine can also
        # draw the noise on the GPU from an Rng, eng(ch, rng, oh); measured
        # slower here: the copy engines move the noise for free while device
        # generation takes SM time from the forward.)
        # streaming use: batch i+1 is submitted while batch i finishes (its
        # first copies overlap i's last kernel and read-back); every batch
        # does its own H2D of contone + noise and D2H of the halftone, and
        # batch i is waited on before i+2 reuses its output buffer
        outs = [oh, torch.empty_like(oh).pin_memory()]

        def stream_batches(n):
            tickets = []
            for i in range(n):
                if i >= 2:
                    eng.wait(tickets[i - 2])
                tickets.append(eng.submit(ch, zh, outs[i % 2]))
            for t_ in tickets[-2:]:
                eng.wait(t_)
            return outs[(n - 1) % 2]

        stream_batches(args.warmup)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        last = stream_batches(args.steps)
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        assert np.array_equal(last.numpy(), h.cpu().numpy()), "e2e output differs from device path"
        e2e = {"value": px_rank * world * args.steps / float(el) / 1e6, "unit": "Mpixel/s",
               "h2d_bytes_per_step": eng.h2d_bytes(), "d2h_bytes_per_step": eng.d2h_bytes(),
               "api": "rl.HalftoneEngine.submit/wait (pinned host fp32 contone+noise -> uint8 "
                      "halftone, batches streamed two deep)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    burst, sustained, hbm, src = load_peaks()
    achieved = FLOP_PER_PX_MIDPASS * px_rank / (mid_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:   # measured DRAM bytes/pixel of this kernel (ncu) x pixels per launch
            traffic = round(json.load(open(tpath))[str(MID_TAG)]["bytes_per_px"] * px_rank)
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": round(achieved, 2), "peak": sustained,
                "unit": "TFLOP/s", "frac": round(achieved / sustained, 4), "traffic": traffic,
                "kernel": "tc_pass_kernel<false,2,false> (2 residual blocks = 4 convs 32->32)",
                "traffic_unit": "bytes per launch (DRAM read+write, ncu)",
                "algorithmic_flop_per_launch": FLOP_PER_PX_MIDPASS * px_rank,
                "mean_launch_ms": round(mid_ms, 4), "launches_timed": len(mid),
                "peak_kind": f"sustained bf16/fp16 dense ({src})",
                "step_frac_of_peak": round(FLOP_PER_PX * px_rank / (ms_step * 1e-3) / 1e12 / sustained, 4),
                "pass_ms": {str(k): round(float(np.mean(v)), 4) for k, v in sorted(per_tag.items())}}

    cpu = None
    if world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        v, wall, px = cpu_sample(c_np, z_np, args.cpu_tile, cores)
        cpu = {"value": round(v, 6), "unit": "Mpixel/s", "cores": cores, "kind": "port",
               "sample": f"{cores} crops of {args.cpu_tile}x{args.cpu_tile} px of the workload "
                         f"images, one per worker process (OPENBLAS_NUM_THREADS=1), "
                         f"oracle/htoracle.py forward+threshold, {wall:.1f} s wall"}

    out = {"metric": METRIC, "value": round(value, 3), "unit": "Mpixel/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16xf16->f32 (fp32 residual)",
           "data": "synthetic (seeded ramp+blob+rect contones, reference-RNG noise), random-init weights std 0.01",
           "config": {"workload": f"BASELINE config 2: {B} x {H}x{W} contones per GPU, policy CNN C=32 B=16",
                      "global_batch": B * world, "image": [H, W], "parallelism": f"images sharded, {world} rank(s), no collective",
                      "l2": "inputs (134 MB) + pass buffers (4.3 GB) larger than L2 (126 MB)"},
           "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
           "gpu_launches": launches_per_step * args.steps,
           "clocks": clk.summary()}
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def run_train(args, rank, world, local):
    """BASELINE config 5: one rl.train_step = batch 16 of 256x256 crops + 4
    flat-gray images, forward, LE estimator (Gaussian HVS), anisotropy loss,
    backward, Adam; data parallel over the ranks with one all-reduce."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2304_12152_b200 import rl, synth
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import Adam, PolicyNetwork
    cfg = rl.TrainConfig(iterations=1000, batch_size=16, crop_size=256, anisotropy_batch_size=4,
                         hvs_model="gaussian")
    ds = [synth.contone(384, 384, seed=100 + i).astype(np.float64) for i in range(8)]
    rng = Rng(cfg.seed)
    net = PolicyNetwork(cfg.channels, cfg.blocks)
    adam = Adam(net.params())
    net.init_params(rng)
    for t in range(args.warmup):
        rl.train_step(net, adam, ds, cfg, rng, t)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # CUDA events on the step stream (they include any host gaps of the step)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(args.steps):
        diag = rl.train_step(net, adam, ds, cfg, rng, args.warmup + t)
    e1.record()
    torch.cuda.synchronize()
    el = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    if rank == 0:
        ms = float(el) / args.steps
        print(json.dumps({"metric": "train steps/s (config 5: 16x256^2 + 4 gray, LE + anisotropy, Adam)",
                          "value": round(1e3 / ms, 3), "unit": "steps/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2),
                          "higher_is_better": True, "scaling": "strong",
                          "dtype": "f32 (32->32 convs: tcgen05 split-bf16, fp32-level; others fp32/fp64)",
                          "last_diag": diag}))
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, rank, world, B, H, W):
    """Reference arm: the reference's CPU path (oracle port of htlab's forward +
    threshold; the reference is pure Python/NumPy) on the host's cores."""
    if rank != 0:
        return
    c_np, z_np = make_inputs(min(B, 8), H, W, seed=2)
    cores = os.cpu_count() or 1
    import multiprocessing as mp
    tile = args.cpu_tile
    jobs = []
    for k in range(cores):
        i = k % c_np.shape[0]
        y0 = (k * 37) % (H - tile + 1)
        x0 = (k * 53) % (W - tile + 1)
        jobs.append((c_np[i, y0:y0 + tile, x0:x0 + tile].copy(), z_np[i, y0:y0 + tile, x0:x0 + tile].copy()))
    ctx = mp.get_context("spawn")
    times = []
    with ctx.Pool(cores, initializer=_cpu_init) as pool:
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(_cpu_worker, jobs)
            if s >= args.warmup:
                times.append(time.perf_counter() - t0)
    px = cores * tile * tile
    ms = float(np.mean(times)) * 1e3
    value = px / (ms * 1e-3) / 1e6
    out = {"metric": METRIC, "value": round(value, 6), "unit": "Mpixel/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (same generator/weights as the GPU arm)",
           "config": {"workload": f"BASELINE config 2 images, bounded sample per step: {cores} x {tile}x{tile} px crops",
                      "global_batch": B, "image": [H, W]},
           "impl": "reference",
           "cpu_baseline": {"value": round(value, 6), "unit": "Mpixel/s", "cores": cores, "kind": "port",
                            "sample": f"{cores} worker processes x one {tile}x{tile} crop per step "
                                      "(oracle/htoracle.py: NumPy restatement of nn.py:138-150 + rl.py:311)"},
           "e2e": {"value": round(value, 6), "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
