"""Multi-process host logic on CPU (gloo, world_size 2): sharding plans, the
data-parallel gradient reduction and the row-strip halo rule.

The GPU kernels are not run here; where numbers are needed, the CPU oracle
plays the per-rank compute (as a checker), so the test exercises exactly the
decomposition the GPU path uses: global 1/batch scaling, one SUM all-reduce.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_12152_b200.parallel import RECEPTIVE_RADIUS, row_strip, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, fn, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return sorted(out, key=lambda x: x[0])


def _worker(rank, world, port, fn, args, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world, *args)))
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------- pure logic
def test_row_strips_cover_page_with_halo():
    for H in (1, 7, 100, 7016):
        for world in (1, 2, 3, 8):
            strips = [row_strip(H, r, world) for r in range(world)]
            assert strips[0].out_row0 == 0
            assert sum(s.out_rows for s in strips) == H
            for s in strips:
                assert s.in_row0 == max(0, s.out_row0 - RECEPTIVE_RADIUS)
                assert s.in_row0 + s.in_rows == min(H, s.out_row0 + s.out_rows + RECEPTIVE_RADIUS)


def test_row_strip_halo_rule_with_oracle():
    """Stitching per-strip forwards (halo = number of conv layers) reproduces
    the full forward -- the rule the fused kernel's row sharding relies on."""
    from oracle import htoracle as O
    params = O.init_params(O.Rng(3), 4, 2, 2, 0.3)    # 6 conv layers -> radius 6
    depth = 2 + 2 * 2
    H, W = 40, 11
    r = O.Rng(5)
    x = np.stack((r.uniforms(H * W).reshape(H, W), r.gaussians(H * W).reshape(H, W)))[None]
    full = O.policy_forward(params, x)[0, 0]
    for world in (2, 3):
        out = np.zeros_like(full)
        for rank in range(world):
            s = row_strip(H, rank, world, halo=depth)
            xs = x[:, :, s.in_row0:s.in_row0 + s.in_rows]
            p = O.policy_forward(params, xs)[0, 0]
            o = s.out_row0 - s.in_row0
            out[s.out_row0:s.out_row0 + s.out_rows] = p[o:o + s.out_rows]
        assert np.max(np.abs(out - full)) < 1e-12
        # one row less of halo is not enough
        s = row_strip(H, 1, 2, halo=depth - 1)
        p = O.policy_forward(params, x[:, :, s.in_row0:s.in_row0 + s.in_rows])[0, 0]
        o = s.out_row0 - s.in_row0
        assert np.max(np.abs(p[o:o + s.out_rows] - full[s.out_row0:s.out_row0 + s.out_rows])) > 1e-9


# ---------------------------------------------------------------- gloo ranks
def _allreduce_body(rank, world):
    from paper_2304_12152_b200.parallel import allreduce_sum_
    g = torch.full((5,), float(rank + 1), dtype=torch.float64)
    s = torch.tensor([rank * 1.0, 2.0, 3.0], dtype=torch.float64)
    allreduce_sum_(g, s)
    return g.tolist(), s.tolist()


def test_allreduce_sum_gloo_world2():
    out = _run(2, _allreduce_body)
    for _, (g, s) in out:
        assert g == [3.0] * 5 and s == [1.0, 4.0, 6.0]


def _dp_grad_body(rank, world, bs, size):
    """Each rank: the reference's host draws (identical on every rank), its
    shard of the batch through the oracle forward/backward with the GLOBAL
    1/batch scaling (rl.py:253), then one SUM all-reduce."""
    from oracle import htoracle as O
    from paper_2304_12152_b200.parallel import allreduce_sum_
    params = O.init_params(O.Rng(0), 4, 1, 2, 0.2)
    rng = O.Rng(7)
    ds = [np.linspace(0, 1, 20 * 20).reshape(20, 20), np.full((20, 20), 0.3)]
    crops, noises = [], []
    for _ in range(bs):                          # rl.py:242-245 draw order
        img = ds[rng.randint(len(ds))]
        crops.append(O.random_crop(rng, img, size))
        noises.append(O.gaussian_noise_map(rng, size, size))
    lo, hi = shard_range(bs, rank, world)
    flat = torch.zeros(sum(p.size for p in params), dtype=torch.float64)
    if hi > lo:
        x = np.stack([np.stack((crops[i], noises[i])) for i in range(lo, hi)])
        p, cache = O.policy_forward(params, x, keep=True)
        dp = np.stack([np.sin(np.arange(size * size) + i).reshape(size, size)
                       for i in range(lo, hi)])[:, None] / bs
        _, grads = O.policy_backward(params, cache, dp)
        flat = torch.from_numpy(np.concatenate([g.ravel() for g in grads]))
    allreduce_sum_(flat)
    return flat.numpy().tolist(), rng.state_words()


@pytest.mark.parametrize("bs", [3, 4])
def test_dp_gradient_equals_single_process(bs):
    size = 8
    multi = _run(2, _dp_grad_body, bs, size)
    single = _dp_grad_body(0, 1, bs, size)
    g1 = np.array(single[0])
    for _, (g, state) in multi:
        assert np.max(np.abs(np.array(g) - g1)) <= 1e-12 * max(1.0, np.abs(g1).max())
        assert list(state) == list(single[1])     # every rank consumed the same stream
