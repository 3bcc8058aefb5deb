"""bench.py's CPU pieces: the reference arm's tiles and worker pool (the real
htlab from baseline/_ref when installed, else the oracle port), and the
strong-sharding input slices (noise stream jump-ahead per image)."""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_ref_tiles_are_quadrants_of_config2_images():
    from paper_2304_12152_b200 import synth
    jobs = bench.ref_tiles(5, 32)
    assert len(jobs) == 5
    c0 = synth.contone(512, 512, seed=bench.noise_seed(2), blobs=8, rects=2, step_edge=True)
    c1 = synth.contone(512, 512, seed=bench.noise_seed(2) + 1, blobs=8, rects=2, step_edge=True)
    assert np.array_equal(jobs[0][0], c0[:32, :32].astype(np.float64))
    assert np.array_equal(jobs[3][0], c0[480:, 480:].astype(np.float64))
    assert np.array_equal(jobs[4][0], c1[:32, :32].astype(np.float64))
    # noise: the reference's own Rng stream, image after image
    from oracle.htoracle import Rng, gaussian_noise_map
    z0 = gaussian_noise_map(Rng(bench.noise_seed(2)), 512, 512).astype(np.float32)
    assert np.array_equal(jobs[1][1], z0[:32, 480:].astype(np.float64))


def test_reference_pool_runs_the_reference_path():
    pool = bench.RefPool(2)
    try:
        jobs = bench.ref_tiles(2, 16)
        px, wall = pool.run(jobs)
    finally:
        pool.close()
    assert px == 2 * 16 * 16 and wall > 0
    want = "reference" if os.path.isdir(os.path.join(bench.REF_PATH, "htlab")) else "port"
    assert pool.kind == want
    assert os.environ["OPENBLAS_NUM_THREADS"] == "1"


def test_headline_config_is_the_same_for_both_arms():
    assert bench.headline_config(1) == bench.headline_config(1)
    cfg = bench.headline_config(8)
    assert cfg["global_batch"] == 64 and cfg["image"] == [512, 512]
    assert "64/8" in cfg["parallelism"]


@pytest.mark.parametrize("world", [1, 2, 8])
def test_noise_jump_ahead_matches_sequential_draws(world):
    """make_inputs' per-rank noise = the maps a single stream draws in image
    order (jump-ahead over the earlier ranks' images), host RNG only."""
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_f32
    from paper_2304_12152_b200.parallel import shard_range
    H = W = 8
    ref = Rng(bench.noise_seed(2))
    seq = [gaussian_noise_map_f32(ref, W, H) for _ in range(64)]
    for rank in range(world):
        lo, hi = shard_range(64, rank, world)
        r = Rng(bench.noise_seed(2))
        r.jump(lo * 2 * ((H * W + 1) // 2))
        got = [gaussian_noise_map_f32(r, W, H) for _ in range(lo, hi)]
        assert all(np.array_equal(a, b) for a, b in zip(got, seq[lo:hi]))
