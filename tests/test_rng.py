"""Device RNG streams with exact jump-ahead.

CPU: the GF(2) jump equals sequential draws.  GPU: device uniforms are the
host stream bit for bit, device gaussians match the host / reference vectors
within the documented ulp bounds, and the host state advances identically
(reference KATs: tests/golden/rng.npz, written by the reference's Rng)."""

import numpy as np
import pytest

from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map


def _advanced(seed, n):
    r = Rng(seed)
    r.uniforms(n)
    return r.state_words()


@pytest.mark.parametrize("n", [0, 1, 2, 3, 63, 64, 65, 255, 1000, 12345, 300_001])
def test_jump_equals_sequential_draws(n):
    r = Rng(17)
    r.jump(n)
    assert r.state_words() == _advanced(17, n)


def test_jump_composes_at_large_distances():
    a, b = (1 << 40) + 12345, (1 << 33) + 7
    r1, r2 = Rng(5), Rng(5)
    r1.jump(a)
    r1.jump(b)
    r2.jump(a + b)
    assert r1.state_words() == r2.state_words()
    # matches the reference KAT after 100k uniforms
    from conftest import golden
    r = Rng(99)
    r.jump(100_000)
    assert list(r.state_words()) == [int(v) for v in golden("rng.npz")["long_state_seed99"]]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 255, 256, 257, 32768 + 3, 1_000_003])
def test_device_uniforms_bit_exact(n):
    import torch
    host, dev = Rng(23), Rng(23)
    host.uniforms(11)
    dev.uniforms(11)                       # start mid-stream
    want = host.uniforms(n)
    got = dev.uniforms_device(n).cpu().numpy()
    assert np.array_equal(got, want)
    assert dev.state_words() == host.state_words()
    got32 = Rng(23).uniforms_device(n, dtype=torch.float32).cpu().numpy()
    assert np.array_equal(got32, Rng(23).uniforms(n).astype(np.float32))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 7, 256, 257, 65_537, 2_000_001])
def test_device_gaussians_match_host_stream(n):
    import torch
    host, dev = Rng(31), Rng(31)
    want = host.gaussians(n)
    got = dev.gaussians_device(n, dtype=torch.float64).cpu().numpy()
    assert dev.state_words() == host.state_words()          # 2*ceil(n/2) draws either way
    ulp = np.spacing(np.abs(want))
    assert np.max(np.abs(got - want) / ulp) <= 4.0
    # fp32 noise as the fused kernel consumes it
    f_host = Rng(31).gaussians_f32(n)
    f_dev = Rng(31).gaussians_device(n).cpu().numpy()
    diff = f_dev != f_host
    assert diff.mean() <= 1e-6
    if diff.any():
        assert np.max(np.abs(f_dev[diff] - f_host[diff]) / np.spacing(np.abs(f_host[diff]))) <= 1.0


@pytest.mark.gpu
def test_device_noise_map_against_reference_vectors():
    from conftest import golden
    from paper_2304_12152_b200.imagecore import gaussian_noise_map_device
    import torch
    g = golden("rng.npz")
    z = gaussian_noise_map_device(Rng(5), 8, 6, dtype=torch.float64).cpu().numpy()
    assert z.shape == (6, 8)
    assert np.max(np.abs(z - g["noise_seed5_w8_h6"])) <= 8.9e-16
    u = Rng(99)
    s = u.uniforms_device(100_000).cpu().numpy()
    assert s.sum() == g["long_uniforms_seed99_sum"][0] and s[-1] == g["long_uniforms_seed99_sum"][1]
    assert list(u.state_words()) == [int(v) for v in g["long_state_seed99"]]


@pytest.mark.gpu
def test_print_page_noise_is_fast():
    """Config 4 page noise (7016 x 4960) on the device: ms, not seconds."""
    import time
    import torch
    from paper_2304_12152_b200.imagecore import gaussian_noise_map_device
    r = Rng(1)
    gaussian_noise_map_device(r, 64, 64)
    torch.cuda.synchronize()
    t = time.perf_counter()
    z = gaussian_noise_map_device(r, 4960, 7016)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    assert z.shape == (7016, 4960) and dt < 0.1
    assert abs(float(z.mean())) < 1e-3 and abs(float(z.std()) - 1.0) < 1e-3


@pytest.mark.gpu
def test_gaussian_maps_from_recorded_states():
    """One launch for maps interleaved with host draws (rl.draw_batch order):
    map m equals the single-stream draw from the state it starts at."""
    import torch
    from paper_2304_12152_b200.imagecore import gaussian_maps_device
    r = Rng(77)
    starts, singles = [], []
    for i in range(5):
        r.randint(7)                               # host draws between maps
        starts.append(r.state_words())
        s = Rng(0)
        s.set_state_words(r.state_words())
        singles.append(s.gaussians_device(30 * 41).cpu().numpy().reshape(30, 41))
        r.jump(2 * ((30 * 41 + 1) // 2))
    maps = gaussian_maps_device(starts, 41, 30).cpu().numpy()
    assert maps.shape == (5, 30, 41)
    assert np.array_equal(maps, np.stack(singles))
    host = Rng(0)
    host.set_state_words(starts[3])
    f = host.gaussians_f32(30 * 41).reshape(30, 41)
    assert np.mean(maps[3] != f) <= 1e-3
    assert gaussian_maps_device([], 4, 4).shape == (0, 4, 4)
