"""CPU-only checks of the product library and host logic (no GPU needed)."""

import ctypes as C
import re
import os

import numpy as np
import pytest

from conftest import ROOT, golden


def header_symbols():
    src = open(os.path.join(ROOT, "include", "htb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(ht_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header():
    from paper_2304_12152_b200 import _lib
    syms = set(header_symbols()) - {"ht_last_error"}
    assert syms <= set(_lib.SIGNATURES), sorted(syms - set(_lib.SIGNATURES))


def test_sm100a_cubin_has_tcgen05(lib):
    """The fused forward must be genuine tcgen05 code (UTCHMMA / LDTM / STTM)."""
    import subprocess
    from paper_2304_12152_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "UTCHMMA" in out and "LDTM" in out and "STTM" in out
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _lib.LIB_PATH],
                                       capture_output=True, text=True).stdout


def test_rng_bit_exact_against_reference_vectors():
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map, splitmix64
    g = golden("rng.npz")
    s, outs = 0, []
    for _ in range(3):
        s, z = splitmix64(s)
        outs.append(z)
    assert outs == [int(v) for v in g["splitmix"]]
    r = Rng(0)
    r.set_state_words((1, 2, 3, 4))
    assert [r.next_uint64() for _ in range(6)] == [int(v) for v in g["xoshiro1234"]]
    assert list(Rng(42).state_words()) == [int(v) for v in g["state_seed42"]]
    assert np.array_equal(Rng(7).uniforms(9), g["uniforms_seed7"])
    # Box-Muller through libm: equal to numpy's log/cos/sin up to 1 ulp
    assert np.max(np.abs(Rng(11).gaussians(7) - g["gaussians_seed11"])) <= 4.5e-16
    nm = gaussian_noise_map(Rng(5), 8, 6)
    assert nm.shape == (6, 8)
    assert np.max(np.abs(nm - g["noise_seed5_w8_h6"])) <= 4.5e-16
    r = Rng(3)
    assert [r.randint(n) for n in (1, 2, 7, 100, 1 << 20)] == list(g["randint_seed3"])
    r = Rng(99)
    u = r.uniforms(100_000)
    assert u.sum() == g["long_uniforms_seed99_sum"][0]
    assert list(r.state_words()) == [int(v) for v in g["long_state_seed99"]]


def test_param_count_and_geometry():
    from paper_2304_12152_b200 import _lib
    from paper_2304_12152_b200.nn import PolicyNetwork
    assert _lib.out_i64("ht_num_params", 32, 16) == 296_833
    net = PolicyNetwork()
    assert net.num_params() == 296_833
    assert [p.value.shape for p in net.params()[:3]] == [(32, 2, 3, 3), (32,), (32, 32, 3, 3)]
    assert _lib.out_i64("ht_num_params", 8, 2) == PolicyNetwork(8, 2).num_params()


def test_init_params_matches_reference_draw_order():
    from oracle import htoracle as O
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = PolicyNetwork(8, 2)
    net.init_params(Rng(0), std=0.05)
    ref = O.init_params(O.Rng(0), 8, 2, 2, 0.05)
    for p, q in zip(net.params(), ref):
        assert np.max(np.abs(p.value - q)) <= 1e-16


def test_cosine_lr_and_config():
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.nn import cosine_lr
    assert cosine_lr(0, 10) == 3e-4 and cosine_lr(10, 10) == 1e-5
    assert abs(cosine_lr(5, 10) - (1e-5 + 0.5 * (3e-4 - 1e-5))) < 1e-18
    with pytest.raises(ValueError):
        cosine_lr(0, 0)
    with pytest.raises(ValueError):
        rl.TrainConfig(estimator="nope").validate()


def test_shard_ranges_cover_batch():
    from paper_2304_12152_b200.rl import shard_range
    for n in (1, 4, 16, 20):
        for world in (1, 2, 3, 8):
            got = [shard_range(n, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1


def test_ring_partition_host_matches_golden():
    import hashlib
    from paper_2304_12152_b200.spectral import ring_partition
    g = golden("spectral.npz")
    for n in (4, 32, 256):
        part = ring_partition((n, n))
        assert part.counts.tolist() == g[f"ring{n}_counts"].tolist()
        assert hashlib.sha256(part.ring_index.astype("<i8").tobytes()).digest() == \
            g[f"ring{n}_sha"].tobytes()
    assert ring_partition((2, 4)).counts.tolist() == g["ring2x4_counts"].tolist()


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.nn import PolicyNetwork
    with pytest.raises(RuntimeError, match="CUDA"):
        rl.halftone(PolicyNetwork(), np.zeros((4, 4)), np.zeros((4, 4)))
