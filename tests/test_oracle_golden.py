"""Pin the CPU oracle (oracle/htoracle.py) to the real reference's outputs.

The fixtures were produced by tests/golden/make_golden.py running
/root/reference (htlab) in the build container.  Tolerances follow the
reference's own oracle tests (test_nn.py:43-56 1e-12, test_metrics.py 1e-12 /
1e-13, test_spectral.py 1e-10): two float64 implementations of the same math.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import htoracle as O


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# --------------------------------------------------------------------- RNG
class TestRng:
    def test_splitmix_and_xoshiro_vectors(self):
        g = golden("rng.npz")
        s, outs = 0, []
        for _ in range(3):
            s, z = O.splitmix64(s)
            outs.append(z)
        assert outs == [int(v) for v in g["splitmix"]]
        r = O.Rng(0)
        r.set_state_words((1, 2, 3, 4))
        assert [r.next_uint64() for _ in range(6)] == [int(v) for v in g["xoshiro1234"]]
        assert list(O.Rng(42).state_words()) == [int(v) for v in g["state_seed42"]]

    def test_uniform_gaussian_noise_randint(self):
        g = golden("rng.npz")
        assert np.array_equal(O.Rng(7).uniforms(9), g["uniforms_seed7"])
        assert np.array_equal(O.Rng(11).gaussians(7), g["gaussians_seed11"])
        assert np.array_equal(O.gaussian_noise_map(O.Rng(5), 8, 6), g["noise_seed5_w8_h6"])
        r = O.Rng(3)
        assert [r.randint(n) for n in (1, 2, 7, 100, 1 << 20)] == list(g["randint_seed3"])


# --------------------------------------------------------------------- policy net
def _params(ch, nb, std, seed=0):
    return O.init_params(O.Rng(seed), ch, nb, 2, std)


class TestForward:
    @pytest.mark.parametrize("std", [0.01, 0.05])
    def test_small_full_arch(self, std):
        g = golden("forward.npz")
        c, z = g["small_c"].astype(np.float64), g["small_z"].astype(np.float64)
        _, p = O.halftone(_params(32, 16, std), c, z)
        assert np.max(np.abs(p - g[f"small_p_std{std}"])) < 1e-12

    def test_small_mini_arch(self):
        g = golden("forward.npz")
        _, p = O.halftone(_params(8, 2, 0.05), g["small_c"], g["small_z"])
        assert np.max(np.abs(p - g["small_p_mini"])) < 1e-12

    @pytest.mark.parametrize("shape", ["1x1", "3x5", "7x2", "37x131"])
    def test_ragged(self, shape):
        g = golden("forward.npz")
        _, p = O.halftone(_params(32, 16, 0.05), g[f"rag_{shape}_c"], g[f"rag_{shape}_z"])
        assert np.max(np.abs(p - g[f"rag_{shape}_p"])) < 1e-12

    @pytest.mark.parametrize("std", [0.01, 0.05])
    def test_config1_256(self, std):
        # BASELINE config 1 at full size (golden p stored as float32)
        g = golden("forward.npz")
        _, p = O.halftone(_params(32, 16, std), g["cfg1_c"], g["cfg1_z"])
        assert np.max(np.abs(p - g[f"cfg1_p_std{std}"])) < 1e-7
        band = np.mean(np.abs(p - 0.5) < 1e-3)
        assert abs(band - g[f"cfg1_band_std{std}"][0]) < 1e-4

    def test_conv_convention_impulse(self):
        # weight cell (0,1) reads the pixel one row up (reference test_nn.py:33-41)
        w = np.zeros((1, 1, 3, 3))
        w[0, 0, 0, 1] = 1.0
        x = np.arange(12.0).reshape(1, 1, 3, 4)
        out = O.conv_forward(x, w, np.zeros(1))
        assert np.array_equal(out[0, 0, 0], np.zeros(4))
        assert np.array_equal(out[0, 0, 1:], x[0, 0, :2])

    def test_threshold_ties_go_white(self):
        assert O.threshold(np.array([0.5, np.nextafter(0.5, 0), 0.7])).tolist() == [1, 0, 1]


class TestBackward:
    @pytest.mark.parametrize("tag,ch,nb", [("mini", 8, 2), ("full", 32, 16)])
    def test_grads_match_reference(self, tag, ch, nb):
        g = golden("backward.npz")
        params = O.init_params(O.Rng(2), ch, nb, 2, 0.05)
        p, cache = O.policy_forward(params, g[f"{tag}_x"], keep=True)
        assert np.max(np.abs(p - g[f"{tag}_p"])) < 1e-12
        dx, grads = O.policy_backward(params, cache, g[f"{tag}_dp"])
        assert rel(dx, g[f"{tag}_dx"]) < 1e-10
        flat = np.concatenate([q.ravel() for q in grads])
        pr = np.random.default_rng(1234).standard_normal((4, flat.size))
        assert rel(pr @ flat, g[f"{tag}_grad_probe"]) < 1e-10
        norms = np.array([np.linalg.norm(q) for q in grads])
        assert np.allclose(norms, g[f"{tag}_grad_norms"], rtol=1e-10, atol=1e-300)
        if tag == "mini":
            assert rel(flat, g["mini_grad"]) < 1e-10

    def test_fd_gradient_tiny(self):
        params = O.init_params(O.Rng(0), 3, 1, 2, 0.3)
        x = O.Rng(1).uniforms(2 * 2 * 5 * 5).reshape(2, 2, 5, 5)
        G = O.Rng(2).gaussians(50).reshape(2, 1, 5, 5)
        p, cache = O.policy_forward(params, x, keep=True)
        _, grads = O.policy_backward(params, cache, G)
        w = params[2]
        idx = (1, 2, 0, 1)
        keep = w[idx]
        w[idx] = keep + 1e-6
        hi = float(np.sum(G * O.policy_forward(params, x)))
        w[idx] = keep - 1e-6
        lo = float(np.sum(G * O.policy_forward(params, x)))
        w[idx] = keep
        assert abs((hi - lo) / 2e-6 - grads[2][idx]) < 1e-6 * max(1.0, abs(grads[2][idx]))


# --------------------------------------------------------------------- reward / LE
class TestReward:
    @pytest.mark.parametrize("model", ["nasanen", "gaussian"])
    def test_maps_delta_le(self, model):
        g = golden("reward.npz")
        k = O.hvs_kernel(model)
        assert np.max(np.abs(k - g[f"{model}_kernel"])) < 1e-15
        w = O.gaussian_kernel(11, 1.5)
        assert np.max(np.abs(w - g["ssim_window"])) < 1e-16
        maps = O.RewardMaps(g["m"], g["c"], k, w)
        r = g[f"{model}_reward"]
        assert abs(maps.reward - r[0]) < 1e-13 and abs(maps.mse - r[1]) < 1e-13
        assert np.max(np.abs(maps.reward_map - g[f"{model}_reward_map"])) < 1e-13
        d = maps.delta_map(1.0 - g["m"])
        assert np.max(np.abs(d - g[f"{model}_delta_flip"])) < 1e-15
        le = O.le_signal(maps, g["m"])
        assert np.max(np.abs(le - g[f"{model}_le"])) < 1e-15

    @pytest.mark.parametrize("model", ["nasanen", "gaussian"])
    @pytest.mark.parametrize("tag", ["h2", "h4"])
    def test_context_maps_float64(self, model, tag):
        """The float64 RewardContext / delta_map fixture (context.npz: inputs
        that are not float32-representable, binary and 4-level h) against the
        oracle's restatement."""
        g = golden("context.npz")
        key = f"{model}_{tag}"
        maps = O.RewardMaps(g[tag], g["c"], O.hvs_kernel(model), O.gaussian_kernel(11, 1.5))
        for ours, ref in (("f_c", "f_c"), ("mu_c", "mu_c"), ("scc", "scc"), ("sigma_c", "sigma_c"),
                          ("e", "e"), ("mu_h", "mu_h"), ("shh", "shh"), ("shc", "shc"),
                          ("ssim", "ssim"), ("cssim", "cssim_map"), ("reward_map", "reward_map")):
            assert np.max(np.abs(getattr(maps, ours) - g[f"{key}_{ref}"])) < 1e-13, ours
        mse, _, rew = g[f"{key}_scalars"]
        assert abs(maps.mse - mse) < 1e-14 and abs(maps.reward - rew) < 1e-14
        other = 1.0 - g["h2"] if tag == "h2" else g["other4"]
        d = maps.delta_map(other)
        assert np.max(np.abs(d - g[f"{key}_delta"])) < 1e-15

    def test_sampling_draw_order(self):
        g = golden("reward.npz")
        u = O.Rng(10).uniforms(64 * 64).reshape(64, 64)
        m = O.sample_actions(g["s64_p"], u)
        assert np.array_equal(m, g["s64_m"])
        maps = O.RewardMaps(m, g["s64_c"], O.hvs_kernel("gaussian"), O.gaussian_kernel(11, 1.5))
        # the contone has flat rectangles: sigma_c = 2 sqrt(E[c^2] - mu_c^2) of a
        # catastrophically cancelled ~1e-17 variance differs at ~1e-8 between
        # two summation orders, so compare at 1e-10 here (1e-13 elsewhere)
        assert abs(maps.reward - g["s64_reward"][0]) < 1e-10
        le = O.le_signal(maps, m)
        assert np.max(np.abs(le - g["s64_le"])) < 1e-9 * np.abs(g["s64_le"]).max()


# --------------------------------------------------------------------- spectral
class TestSpectral:
    @pytest.mark.parametrize("n", [4, 32, 256])
    def test_ring_partition(self, n):
        import hashlib
        g = golden("spectral.npz")
        ring, radii, counts = O.ring_partition((n, n))
        assert counts.tolist() == g[f"ring{n}_counts"].tolist()
        assert radii.tolist() == g[f"ring{n}_radii"].tolist()
        sha = hashlib.sha256(ring.astype("<i8").tobytes()).digest()
        assert sha == g[f"ring{n}_sha"].tobytes()

    def test_loss_and_grad(self):
        g = golden("spectral.npz")
        part = O.ring_partition((32, 32))
        assert abs(O.anisotropy_loss(g["x32"], part) / g["x32_loss"][0] - 1) < 1e-12
        assert rel(O.anisotropy_loss_backward(g["x32"], part), g["x32_grad"]) < 1e-12
        part = O.ring_partition((256, 256))
        x = g["x256"].astype(np.float64)
        assert abs(O.anisotropy_loss(x, part) / g["x256_loss"][0] - 1) < 1e-12
        gr = O.anisotropy_loss_backward(x, part)
        assert abs(np.linalg.norm(gr) / g["x256_grad_norm"][0] - 1) < 1e-12
        assert np.max(np.abs(gr[:16, :16] - g["x256_grad_crop"])) < 1e-12 * np.abs(gr).max()

    def test_rapsd(self):
        g = golden("spectral.npz")
        part = O.ring_partition((32, 32))
        power, anis, dc = O.rapsd(O.periodogram(g["h32"]), part)
        assert np.allclose(power, g["h32_power"], rtol=1e-12, atol=0)
        assert np.allclose(anis, g["h32_anis"], rtol=1e-10, atol=0, equal_nan=True)
        assert abs(dc - g["h32_dc"][0]) < 1e-12


# --------------------------------------------------------------------- training step
class TestTrainStep:
    @pytest.mark.parametrize("tag,ch,nb,bs,crop,ba", [("mini", 8, 2, 2, 24, 2),
                                                      ("full", 32, 16, 2, 32, 1)])
    def test_one_step(self, tag, ch, nb, bs, crop, ba):
        g = golden("train.npz")
        rng = O.Rng(0)
        params = O.init_params(rng, ch, nb, 2, 0.01)      # rl.py:290-293 order
        assert list(rng.state_words()) == [int(v) for v in g[f"{tag}_state0"]]
        p0 = np.concatenate([q.ravel() for q in params])
        ds = list(g[f"{tag}_ds"])
        st = {"m": [np.zeros_like(q) for q in params],
              "v": [np.zeros_like(q) for q in params], "t": 0}
        cfg = dict(batch_size=bs, crop_size=crop, anisotropy_batch_size=ba, w_s=0.06,
                   w_a=0.002, iterations=10, lr_start=3e-4, lr_end=1e-5)
        diag, grads = O.train_step(params, st, ds, cfg, rng, 0,
                                   O.hvs_kernel("gaussian"), O.gaussian_kernel(11, 1.5))
        assert list(rng.state_words()) == [int(v) for v in g[f"{tag}_state1"]]
        d = g[f"{tag}_diag"]
        assert abs(diag["reward"] - d[0]) < 1e-12
        assert abs(diag["l_as"] / d[1] - 1) < 1e-9
        assert abs(diag["bin_gap"] - d[2]) < 1e-12 and diag["lr"] == d[3]
        flat = np.concatenate([q.ravel() for q in grads])
        pr = np.random.default_rng(1234).standard_normal((4, flat.size))
        assert rel(pr @ flat, g[f"{tag}_grad_probe"]) < 1e-9
        p1 = np.concatenate([q.ravel() for q in params])
        assert rel(pr @ (p1 - p0), g[f"{tag}_dparam_probe"]) < 1e-9
