"""Estimators (REINFORCE, REINFORCE + mean baseline, COMA, local expectation)
and the multitone (L > 2) path, SURVEY §8f row 4.

CPU: the oracle restatement against vectors the reference computed
(tests/golden/make_estimators_golden.py).  GPU: the device kernels
(ht_reward_signal, ht_reinforce_signal, ht_multitone) against the oracle on
the same inputs, plus the host API (rl.*_signal, multitone.*)."""

import numpy as np
import pytest

from conftest import golden
from oracle import htoracle as O
from paper_2304_12152_b200.imagecore import Rng

REL = 1e-4          # signals within 1e-4 relative (normwise)


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def _maps(m, c):
    return O.RewardMaps(m, c, O.hvs_kernel("gaussian"), O.gaussian_kernel(11, 1.5))


# ---------------------------------------------------------------- oracle pins
def test_oracle_binary_estimators_match_reference():
    g = golden("estimators.npz")
    p, c = g["bin_p"], g["bin_c"]
    u = Rng(21).uniforms(p.size).reshape(p.shape)
    fl, ce, pc = O.cast_two_point(p, 2)
    m = O.sample_two_point(fl, ce, pc, u)
    assert np.array_equal(m, g["bin_m"])
    maps = _maps(m, c)
    assert abs(maps.reward - g["bin_reward"][0]) <= 1e-12
    assert _rel(O.le_signal_levels(maps, m, fl, ce, 2), g["bin_le"]) < 1e-10
    assert _rel(O.coma_signal(maps, m, p), g["bin_coma"]) < 1e-10
    assert _rel(O.reinforce_signal(maps.reward, m, p), g["bin_reinforce"]) < 1e-12
    assert _rel(O.reinforce_signal(maps.reward, m, p, 0.0123), g["bin_reinforce_b"]) < 1e-12


@pytest.mark.parametrize("L", [3, 4])
def test_oracle_multitone_sample_and_le_match_reference(L):
    g = golden("estimators.npz")
    v, c = g[f"mt{L}_v"], g[f"mt{L}_c"]
    fl, ce, pc = O.cast_two_point(v, L)
    assert np.array_equal(fl, g[f"mt{L}_floor"]) and np.array_equal(ce, g[f"mt{L}_ceil"])
    assert np.array_equal(pc, g[f"mt{L}_pceil"])
    m = O.sample_two_point(fl, ce, pc, Rng(60 + L).uniforms(v.size).reshape(v.shape))
    assert np.array_equal(m, g[f"mt{L}_m"])
    maps = _maps(m, c)
    assert abs(maps.reward - g[f"mt{L}_reward"][0]) <= 1e-12
    assert _rel(O.le_signal_levels(maps, m, fl, ce, L), g[f"mt{L}_le"]) < 1e-10


def test_oracle_quantize_matches_reference():
    g = golden("estimators.npz")
    for L in range(2, 8):
        assert np.array_equal(O.quantize_multitone(g["q_v"], L), g[f"q_L{L}"])


def test_host_cast_and_quantize_match_reference():
    from paper_2304_12152_b200 import multitone as MT
    from paper_2304_12152_b200 import rl
    g = golden("estimators.npz")
    for L in (3, 4):
        fl, ce, pc = rl._cast_two_point(g[f"mt{L}_v"], L)
        assert np.array_equal(fl, g[f"mt{L}_floor"]) and np.array_equal(ce, g[f"mt{L}_ceil"])
        assert np.array_equal(pc, g[f"mt{L}_pceil"])
        m = MT.sample_multitone(g[f"mt{L}_v"], MT.LevelSet(L), Rng(60 + L))
        assert np.array_equal(m, g[f"mt{L}_m"])
    for L in range(2, 8):
        assert np.array_equal(MT.quantize_multitone(g["q_v"], MT.LevelSet(L)), g[f"q_L{L}"])
    with pytest.raises(ValueError):
        MT.LevelSet(1)
    with pytest.raises(ValueError):
        rl._cast_two_point(np.array([1.5]), 3)


def test_train_config_estimator_rules():
    from paper_2304_12152_b200 import rl
    for est in ("reinforce", "reinforce_meanbaseline", "coma", "local_expectation"):
        rl.TrainConfig(estimator=est).validate()
    rl.TrainConfig(levels=4).validate()
    for bad in (dict(levels=4, estimator="coma"), dict(estimator="nope"), dict(levels=1)):
        with pytest.raises(ValueError):
            rl.TrainConfig(**bad).validate()


# ---------------------------------------------------------------- GPU parity
def _device_signal(p, u, c, levels, estimator, scale=1.0):
    import torch
    from paper_2304_12152_b200.metrics import MetricConfig, reward_signal_device
    from paper_2304_12152_b200.hvs import HvsConfig
    cfg = MetricConfig(hvs=HvsConfig(model="gaussian"))
    dev = torch.device("cuda")
    t = lambda a, dt: torch.from_numpy(np.asarray(a, dt))[None].to(dev)      # noqa: E731
    m, sig, rew = reward_signal_device(t(p, np.float32), t(u, np.float64), t(c, np.float32), cfg,
                                       scale=scale, levels=levels, estimator=estimator)
    return (m[0].double().cpu().numpy(), None if sig is None else sig[0].double().cpu().numpy(),
            float(rew[0]))


@pytest.mark.gpu
@pytest.mark.parametrize("estimator", ["local_expectation", "coma"])
def test_device_binary_signals(estimator):
    g = golden("estimators.npz")
    p, c = g["bin_p"], g["bin_c"]
    u = Rng(21).uniforms(p.size).reshape(p.shape)
    m, sig, rew = _device_signal(p, u, c, 2, estimator, scale=0.5)
    assert np.array_equal(m, g["bin_m"])
    assert abs(rew - g["bin_reward"][0]) <= 1e-9
    want = g["bin_le"] if estimator == "local_expectation" else g["bin_coma"]
    assert _rel(sig, 0.5 * want) < REL


@pytest.mark.gpu
def test_device_reinforce_signals():
    import torch
    from paper_2304_12152_b200.metrics import reinforce_signal_device
    g = golden("estimators.npz")
    p = g["bin_p"]
    dev = torch.device("cuda")
    pd = torch.from_numpy(p.astype(np.float32))[None].to(dev)
    md = torch.from_numpy(g["bin_m"].astype(np.float32))[None].to(dev)
    rd = torch.tensor([g["bin_reward"][0]], dtype=torch.float64, device=dev)
    for base, key in ((0.0, "bin_reinforce"), (0.0123, "bin_reinforce_b")):
        got = reinforce_signal_device(pd, md, rd, base, scale=0.25)[0].double().cpu().numpy()
        # float32 p in both: the reference's clip/1/p on the same values
        assert _rel(got, 0.25 * g[key]) < REL


@pytest.mark.gpu
@pytest.mark.parametrize("L", [3, 4])
def test_device_multitone_sample_and_le(L):
    g = golden("estimators.npz")
    v, c = g[f"mt{L}_v"], g[f"mt{L}_c"]
    u = Rng(60 + L).uniforms(v.size).reshape(v.shape)
    m, sig, rew = _device_signal(v, u, c, L, "local_expectation")
    assert np.array_equal(m, g[f"mt{L}_m"].astype(np.float32))     # m_out is float32
    assert abs(rew - g[f"mt{L}_reward"][0]) <= 1e-9
    assert _rel(sig, g[f"mt{L}_le"]) < REL


@pytest.mark.gpu
def test_host_api_estimators_and_multitone_sample():
    """rl.make_sample / le_signal / coma_signal / reinforce_signal (GPU
    reward context) on the golden inputs, and the eval counts of the reference."""
    from paper_2304_12152_b200 import multitone as MT
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.metrics import MetricConfig
    from paper_2304_12152_b200.hvs import HvsConfig
    g = golden("estimators.npz")
    cfg = MetricConfig(hvs=HvsConfig(model="gaussian"))
    s = rl.make_sample(g["bin_p"], g["bin_c"], None, Rng(21), cfg)
    assert np.array_equal(s.m, g["bin_m"]) and s.ctx.eval_count == 1
    assert _rel(rl.le_signal(s), g["bin_le"]) < REL and s.ctx.eval_count == 1 + s.m.size
    assert _rel(rl.coma_signal(s), g["bin_coma"]) < REL
    assert _rel(rl.reinforce_signal(s, 0.0123), g["bin_reinforce_b"]) < REL
    s4 = MT.make_multitone_sample(g["mt4_v"], g["mt4_c"], None, MT.LevelSet(4), Rng(64), cfg)
    assert np.array_equal(s4.m, g["mt4_m"])
    assert _rel(MT.le_signal_multitone(s4), g["mt4_le"]) < REL
    with pytest.raises(ValueError):
        rl.coma_signal(s4)
    with pytest.raises(ValueError):
        rl.reinforce_signal(s4)


@pytest.mark.gpu
@pytest.mark.parametrize("L", [2, 3, 5])
@pytest.mark.parametrize("impl", [0, 1])
def test_multitone_inference_matches_oracle(L, impl):
    """ht_multitone: level index of the fused forward's p, exact outside a
    1e-3 band around the half-step boundaries (the L=2 rule generalised)."""
    from paper_2304_12152_b200 import multitone as MT
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = PolicyNetwork(32, 2)
    net.init_params(Rng(5), std=0.05)
    r = Rng(9)
    c = r.uniforms(40 * 52).reshape(40, 52).astype(np.float32)
    z = r.gaussians(40 * 52).reshape(40, 52).astype(np.float32)
    m, v = MT.multitone(net, c, z, MT.LevelSet(L), impl=impl)
    params = [p.value for p in net.params()]
    v_ref = O.policy_forward(params, np.stack((c, z)).astype(np.float64)[None])[0, 0]
    assert np.max(np.abs(v - v_ref)) <= 1e-3
    m_ref = O.quantize_multitone(v_ref, L)
    steps = L - 1
    band = np.abs(v_ref * steps + 0.5 - np.round(v_ref * steps + 0.5)) < 1e-3 * steps
    assert np.array_equal(m[~band], m_ref[~band])
    assert set(np.unique(m * steps)) <= set(range(L))
    if L == 2:
        from paper_2304_12152_b200 import rl
        h, _ = rl.halftone(net, c, z, impl=impl)
        assert np.array_equal(m, h)


@pytest.mark.gpu
@pytest.mark.parametrize("estimator,levels", [("coma", 2), ("reinforce", 2),
                                              ("reinforce_meanbaseline", 2),
                                              ("local_expectation", 3)])
def test_train_step_runs_every_estimator(estimator, levels):
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.nn import Adam, PolicyNetwork
    cfg = rl.TrainConfig(iterations=3, batch_size=2, crop_size=16, anisotropy_batch_size=1,
                         channels=8, blocks=1, hvs_size=5, estimator=estimator, levels=levels,
                         multitone_anisotropy=levels > 2)
    r = Rng(4)
    ds = [r.uniforms(24 * 24).reshape(24, 24)]
    net = PolicyNetwork(8, 1)
    rng = Rng(0)
    net.init_params(rng)
    adam = Adam(net.params())
    before = net.flat_values().copy()
    diag = rl.train_step(net, adam, ds, cfg, rng, 0)
    assert np.isfinite(diag["reward"]) and np.isfinite(net.flat_values()).all()
    assert not np.array_equal(before, net.flat_values())


# ------------------------------------------------- unbiasedness (rl.py:139-164)
def _exact_cases():
    g = golden("exact_grad.npz")
    return g, [str(n) for n in g["names"]]


def test_oracle_exact_gradient_matches_reference():
    """The enumeration oracle against the reference's exact_gradient_oracle
    (tests/golden/make_exact_grad_golden.py), incl. the 1x1 identity-filter
    closed form dE[R]/dp = 2c - 1 (R = -(h - c)^2)."""
    g, names = _exact_cases()
    for name in names:
        w_s, hs, hsg, win, L = g[f"{name}_cfg"]
        k, w = O.gaussian_kernel(int(hs), hsg), O.gaussian_kernel(int(win), 1.5)
        got = O.exact_gradient_oracle(g[f"{name}_p"], g[f"{name}_c"], k, w, w_s=w_s, levels=int(L))
        assert _rel(got, g[f"{name}_grad"]) < 1e-12, name
    assert abs(g["identity_1x1_grad"][0, 0] - (2 * g["identity_1x1_c"][0, 0] - 1)) < 1e-15


def _expected_device_signal(p, c, cfg, levels, estimator):
    """Policy-weighted average of the device signal over every joint action
    map (all 2^n maps in one batched launch; map b forced through the
    uniforms: u = 0 selects the upper support point, u ~ 1 the lower)."""
    import torch
    from paper_2304_12152_b200.metrics import reinforce_signal_device, reward_signal_device
    n = p.size
    fl, ce, q = O.cast_two_point(p, levels)
    bits = (np.arange(1 << n)[:, None] >> np.arange(n)[None, :]) & 1
    up = bits.astype(bool).reshape((-1,) + p.shape)
    weight = np.prod(np.where(up, q[None], 1.0 - q[None]).reshape(len(up), -1), axis=1)
    u = np.where(up, 0.0, np.nextafter(1.0, 0.0))
    B = len(up)
    pd = torch.from_numpy(np.broadcast_to(p, up.shape).astype(np.float32).copy()).cuda()
    cd = torch.from_numpy(np.broadcast_to(c, up.shape).astype(np.float32).copy()).cuda()
    ud = torch.from_numpy(u).cuda()
    if estimator == "reinforce":
        m, _, rew = reward_signal_device(pd, ud, cd, cfg, want_signal=False, levels=levels)
        sig = reinforce_signal_device(pd, m, rew, 0.0)
    else:
        m, sig, _ = reward_signal_device(pd, ud, cd, cfg, levels=levels, estimator=estimator)
    assert np.array_equal(m.cpu().numpy(), np.where(up, ce[None], fl[None]).astype(np.float32))
    s = sig.double().cpu().numpy().reshape(B, -1)
    return (weight[:, None] * s).sum(0).reshape(p.shape), (weight[:, None] * np.abs(s)).sum(0).reshape(p.shape)


@pytest.mark.gpu
@pytest.mark.parametrize("estimator", ["local_expectation", "coma", "reinforce"])
def test_device_estimators_unbiased(estimator):
    """The reference's core claim (tests/test_rl.py:108-119): for every
    estimator the policy-weighted average of the injected signal over all
    joint action maps equals minus the exact gradient of the expected
    reward -- here for the device kernels, against the reference-computed
    gradients; tolerance: fp32 signal rounding (1e-6 of sum_b w_b |s_b|)."""
    from paper_2304_12152_b200.hvs import HvsConfig
    from paper_2304_12152_b200.metrics import MetricConfig
    g, names = _exact_cases()
    for name in names:
        w_s, hs, hsg, win, L = g[f"{name}_cfg"]
        if estimator != "local_expectation" and L != 2:
            continue                      # COMA / REINFORCE are binary-policy estimators
        cfg = MetricConfig(w_s=float(w_s), ssim_window=int(win),
                           hvs=HvsConfig(model="gaussian", size=int(hs), sigma=float(hsg)))
        got, mag = _expected_device_signal(g[f"{name}_p"], g[f"{name}_c"], cfg, int(L), estimator)
        want = -g[f"{name}_grad"]
        assert np.all(np.abs(got - want) <= 1e-6 * mag + 1e-12), (name, got, want)


@pytest.mark.gpu
def test_rl_exact_gradient_oracle_matches_reference():
    """rl.exact_gradient_oracle (rewards of all 2^n maps from the device
    reward kernel) against the reference's values; the 20-pixel guard."""
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.hvs import HvsConfig
    from paper_2304_12152_b200.metrics import MetricConfig
    g, names = _exact_cases()
    for name in names:
        w_s, hs, hsg, win, L = g[f"{name}_cfg"]
        cfg = MetricConfig(w_s=float(w_s), ssim_window=int(win),
                           hvs=HvsConfig(model="gaussian", size=int(hs), sigma=float(hsg)))
        got = rl.exact_gradient_oracle(g[f"{name}_p"], g[f"{name}_c"], cfg, level_count=int(L))
        assert _rel(got, g[f"{name}_grad"]) < 1e-6, (name, _rel(got, g[f"{name}_grad"]))
    with pytest.raises(ValueError):
        rl.exact_gradient_oracle(np.full((3, 7), 0.5), np.zeros((3, 7)))
