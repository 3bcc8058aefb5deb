"""GPU parity of the training path (K2-K7) against the reference, staged.

north_star tolerance: losses and gradients within 1e-4 relative.  Gradient
vectors are compared normwise (and by fixed random probes, see
tests/golden/make_golden.py); the training forward/backward run in fp32.
Following SURVEY.md §0 finding 5, the estimator and backward are first
checked on identical inputs, then a whole train_step end to end.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

REL = 1e-4


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _net(ch, nb, std, seed):
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = PolicyNetwork(ch, nb)
    net.init_params(Rng(seed), std=std)
    return net


@pytest.mark.parametrize("tag,ch,nb", [("mini", 8, 2), ("full", 32, 16)])
def test_forward_backward_vs_reference(tag, ch, nb):
    g = golden("backward.npz")
    net = _net(ch, nb, 0.05, 2)
    p = net.forward(g[f"{tag}_x"])
    assert np.max(np.abs(p - g[f"{tag}_p"])) < 2e-5
    net.zero_grad()
    dx = net.backward(g[f"{tag}_dp"])
    assert rel(dx, g[f"{tag}_dx"]) < REL
    flat = np.concatenate([q.grad.ravel() for q in net.params()])
    pr = np.random.default_rng(1234).standard_normal((4, flat.size))
    assert rel(pr @ flat, g[f"{tag}_grad_probe"]) < REL
    norms = np.array([np.linalg.norm(q.grad) for q in net.params()])
    ok = g[f"{tag}_grad_norms"] > 1e-12
    assert np.all(np.abs(norms[ok] / g[f"{tag}_grad_norms"][ok] - 1) < REL)
    if tag == "mini":
        assert rel(flat, g["mini_grad"]) < REL
    else:
        head = np.concatenate([q.grad.ravel() for q in net.params()[:4]])
        tail = np.concatenate([q.grad.ravel() for q in net.params()[-4:]])
        assert rel(head, g["full_grad_head"]) < REL and rel(tail, g["full_grad_tail"]) < REL


def test_backward_accumulates_like_reference():
    g = golden("backward.npz")
    net = _net(8, 2, 0.05, 2)
    net.forward(g["mini_x"])
    net.zero_grad()
    net.backward(g["mini_dp"])
    net.backward(g["mini_dp"])
    flat = np.concatenate([q.grad.ravel() for q in net.params()])
    assert rel(flat, 2 * g["mini_grad"]) < REL


@pytest.mark.parametrize("model", ["nasanen", "gaussian"])
def test_reward_delta_le(model):
    from paper_2304_12152_b200 import metrics, rl
    from paper_2304_12152_b200.hvs import HvsConfig
    g = golden("reward.npz")
    cfg = metrics.MetricConfig(hvs=HvsConfig(model=model))
    ctx = metrics.reward(g["m"], g["c"], cfg)
    assert abs(ctx.reward / g[f"{model}_reward"][0] - 1) < 1e-10
    d = metrics.delta_map(ctx, 1.0 - g["m"])
    assert rel(d, g[f"{model}_delta_flip"]) < 1e-6       # fp32 signal storage
    s = rl.EpisodeSample(c=g["c"], z=None, p=None, m=g["m"], floor_vals=np.zeros_like(g["m"]),
                         ceil_vals=np.ones_like(g["m"]), p_ceil=None, level_count=2, ctx=ctx)
    assert rel(rl.le_signal(s), g[f"{model}_le"]) < 1e-6


def test_make_sample_draw_order_and_le():
    from paper_2304_12152_b200 import metrics, rl
    from paper_2304_12152_b200.hvs import HvsConfig
    from paper_2304_12152_b200.imagecore import Rng
    g = golden("reward.npz")
    s = rl.make_sample(g["s64_p"], g["s64_c"], None, Rng(10),
                       metrics.MetricConfig(hvs=HvsConfig(model="gaussian")))
    assert np.array_equal(s.m, g["s64_m"])
    assert abs(s.ctx.reward / g["s64_reward"][0] - 1) < 1e-9
    assert rel(rl.le_signal(s), g["s64_le"]) < 1e-6


def test_anisotropy_loss_and_grad():
    from paper_2304_12152_b200 import spectral
    g = golden("spectral.npz")
    assert abs(spectral.anisotropy_loss(g["x32"]) / g["x32_loss"][0] - 1) < 1e-9
    assert rel(spectral.anisotropy_loss_backward(g["x32"]), g["x32_grad"]) < 1e-6
    x = g["x256"].astype(np.float64)
    assert abs(spectral.anisotropy_loss(x) / g["x256_loss"][0] - 1) < 1e-9
    gr = spectral.anisotropy_loss_backward(x)
    assert abs(np.linalg.norm(gr) / g["x256_grad_norm"][0] - 1) < 1e-6
    pr = np.random.default_rng(1234).standard_normal((4, gr.size))
    assert rel(pr @ gr.ravel(), g["x256_grad_probe"]) < 1e-6


def test_anisotropy_float64_api_is_float64():
    """spectral.anisotropy_loss(_backward) on float64 arrays compute in
    float64 (no float32 round trip): 1e-12 against the reference's goldens."""
    from paper_2304_12152_b200 import spectral
    g = golden("spectral.npz")
    assert abs(spectral.anisotropy_loss(g["x32"]) / g["x32_loss"][0] - 1) < 1e-12
    assert rel(spectral.anisotropy_loss_backward(g["x32"]), g["x32_grad"]) < 1e-12
    x = g["x256"].astype(np.float64)
    assert abs(spectral.anisotropy_loss(x) / g["x256_loss"][0] - 1) < 1e-12
    gr = spectral.anisotropy_loss_backward(x)
    assert abs(np.linalg.norm(gr) / g["x256_grad_norm"][0] - 1) < 1e-12
    assert rel(gr[:16, :16], g["x256_grad_crop"]) < 1e-10


def test_periodogram_and_rapsd_of_periodogram():
    """spectral.periodogram (spectral.py:17-24) and spectral.rapsd(p_hat,
    part) (spectral.py:74-88) against the reference's rapsd(periodogram(h))
    and the oracle's periodogram; Parseval sum(P) = sum(x^2)."""
    from oracle import htoracle as O
    from paper_2304_12152_b200 import spectral
    g = golden("spectral.npz")
    P = spectral.periodogram(g["h32"])
    assert P.dtype == np.float64 and P.shape == (32, 32)
    assert np.allclose(P, O.periodogram(g["h32"]), rtol=1e-12, atol=1e-12)
    assert abs(P.sum() - np.sum(g["h32"] ** 2)) < 1e-9
    part = spectral.ring_partition((32, 32))
    cur = spectral.rapsd(P, part)
    assert np.allclose(cur.power, g["h32_power"], rtol=1e-12, atol=0)
    assert np.allclose(cur.anisotropy, g["h32_anis"], rtol=1e-10, atol=0, equal_nan=True)
    assert abs(cur.dc_power - g["h32_dc"][0]) < 1e-12
    assert np.array_equal(cur.radii, part.radii) and np.array_equal(cur.counts, part.counts)
    rng = np.random.default_rng(3)
    x = rng.standard_normal((7, 12))                 # ragged, odd height
    assert np.allclose(spectral.periodogram(x), O.periodogram(x), rtol=1e-12, atol=1e-12)
    with pytest.raises(ValueError):
        spectral.periodogram(np.zeros((0, 4)))
    with pytest.raises(ValueError):
        spectral.rapsd(P, spectral.ring_partition((16, 32)))


def test_rapsd_of_halftone():
    from paper_2304_12152_b200 import spectral
    g = golden("spectral.npz")
    cur = spectral.image_rapsd(g["h32"])
    assert np.allclose(cur.power, g["h32_power"], rtol=1e-9, atol=0)
    assert np.allclose(cur.anisotropy, g["h32_anis"], rtol=1e-7, atol=0, equal_nan=True)
    assert abs(cur.dc_power - g["h32_dc"][0]) < 1e-9


def test_adam_matches_reference():
    from oracle import htoracle as O
    from paper_2304_12152_b200.nn import Adam, Parameter
    rng = np.random.default_rng(0)
    vals = [rng.standard_normal((4, 3)), rng.standard_normal(5)]
    params = [Parameter(v.copy()) for v in vals]
    ref_vals = [v.copy() for v in vals]
    m = [np.zeros_like(v) for v in vals]
    v_ = [np.zeros_like(v) for v in vals]
    adam = Adam(params)
    t = 0
    for step in range(3):
        grads = [rng.standard_normal(v.shape) for v in vals]
        for p, gr in zip(params, grads):
            p.grad[...] = gr
        adam.step(1e-3)
        t = O.adam_step(ref_vals, grads, m, v_, t, 1e-3)
    for p, r in zip(params, ref_vals):
        assert np.max(np.abs(p.value - r)) < 1e-15


@pytest.mark.parametrize("tag,ch,nb,bs,crop,ba", [("mini", 8, 2, 2, 24, 2),
                                                  ("full", 32, 16, 2, 32, 1)])
def test_train_step_vs_reference(tag, ch, nb, bs, crop, ba):
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import Adam, PolicyNetwork
    g = golden("train.npz")
    cfg = rl.TrainConfig(iterations=10, batch_size=bs, crop_size=crop, channels=ch, blocks=nb,
                         anisotropy_batch_size=ba, hvs_model="gaussian")
    rng = Rng(cfg.seed)
    net = PolicyNetwork(ch, nb)
    adam = Adam(net.params())
    net.init_params(rng)
    p0 = net.flat_values()
    assert list(rng.state_words()) == [int(v) for v in g[f"{tag}_state0"]]
    diag = rl.train_step(net, adam, list(g[f"{tag}_ds"]), cfg, rng, 0)
    assert list(rng.state_words()) == [int(v) for v in g[f"{tag}_state1"]]
    d = g[f"{tag}_diag"]
    assert abs(diag["reward"] / d[0] - 1) < 1e-6
    assert abs(diag["l_as"] / d[1] - 1) < REL
    assert abs(diag["bin_gap"] / d[2] - 1) < 1e-5
    assert diag["lr"] == d[3]
    gr = net._last_grad.cpu().numpy()
    pr = np.random.default_rng(1234).standard_normal((4, gr.size))
    assert rel(pr @ gr, g[f"{tag}_grad_probe"]) < REL
    p1 = net.flat_values()
    if tag == "mini":
        assert rel(gr, g["mini_grad"]) < REL
        # Adam's first step is ~ -lr*sign(g): compare where the sign is stable
        stable = np.abs(g["mini_grad"]) > 1e-7
        assert np.max(np.abs((p1 - g["mini_p1"])[stable])) < 1e-9
    dn = np.array([np.linalg.norm(a) for a in np.split(p1 - p0, np.cumsum(
        [q.value.size for q in net.params()])[:-1])])
    assert np.all(np.abs(dn / g[f"{tag}_dparam_norms"] - 1) < 1e-3)


def test_train_step_nonfinite_raises_before_update():
    """A non-finite logit (nn.py:147-148) raises FloatingPointError from
    train_step with the parameters, the Adam state and the RNG stream where
    the reference leaves them (its forward raises before backward / Adam).
    The device forward only flags it; train_step checks once per step."""
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import Adam, PolicyNetwork
    g = golden("train.npz")
    cfg = rl.TrainConfig(iterations=10, batch_size=2, crop_size=24, channels=8, blocks=2,
                         anisotropy_batch_size=2, hvs_model="gaussian")
    ds = list(g["mini_ds"])
    net = PolicyNetwork(8, 2)
    adam = Adam(net.params())
    rng = Rng(cfg.seed)
    net.init_params(rng)
    net.conv_out.bias.value[0] = np.inf          # every logit non-finite
    expect = Rng(0)
    expect.set_state_words(rng.state_words())
    rl.draw_batch(ds, cfg, expect)               # the reference raises right after this
    p0 = net.flat_values()
    with pytest.raises(FloatingPointError):
        rl.train_step(net, adam, ds, cfg, rng, 0)
    assert np.array_equal(net.flat_values(), p0, equal_nan=True)
    assert adam.t == 0
    assert rng.state_words() == expect.state_words()


def test_train_step_nonfinite_two_ranks_both_flag_marl(monkeypatch):
    """Data parallel: when two ranks both see a non-finite MARL logit, the
    summed flags still name the MARL forward (separate statistics slots), so
    the RNG is rewound to where the reference's first forward raises."""
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import Adam, PolicyNetwork
    g = golden("train.npz")
    cfg = rl.TrainConfig(iterations=10, batch_size=2, crop_size=24, channels=8, blocks=2,
                         anisotropy_batch_size=2, hvs_model="gaussian")
    ds = list(g["mini_ds"])
    net = PolicyNetwork(8, 2)
    rng = Rng(cfg.seed)
    net.init_params(rng)
    net.conv_out.bias.value[0] = np.inf
    expect = Rng(0)
    expect.set_state_words(rng.state_words())
    rl.draw_batch(ds, cfg, expect)

    def fake_allreduce(*tensors, group=None):    # a second rank with the same flags
        for t in tensors:
            t.mul_(2.0)
        return tensors

    monkeypatch.setattr(rl, "_dist_info", lambda group=None: (0, 2))
    monkeypatch.setattr(rl, "allreduce_sum_", fake_allreduce)
    with pytest.raises(FloatingPointError):
        rl.train_step(net, Adam(net.params()), ds, cfg, rng, 0, prefetch=False)
    assert rng.state_words() == expect.state_words()


def test_train_step_prefetch_false_draws_afresh():
    """prefetch=False after a prefetching step: the batch is drawn from the
    (edited) dataset, not taken from the prepared one."""
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import Adam, PolicyNetwork
    g = golden("train.npz")
    cfg = rl.TrainConfig(iterations=10, batch_size=2, crop_size=24, channels=8, blocks=2,
                         anisotropy_batch_size=2, hvs_model="gaussian")

    def run(edit):
        ds = [a.copy() for a in g["mini_ds"]]
        net = PolicyNetwork(8, 2)
        adam = Adam(net.params())
        rng = Rng(cfg.seed)
        net.init_params(rng)
        rl.train_step(net, adam, ds, cfg, rng, 0)          # prefetches step 1's batch
        if edit:
            for a in ds:
                a[...] = 1.0 - a                           # in place: same arrays
        d = rl.train_step(net, adam, ds, cfg, rng, 1, prefetch=False)
        rl.reset_prefetch()
        return d["reward"]

    fresh = run(True)
    rl.reset_prefetch()
    ds = [1.0 - a for a in g["mini_ds"]]
    net = PolicyNetwork(8, 2)
    adam = Adam(net.params())
    rng = Rng(cfg.seed)
    net.init_params(rng)
    rl.train_step(net, adam, [a.copy() for a in g["mini_ds"]], cfg, rng, 0, prefetch=False)
    want = rl.train_step(net, adam, ds, cfg, rng, 1, prefetch=False)["reward"]
    assert abs(fresh - want) <= 1e-9 * max(1.0, abs(want))


def test_train_step_prefetch_is_transparent():
    """train_step prepares the next step's batch from a copy of the RNG
    stream while the GPU works, and queues that batch's forward after Adam;
    with or without it, three steps draw the same stream (RNG state bit for
    bit) and give the same parameters and diagnostics (to the run-to-run
    noise of atomic sums), and a dataset image replaced between steps (or an
    RNG moved by the caller) makes the next step draw afresh, a weight edited
    by the caller makes it recompute the forward."""
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import Adam, PolicyNetwork
    g = golden("train.npz")
    cfg = rl.TrainConfig(iterations=10, batch_size=2, crop_size=24, channels=8, blocks=2,
                         anisotropy_batch_size=2, hvs_model="gaussian")

    def run(prefetch, swap=False, poke=False, edit=False):
        ds = list(g["mini_ds"])
        net = PolicyNetwork(8, 2)
        adam = Adam(net.params())
        rng = Rng(cfg.seed)
        net.init_params(rng)
        rows = []
        for t in range(3):
            if swap and t == 1:
                ds[0] = ds[0][::-1].copy()        # a different image in the same list
            if poke and t == 2:
                rng.uniform()                      # the caller draws from the stream
            if edit and t == 1:
                net.params()[0].value[0, 0, 1, 1] += 1e-2   # the caller edits a weight (the
                #                                    forward queued by step 0 must be dropped)
            rows.append(rl.train_step(net, adam, ds, cfg, rng, t, prefetch=prefetch))
        return net.flat_values(), rows, rng.state_words()

    # gradients are summed with fp64 atomics (order varies run to run: two
    # runs of the same path differ by ~1e-18); the draws must match exactly
    for kw in ({}, {"swap": True}, {"poke": True}, {"edit": True}):
        a = run(True, **kw)
        b = run(False, **kw)
        assert a[2] == b[2], kw
        assert np.max(np.abs(a[0] - b[0])) < 1e-15, kw
        for ra, rb in zip(a[1], b[1]):
            for key in ("reward", "l_as", "bin_gap"):
                assert abs(ra[key] - rb[key]) <= 1e-12 * max(1.0, abs(rb[key])), (kw, key)
            assert ra["lr"] == rb["lr"] and ra["iteration"] == rb["iteration"]


def test_host_parameter_edits_between_steps_reach_the_device():
    """The device copy of the parameters follows the host Parameter arrays
    (nn.py's API surface): after a train_step pulled the Adam update back,
    an in-place edit of one tensor's .value -- and a whole-array replace of
    another's contents -- must be seen by the next forward, which must then
    equal the oracle forward with the edited parameters; an untouched net
    must not re-upload."""
    import torch

    from oracle import htoracle as O
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import Adam, PolicyNetwork
    g = golden("train.npz")
    cfg = rl.TrainConfig(iterations=10, batch_size=2, crop_size=24, channels=8, blocks=2,
                         anisotropy_batch_size=2, hvs_model="gaussian")
    net = PolicyNetwork(8, 2)
    adam = Adam(net.params())
    rng = Rng(cfg.seed)
    net.init_params(rng)
    rl.train_step(net, adam, list(g["mini_ds"]), cfg, rng, 0)
    r = Rng(9)
    x = np.stack((r.uniforms(20 * 22).reshape(20, 22), r.gaussians(20 * 22).reshape(20, 22)))[None]
    x = x.astype(np.float32).astype(np.float64)
    xd = torch.from_numpy(x.astype(np.float32)).cuda()
    uploaded = net._uploaded
    p0 = net.forward_device(xd).double().cpu().numpy()
    assert net._uploaded is uploaded                      # nothing changed: no re-upload
    ps = net.params()
    ps[0].value[0, 1, 2, 2] += 0.25                        # in place, one element
    ps[-2].value[...] = ps[-2].value * 0.5                 # whole tensor
    p1 = net.forward_device(xd).double().cpu().numpy()
    ref = O.policy_forward([q.value for q in ps], x)
    assert np.max(np.abs(p1 - ref[:, 0])) < 2e-5
    assert np.max(np.abs(p1 - p0)) > 1e-4
