"""GPU parity of the drop-in API surface around the hot path.

* metrics.RewardContext (metrics.py:165-204): every map and scalar, float64
  inputs kept float64, against the REAL reference's values
  (tests/golden/make_context_golden.py), binary and 4-level action maps, both
  HVS models; metrics.delta_map (metrics.py:333-392) likewise.
* nn.Conv2d / ResidualBlock .forward / .backward (nn.py:36-103) and
  PolicyNetwork(in_channels != 2) forward / backward (nn.py:109-160),
  float64 on the device, against the oracle's float64 restatement; the
  reference's conv-convention impulse (test_nn.py:33-41).
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

MAPS = ("f_c", "mu_c", "scc", "sigma_c", "f_h", "e", "sq_err", "mu_h", "shh", "shc",
        "cssim_map", "reward_map")


@pytest.mark.parametrize("model", ["nasanen", "gaussian"])
@pytest.mark.parametrize("tag", ["h2", "h4"])
def test_reward_context_maps_match_reference(model, tag):
    from paper_2304_12152_b200 import hvs, metrics
    g = golden("context.npz")
    key = f"{model}_{tag}"
    cfg = metrics.MetricConfig(hvs=hvs.HvsConfig(model=model))
    ctx = metrics.reward(g[tag], g["c"], cfg, region="full")
    for m in MAPS:
        got = getattr(ctx, m)
        assert got.dtype == np.float64 and got.shape == g["c"].shape
        assert np.allclose(got, g[f"{key}_{m}"], rtol=1e-12, atol=1e-13), m
    for name, ref in (("ssim", "ssim"), ("luminance", "lum"), ("contrast", "con"),
                      ("structure", "str")):
        assert np.allclose(getattr(ctx.ssim_maps, name), g[f"{key}_{ref}"], rtol=1e-12, atol=1e-13)
    mse, css, rew = g[f"{key}_scalars"]
    assert abs(ctx.mse - mse) <= 1e-13 * max(1.0, abs(mse))
    assert abs(ctx.cssim_scalar - css) <= 1e-13
    assert abs(ctx.reward - rew) <= 1e-13
    assert abs(ctx.reward - float(ctx.reward_map.mean())) <= 1e-12   # test_metrics.py:236-241
    assert ctx.n_region == g["c"].size and ctx.eval_count == 1
    other = 1.0 - g["h2"] if tag == "h2" else g["other4"]
    d = metrics.delta_map(ctx, other)
    ref = g[f"{key}_delta"]
    assert d.dtype == np.float64
    assert np.allclose(d, ref, rtol=1e-9, atol=1e-15 * np.abs(ref).max())
    assert ctx.eval_count == 1 + g["c"].size


def test_conv2d_impulse_convention():
    """test_nn.py:33-41: weight (0, 1) reads the pixel one row up."""
    from paper_2304_12152_b200.nn import Conv2d
    conv = Conv2d(1, 1)
    conv.weight.value[0, 0, 0, 1] = 1.0
    x = np.zeros((1, 1, 5, 5))
    x[0, 0, 2, 2] = 1.0
    out = conv.forward(x)
    want = np.zeros((1, 1, 5, 5))
    want[0, 0, 3, 2] = 1.0
    assert np.array_equal(out, want)


@pytest.mark.parametrize("ci,co,shape", [(2, 5, (2, 7, 9)), (3, 1, (1, 1, 1)), (4, 4, (3, 6, 2))])
def test_conv2d_forward_backward_float64(ci, co, shape):
    from oracle import htoracle as O
    from paper_2304_12152_b200.nn import Conv2d
    rng = np.random.default_rng(ci * 10 + co)
    b, h, w = shape
    conv = Conv2d(ci, co)
    conv.weight.value[...] = rng.standard_normal(conv.weight.value.shape)
    conv.bias.value[...] = rng.standard_normal(co)
    x = rng.standard_normal((b, ci, h, w))
    out = conv.forward(x)
    ref = O.conv_forward(x, conv.weight.value, conv.bias.value)
    assert np.allclose(out, ref, rtol=1e-12, atol=1e-12)
    dout = rng.standard_normal(out.shape)
    conv.weight.grad[...] = 1.0                      # backward accumulates into .grad
    dx = conv.backward(dout)
    rdx, rdw, rdb = O.conv_backward(x, conv.weight.value, dout)
    assert np.allclose(dx, rdx, rtol=1e-12, atol=1e-12)
    assert np.allclose(conv.weight.grad, rdw + 1.0, rtol=1e-12, atol=1e-12)
    assert np.allclose(conv.bias.grad, rdb, rtol=1e-12, atol=1e-12)
    with pytest.raises(ValueError):
        conv.forward(np.zeros((1, ci + 1, 3, 3)))


def test_residual_block_forward_backward_float64():
    from oracle import htoracle as O
    from paper_2304_12152_b200.nn import ResidualBlock
    rng = np.random.default_rng(5)
    blk = ResidualBlock(4)
    for q in blk.params():
        q.value[...] = 0.3 * rng.standard_normal(q.value.shape)
    x = rng.standard_normal((2, 4, 6, 7))
    y = blk.forward(x)
    t = O.conv_forward(x, blk.conv1.weight.value, blk.conv1.bias.value)
    r = np.maximum(t, 0.0)
    assert np.allclose(y, x + O.conv_forward(r, blk.conv2.weight.value, blk.conv2.bias.value),
                       rtol=1e-12, atol=1e-12)
    dout = rng.standard_normal(y.shape)
    dx = blk.backward(dout)
    dr, dw2, db2 = O.conv_backward(r, blk.conv2.weight.value, dout)
    dx1, dw1, db1 = O.conv_backward(x, blk.conv1.weight.value, dr * (t > 0))
    assert np.allclose(dx, dout + dx1, rtol=1e-12, atol=1e-12)
    for q, ref in zip(blk.params(), (dw1, db1, dw2, db2)):
        assert np.allclose(q.grad, ref, rtol=1e-12, atol=1e-12)


def test_policy_network_other_in_channels():
    """PolicyNetwork(in_channels=3) (nn.py:109-116): forward / backward layer
    by layer in float64 on the device, against the oracle (1e-12)."""
    from oracle import htoracle as O
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = PolicyNetwork(channels=6, blocks=2, in_channels=3)
    net.init_params(Rng(9), std=0.2)
    params = O.init_params(O.Rng(9), 6, 2, 3, 0.2)
    for q, r in zip(net.params(), params):      # same draws (Box-Muller to 1-2 ulp)
        assert np.allclose(q.value, r, rtol=1e-14, atol=1e-17)
    params = [q.value.copy() for q in net.params()]
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, 3, 9, 8))
    p = net.forward(x)
    p_ref, cache = O.policy_forward(params, x, keep=True)
    assert p.shape == (2, 1, 9, 8)
    assert np.allclose(p, p_ref, rtol=1e-12, atol=1e-14)
    dp = rng.standard_normal(p.shape)
    net.zero_grad()
    dx = net.backward(dp)
    dx_ref, grads = O.policy_backward(params, cache, dp)
    assert np.allclose(dx, dx_ref, rtol=1e-10, atol=1e-14)
    for q, gr in zip(net.params(), grads):
        assert np.allclose(q.grad, gr, rtol=1e-10, atol=1e-14)
    with pytest.raises(ValueError):
        net.forward(np.zeros((1, 2, 4, 4)))
    net.conv_out.bias.value[0] = np.inf
    with pytest.raises(FloatingPointError):
        net.forward(x)


@pytest.mark.parametrize("separable", [True, False])
def test_reward_maps_any_window_against_oracle(separable):
    """The reward-map kernel takes the separable path (2 x 11 products per
    window sum) only when the stencils are outer products (the reference's
    Gaussians, hvs.py:54-64) and the 2-D loop otherwise: both against the
    oracle's RewardContext / delta_map with the same stencils (float64)."""
    import torch
    from oracle import htoracle as O
    from paper_2304_12152_b200 import _lib
    rs = np.random.default_rng(3)
    H, W = 37, 45
    h = (rs.random((H, W)) < 0.5).astype(np.float64)
    c = rs.random((H, W))
    if separable:
        k, w = O.gaussian_kernel(11, 2.0), O.gaussian_kernel(11, 1.5)
    else:
        k = rs.random((9, 9)); k /= k.sum()
        w = rs.random((11, 11)); w /= w.sum()
    ref = O.RewardMaps(h, c, k, w)
    dev = torch.device("cuda")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(dev)   # noqa: E731
    hd, cd, kd, wd = t(h)[None], t(c)[None], t(k), t(w)
    maps = torch.empty((1, 8, H, W), dtype=torch.float64, device=dev)
    extra = torch.empty((1, 7, H, W), dtype=torch.float64, device=dev)
    sums = torch.empty((1, 2), dtype=torch.float64, device=dev)
    scratch = torch.empty((1, H, W), dtype=torch.float64, device=dev)
    _lib.call("ht_reward_context_f64", _lib.ptr(hd), _lib.ptr(cd), 1, H, W, _lib.ptr(kd), k.shape[0],
              _lib.ptr(wd), w.shape[0], 0.06, 1e-4, 9e-4, 2.0, _lib.ptr(maps), _lib.ptr(extra),
              _lib.ptr(sums), _lib.ptr(scratch), 0)
    m = maps[0].cpu().numpy()
    for got, want in ((m[0], ref.e), (m[1], ref.mu_h), (m[2], ref.shc), (m[3], ref.mu_c), (m[4], ref.scc),
                      (m[5], ref.sigma_c), (m[6], ref.ssim), (m[7], ref.shh)):
        assert np.allclose(got, want, rtol=1e-12, atol=1e-14)
    other = 1.0 - h
    od = t(other)[None]
    out = torch.empty((1, H, W), dtype=torch.float64, device=dev)
    nbytes = _lib.out_i64("ht_reward_workspace_bytes", 1, H, W) + 8 * H * W
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    _lib.call("ht_reward_delta_f64", _lib.ptr(hd), _lib.ptr(od), _lib.ptr(cd), 1, H, W, _lib.ptr(kd), k.shape[0],
              _lib.ptr(wd), w.shape[0], 0.06, 1e-4, 9e-4, 2.0, _lib.ptr(out), _lib.ptr(ws), nbytes, 0)
    d_ref = ref.delta_map(other)
    assert np.allclose(out[0].cpu().numpy(), d_ref, rtol=1e-9, atol=1e-15 * np.abs(d_ref).max())
