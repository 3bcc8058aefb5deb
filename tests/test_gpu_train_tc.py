"""Training convolutions on tcgen05 (split-bf16, csrc/conv_tc.cu) against the fp32
SIMT kernels and the oracle: forward p and every parameter / input gradient of
the paper architecture (the golden-vector training tests in test_gpu_train.py
run on the tensor-core path too, since it is the default)."""

import numpy as np
import pytest

from paper_2304_12152_b200.imagecore import Rng

pytestmark = pytest.mark.gpu


def _run(impl, net, x, dp, wgrad_parts=2):
    import torch
    from paper_2304_12152_b200 import _lib
    _lib.call("ht_set_train_conv_impl", impl)
    _lib.call("ht_set_wgrad_parts", wgrad_parts)
    try:
        xd = torch.from_numpy(x.astype(np.float32)).cuda()
        p = net.forward_device(xd)
        grad = torch.zeros(net.num_params(), dtype=torch.float64, device="cuda")
        dx = torch.zeros_like(xd)
        net.backward_device(torch.from_numpy(dp.astype(np.float32)).cuda(), grad, dx)
        return p.double().cpu().numpy(), grad.cpu().numpy(), dx.double().cpu().numpy()
    finally:
        _lib.call("ht_set_train_conv_impl", 0)
        _lib.call("ht_set_wgrad_parts", 2)


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("parts", [2, 3])
@pytest.mark.parametrize("B,H,W", [(3, 40, 52), (1, 96, 150), (1, 7, 300)])
def test_tensor_core_training_convs_vs_oracle(B, H, W, parts):
    """Both the tcgen05 path (impl 0) and the SIMT path (impl 1) against the
    fp64 oracle: p, parameter gradients per tensor and dx within 1e-4
    relative.  With the weight gradient's operands split into three bf16
    parts (six products) the tensor-core path is no less accurate than SIMT
    (split-bf16 convs with short accumulation chains: ~1e-7 per conv); the
    default two parts (three products) stay well inside the 1e-4 bar."""
    from oracle import htoracle as O
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = PolicyNetwork(32, 3)
    net.init_params(Rng(7), std=0.05)
    r = Rng(11)
    x = np.stack([np.stack((r.uniforms(H * W).reshape(H, W), r.gaussians(H * W).reshape(H, W)))
                  for _ in range(B)]).astype(np.float32).astype(np.float64)
    dp = (r.gaussians(B * H * W).reshape(B, H, W) * 1e-3).astype(np.float32).astype(np.float64)
    params = [q.value for q in net.params()]
    p_ref, cache = O.policy_forward(params, x, keep=True)
    dx_ref, grads = O.policy_backward(params, cache, dp[:, None])
    g_ref = np.concatenate([g.ravel() for g in grads])
    errs = {}
    for impl in (0, 1):
        p, g, dx = _run(impl, net, x, dp, parts)
        assert np.max(np.abs(p - p_ref[:, 0])) < 2e-5
        at = 0
        worst = 0.0
        for t in grads:
            n = t.size
            if np.linalg.norm(t) > 0:
                worst = max(worst, _rel(g[at:at + n], t.ravel()))
            at += n
        errs[impl] = (worst, _rel(g, g_ref), _rel(dx, dx_ref))
        assert worst < 1e-4 and errs[impl][2] < 1e-4, (impl, errs[impl])
    if parts == 3:
        assert errs[0][1] <= 1.5 * errs[1][1] + 1e-7, errs
    else:
        assert errs[0][0] < 2e-5, errs


def test_tensor_core_matches_simt_at_config5_size():
    """2 x 256^2 (config-5 crops): the two paths agree on p and, normwise, on
    the gradients to within the cancellation-limited fp32 noise."""
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = PolicyNetwork(32, 3)
    net.init_params(Rng(7), std=0.05)
    r = Rng(12)
    B, H, W = 2, 256, 256
    x = np.stack([np.stack((r.uniforms(H * W).reshape(H, W), r.gaussians(H * W).reshape(H, W)))
                  for _ in range(B)])
    dp = r.gaussians(B * H * W).reshape(B, H, W) * 1e-3
    p0, g0, dx0 = _run(0, net, x, dp)
    p1, g1, dx1 = _run(1, net, x, dp)
    assert np.max(np.abs(p0 - p1)) < 2e-6
    assert _rel(g0, g1) < 1e-3 and _rel(dx0, dx1) < 1e-3


def test_tensor_core_forward_matches_oracle():
    from oracle import htoracle as O
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = PolicyNetwork(32, 2)
    net.init_params(Rng(3), std=0.05)
    r = Rng(5)
    x = np.stack((r.uniforms(33 * 47).reshape(33, 47), r.gaussians(33 * 47).reshape(33, 47)))[None]
    p, _, _ = _run(0, net, x, np.zeros((1, 33, 47)))
    ref = O.policy_forward([q.value for q in net.params()], x.astype(np.float32).astype(np.float64))
    assert np.max(np.abs(p - ref[:, 0])) < 2e-5


@pytest.mark.parametrize("C,NB", [(32, 2), (8, 2)])
@pytest.mark.parametrize("B,H,W", [(2, 37, 61), (3, 40, 256), (1, 70, 264), (2, 33, 300)])
def test_edge_convs_warp_row_kernels(C, NB, B, H, W):
    """The warp-row edge kernels (default: conv_in's forward and weight
    gradient, conv_out's weight and input gradients) against the generic SIMT
    tile kernels (ht_set_edge_conv_impl(1)): p and every gradient tensor
    agree to fp32 summation-order level, on aligned and ragged widths."""
    import torch
    from paper_2304_12152_b200 import _lib
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = PolicyNetwork(C, NB)
    net.init_params(Rng(5), std=0.05)
    r = Rng(6)
    x = np.stack((r.uniforms(B * H * W).reshape(B, H, W), r.gaussians(B * H * W).reshape(B, H, W)), axis=1)
    dp = r.gaussians(B * H * W).reshape(B, H, W) * 1e-3
    grads, ps = [], []
    for impl in (0, 1):
        _lib.call("ht_set_edge_conv_impl", impl)
        try:
            xd = torch.from_numpy(x.astype(np.float32)).cuda()
            ps.append(net.forward_device(xd).double().cpu().numpy())
            g = torch.zeros(net.num_params(), dtype=torch.float64, device="cuda")
            net.backward_device(torch.from_numpy(dp.astype(np.float32)).cuda(), g)
            grads.append(g.cpu().numpy())
        finally:
            _lib.call("ht_set_edge_conv_impl", 0)
    assert np.max(np.abs(ps[0] - ps[1])) <= 1e-6
    sizes = [p.value.size for p in net.params()]
    offs = np.cumsum([0] + sizes)
    for k in range(len(sizes)):
        a, b = grads[0][offs[k]:offs[k + 1]], grads[1][offs[k]:offs[k + 1]]
        assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b) + 1e-30, k


@pytest.mark.parametrize("B,H,W", [(2, 33, 256), (1, 7, 300), (3, 20, 132)])
def test_relu_bits_and_in_place_skip_gradient(B, H, W):
    """Training ReLU bits (default on the TMA-staged path: each conv1's mask
    stored as 4 B per pixel, conv2's input gradient reads the bits, conv1's
    input gradient is added onto the skip gradient in place) against the fp32
    mask / residual epilogue inputs (ht_set_train_bits(0)): p bitwise, dx and
    every gradient tensor to fp32 summation-order level.  A backward follows
    its forward's setting even when the setting changes in between."""
    import torch
    from paper_2304_12152_b200 import _lib
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = PolicyNetwork(32, 3)
    net.init_params(Rng(8), std=0.05)
    r = Rng(9)
    x = np.stack((r.uniforms(B * H * W).reshape(B, H, W), r.gaussians(B * H * W).reshape(B, H, W)), axis=1)
    dp = r.gaussians(B * H * W).reshape(B, H, W) * 1e-3
    out = []
    for fwd_bits, bwd_bits in ((1, 1), (0, 0), (1, 0), (0, 1)):
        try:
            _lib.call("ht_set_train_bits", fwd_bits)
            xd = torch.from_numpy(x.astype(np.float32)).cuda()
            p = net.forward_device(xd).double().cpu().numpy()
            _lib.call("ht_set_train_bits", bwd_bits)
            g = torch.zeros(net.num_params(), dtype=torch.float64, device="cuda")
            dx = torch.zeros_like(xd)
            net.backward_device(torch.from_numpy(dp.astype(np.float32)).cuda(), g, dx)
            out.append((p, g.cpu().numpy(), dx.double().cpu().numpy()))
        finally:
            _lib.call("ht_set_train_bits", 1)
    sizes = [q.value.size for q in net.params()]
    offs = np.cumsum([0] + sizes)
    p0, g0, dx0 = out[1]   # fp32 epilogue inputs throughout
    for p, g, dx in out:
        assert np.array_equal(p, p0)
        assert np.linalg.norm(dx - dx0) <= 1e-6 * np.linalg.norm(dx0)
        for k in range(len(sizes)):
            a, b = g[offs[k]:offs[k + 1]], g0[offs[k]:offs[k + 1]]
            assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b) + 1e-30, k
