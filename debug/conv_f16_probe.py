"""Scaled-fp16-pair training conv (impl 2) vs split-bf16 (impl 0) and SIMT (1):
single-conv error at three input scales, full-depth gradient error vs the
fp64 oracle, and per-launch time at 20 x 256^2."""
import ctypes as C, sys, time, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_gpu_conv_tc import _conv64, _run
from paper_2304_12152_b200 import _lib
from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import PolicyNetwork
from oracle import htoracle as O

r = Rng(3)
B, H, W = 2, 24, 30
for xs, ws in ((1.0, 0.05), (1e-6, 0.05), (1e-9, 0.05), (1.0, 1e-4)):
    x = (r.gaussians(B * 32 * H * W).reshape(B, 32, H, W) * xs).astype(np.float32).astype(np.float64)
    w = (r.gaussians(32 * 32 * 9).reshape(32, 32, 3, 3) * ws).astype(np.float32).astype(np.float64)
    ref = _conv64(x, w)
    scale = np.abs(_conv64(np.abs(x), np.abs(w))).max()
    msg = []
    for impl in (0, 1, 2):
        out = _run(impl, x, w)
        e = np.abs(out - ref)
        msg.append(f"impl{impl} max/scale {e.max() / scale:.2e} rel {np.linalg.norm(out - ref) / np.linalg.norm(ref):.2e}")
    print(f"x~{xs:g} w~{ws:g}: " + " | ".join(msg))

def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
for NB, (B, H, W), std in ((16, (2, 40, 52), 0.05), (16, (1, 64, 64), 0.01), (3, (3, 40, 52), 0.05)):
    net = PolicyNetwork(32, NB); net.init_params(Rng(7), std=std)
    rr = Rng(11)
    x = np.stack([np.stack((rr.uniforms(H * W).reshape(H, W), rr.gaussians(H * W).reshape(H, W)))
                  for _ in range(B)]).astype(np.float32).astype(np.float64)
    dp = (rr.gaussians(B * H * W).reshape(B, H, W) * 1e-3).astype(np.float32).astype(np.float64)
    params = [q.value for q in net.params()]
    p_ref, cache = O.policy_forward(params, x, keep=True)
    dx_ref, grads = O.policy_backward(params, cache, dp[:, None])
    g_ref = np.concatenate([g.ravel() for g in grads])
    for impl in (0, 1, 2):
        _lib.call("ht_set_train_conv_impl", impl)
        xd = torch.from_numpy(x.astype(np.float32)).cuda()
        p = net.forward_device(xd)
        g = torch.zeros(net.num_params(), dtype=torch.float64, device="cuda")
        dx = torch.zeros_like(xd)
        net.backward_device(torch.from_numpy(dp.astype(np.float32)).cuda(), g, dx)
        p, g, dx = p.double().cpu().numpy(), g.cpu().numpy(), dx.double().cpu().numpy()
        at, worst = 0, 0.0
        for t in grads:
            n = t.size
            if np.linalg.norm(t) > 0: worst = max(worst, rel(g[at:at + n], t.ravel()))
            at += n
        print(f"NB={NB} {B}x{H}x{W} std {std} impl {impl}: p {np.max(np.abs(p - p_ref[:, 0])):.2e} "
              f"grad worst-tensor {worst:.2e} all {rel(g, g_ref):.2e} dx {rel(dx, dx_ref):.2e}")
    _lib.call("ht_set_train_conv_impl", 0)

for impl in (0, 2):
    B = 20; H = W = 256
    x = torch.randn(B, 32, H, W, device='cuda'); w = torch.randn(32, 32, 3, 3, device='cuda') * 0.05
    bias = torch.randn(32, device='cuda'); o = torch.empty_like(x)
    f = lambda: _lib.call("ht_conv3x3_32", C.c_void_p(x.data_ptr()), B, H, W, C.c_void_p(w.data_ptr()),
                          C.c_void_p(bias.data_ptr()), None, None, C.c_void_p(o.data_ptr()), 1, impl, None)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(30): f()
    b.record(); torch.cuda.synchronize()
    print(f"impl {impl}: {a.elapsed_time(b) / 30 * 1e3:.1f} us per launch at 20 x 256^2")
