import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
from paper_2304_12152_b200.nn import PolicyNetwork
from paper_2304_12152_b200.imagecore import Rng
net = PolicyNetwork(32, 3); net.init_params(Rng(7), std=0.05)
r = Rng(11); B, H, W = 3, 40, 52
x = np.stack([np.stack((r.uniforms(H * W).reshape(H, W), r.gaussians(H * W).reshape(H, W))) for _ in range(B)])
xd = torch.from_numpy(x.astype(np.float32)).cuda()
acts = {}
for impl in (1, 0):
    _lib.call("ht_set_train_conv_impl", impl)
    p = net.forward_device(xd); torch.cuda.synchronize()
    acts[impl] = (net._cache[1].clone(), p.clone())
a = B * 32 * H * W
for k in range(2 * 3 + 1):
    s1 = acts[1][0][a * 4 * k: a * 4 * (k + 1)].view(torch.float32).double()
    s0 = acts[0][0][a * 4 * k: a * 4 * (k + 1)].view(torch.float32).double()
    d = (s0 - s1).abs()
    print(k, "max|diff|", d.max().item(), "max|v|", s1.abs().max().item(), "argmax", np.unravel_index(d.argmax().item(), (B, 32, H, W)))
print("p", (acts[0][1] - acts[1][1]).abs().max().item())
