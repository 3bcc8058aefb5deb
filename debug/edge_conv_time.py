"""Per-step GPU time of the edge-conv kernels (forward and weight-gradient) (impl 0 warp-row vs 1
generic tile) inside a config-5-sized backward: 20 x 256^2."""
import sys, collections, numpy as np, torch
sys.path.insert(0, '.')
from paper_2304_12152_b200 import _lib
from paper_2304_12152_b200.nn import PolicyNetwork
from paper_2304_12152_b200.imagecore import Rng
from torch.profiler import profile, ProfilerActivity
net = PolicyNetwork(32, 16); net.init_params(Rng(0))
x = torch.rand(20, 2, 256, 256, device='cuda'); dp = torch.randn(20, 256, 256, device='cuda') * 1e-4
for impl in (0, 1):
    _lib.call("ht_set_edge_conv_impl", impl)
    for _ in range(2):
        net.forward_device(x); g = torch.zeros(net.num_params(), dtype=torch.float64, device='cuda'); net.backward_device(dp, g)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        net.forward_device(x); g = torch.zeros(net.num_params(), dtype=torch.float64, device='cuda'); net.backward_device(dp, g)
        torch.cuda.synchronize()
    tot = collections.defaultdict(float)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and ('wgrad' in e.name or 'edge' in e.name or 'fwd_kernel' in e.name):
            tot[e.name[:60]] += e.time_range.end - e.time_range.start
    print("impl", impl, {k: round(v, 1) for k, v in tot.items() if 'wgt::' not in k})
