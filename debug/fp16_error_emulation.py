import numpy as np, sys
sys.path.insert(0, '.')
from oracle import htoracle as O
from paper_2304_12152_b200 import synth
def f16(a): return a.astype(np.float16).astype(np.float64)
def f32(a): return a.astype(np.float32).astype(np.float64)
params = O.init_params(O.Rng(0), 32, 16, 2, 0.05)
H = W = 160
c = synth.contone(H, W, seed=3).astype(np.float64); z = np.random.default_rng(1).standard_normal((H, W)).astype(np.float32).astype(np.float64)
x = np.stack((c, z))[None]
def fwd(mode_out):
    # conv_in fp32-ish (hi/lo), mid convs fp16 operands with fp32 residual stream
    y = f32(O.conv_forward(x, params[0], params[1]))
    for i in range(16):
        w1,b1,w2,b2 = params[2+4*i:6+4*i]
        t = O.conv_forward(f16(y), f16(w1), b1)
        r = np.maximum(t, 0)
        y = f32(y + O.conv_forward(f16(r), f16(w2), b2))
    if mode_out == 'f16':
        lg = O.conv_forward(f16(y), f16(params[-2]), params[-1])
    else:
        lg = O.conv_forward(y, params[-2], params[-1])
    return 1/(1+np.exp(-lg))
p_ref = O.policy_forward(params, x)
for m in ('f16', 'f32'):
    p = fwd(m); e = np.abs(p - p_ref); print(m, 'max', e.max(), 'mean', e.mean())
