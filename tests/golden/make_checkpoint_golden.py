"""Write tests/golden/ckpt_ref.htnn and ckpt_ref_bare.htnn with the REAL
reference's save_checkpoint (nn.py:209-217), plus the expected decoded
contents in ckpt_ref.npz.  Run in the build container only:

    python tests/golden/make_checkpoint_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from htlab import nn  # noqa: E402
from htlab.imagecore import Rng  # noqa: E402


def main():
    net = nn.PolicyNetwork(channels=4, blocks=2, in_channels=2)
    net.init_params(Rng(31), std=0.3)
    adam = nn.Adam(net.params())
    rng = Rng(37)
    for _ in range(3):
        for p in net.params():
            p.grad[...] = rng.gaussians(p.value.size).reshape(p.value.shape)
        adam.step(1e-3)
    words = (11, 22, 33, 2 ** 64 - 1)
    nn.save_checkpoint(os.path.join(HERE, "ckpt_ref.htnn"), net, adam, iteration=5, rng_state=words)
    nn.save_checkpoint(os.path.join(HERE, "ckpt_ref_bare.htnn"), net)
    flat = lambda bufs: np.concatenate([b.ravel() for b in bufs])
    np.savez_compressed(os.path.join(HERE, "ckpt_ref.npz"),
                        values=flat([p.value for p in net.params()]), m=flat(adam.m), v=flat(adam.v),
                        adam_t=adam.t, iteration=5, rng_state=np.array(words, dtype=np.uint64))
    print("wrote ckpt_ref.htnn, ckpt_ref_bare.htnn, ckpt_ref.npz")


if __name__ == "__main__":
    main()
