"""Generate the golden fixtures in tests/golden/ by running the REAL reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the htlab reference package read-only from
/root/reference/pkg/src, feeds it seeded inputs (rounded to float32 once, so
the GPU path and the reference see identical values) and stores the inputs
and the reference outputs as compressed .npz files next to this script.
Nothing on the GPU box reads /root/reference; the fixtures travel instead.
"""

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from htlab import hvs, imagecore, metrics, nn, rl, spectral  # noqa: E402
from htlab.imagecore import Rng  # noqa: E402

from paper_2304_12152_b200 import synth  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def flat_params(net):
    return np.concatenate([p.value.ravel() for p in net.params()])


def flat_grads(net):
    return np.concatenate([p.grad.ravel() for p in net.params()])


def probes(n, k=4, seed=1234):
    return np.random.default_rng(seed).standard_normal((k, n))


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name} ({os.path.getsize(path) / 1e3:.1f} kB)")


def gen_rng():
    s, sm = 0, []
    for _ in range(3):
        s, z = imagecore.splitmix64(s)
        sm.append(z)
    r = Rng(0)
    r.set_state_words((1, 2, 3, 4))
    xo = [r.next_uint64() for _ in range(6)]
    r = Rng(7)
    uni = r.uniforms(9)
    g = Rng(11).gaussians(7)
    noise = imagecore.gaussian_noise_map(Rng(5), 8, 6)
    r = Rng(3)
    ints = [r.randint(n) for n in (1, 2, 7, 100, 1 << 20)]
    words = Rng(42).state_words()
    # a long stream: checksum of 100k uniforms (pins the C implementation)
    r = Rng(99)
    long_u = r.uniforms(100_000)
    save("rng.npz",
         splitmix=np.array(sm, dtype=np.uint64),
         xoshiro1234=np.array(xo, dtype=np.uint64),
         uniforms_seed7=uni, gaussians_seed11=g, noise_seed5_w8_h6=noise,
         randint_seed3=np.array(ints), state_seed42=np.array(words, dtype=np.uint64),
         long_uniforms_seed99_sum=np.array([long_u.sum(), long_u[-1], long_u[12345]]),
         long_state_seed99=np.array(r.state_words(), dtype=np.uint64))


def forward_case(channels, blocks, std, c, z, seed=0):
    net = nn.PolicyNetwork(channels=channels, blocks=blocks)
    net.init_params(Rng(seed), std=std)
    x = np.stack((c, z))[None]
    p = net.forward(x)[0, 0]
    return net, p


def gen_forward():
    t0 = time.time()
    out = {}
    # small full-arch and mini-arch cases
    c = f32(synth.contone(40, 48, seed=11))
    z = f32(imagecore.gaussian_noise_map(Rng(1), 48, 40))
    out["small_c"], out["small_z"] = c.astype(np.float32), z.astype(np.float32)
    for std in (0.01, 0.05):
        _, p = forward_case(32, 16, std, c, z)
        out[f"small_p_std{std}"] = p
    _, p = forward_case(8, 2, 0.05, c, z)
    out["small_p_mini"] = p
    # ragged / tiny shapes
    for (hh, ww) in ((1, 1), (3, 5), (7, 2), (37, 131)):
        cc = f32(synth.contone(hh, ww, seed=hh * 100 + ww))
        zz = f32(imagecore.gaussian_noise_map(Rng(hh + ww), ww, hh))
        _, p = forward_case(32, 16, 0.05, cc, zz)
        out[f"rag_{hh}x{ww}_c"] = cc.astype(np.float32)
        out[f"rag_{hh}x{ww}_z"] = zz.astype(np.float32)
        out[f"rag_{hh}x{ww}_p"] = p
    # BASELINE config 1: one 256x256 contone (seed 0), full arch
    c1 = f32(synth.contone(256, 256, seed=0, blobs=8, rects=2))
    z1 = f32(imagecore.gaussian_noise_map(Rng(0), 256, 256))
    out["cfg1_c"], out["cfg1_z"] = c1.astype(np.float32), z1.astype(np.float32)
    for std in (0.01, 0.05):
        _, p = forward_case(32, 16, std, c1, z1)
        out[f"cfg1_p_std{std}"] = p.astype(np.float32)
        out[f"cfg1_band_std{std}"] = np.array([np.mean(np.abs(p - 0.5) < 1e-3)])
    save("forward.npz", **out)
    print(f"  forward fixtures in {time.time() - t0:.1f}s")


def gen_backward():
    out = {}
    for tag, (ch, nb, hh, ww) in {"mini": (8, 2, 9, 11),
                                  "full": (32, 16, 20, 24)}.items():
        net = nn.PolicyNetwork(channels=ch, blocks=nb)
        net.init_params(Rng(2), std=0.05)
        r = Rng(4)
        x = f32(r.uniforms(2 * 2 * hh * ww).reshape(2, 2, hh, ww))
        p = net.forward(x)
        dp = f32(r.gaussians(p.size).reshape(p.shape))
        net.zero_grad()
        dx = net.backward(dp)
        g = flat_grads(net)
        out[f"{tag}_x"], out[f"{tag}_dp"] = x, dp
        out[f"{tag}_p"], out[f"{tag}_dx"] = p, dx
        out[f"{tag}_grad_probe"] = probes(g.size) @ g
        out[f"{tag}_grad_norms"] = np.array(
            [np.linalg.norm(q.grad) for q in net.params()])
        if tag == "mini":
            out["mini_grad"] = g
        else:
            out["full_grad_head"] = np.concatenate(
                [q.grad.ravel() for q in net.params()[:4]])
            out["full_grad_tail"] = np.concatenate(
                [q.grad.ravel() for q in net.params()[-4:]])
    save("backward.npz", **out)


def gen_reward():
    out = {}
    hh, ww = 24, 28
    r = Rng(8)
    c = f32(synth.contone(hh, ww, seed=5))
    m = (r.uniforms(hh * ww).reshape(hh, ww) < 0.5).astype(np.float64)
    out["c"], out["m"] = c, m
    for model in ("nasanen", "gaussian"):
        cfg = metrics.MetricConfig(hvs=hvs.HvsConfig(model=model))
        ctx = metrics.reward(m, c, cfg, region="full")
        sample = rl.EpisodeSample(c=c, z=None, p=None, m=m, floor_vals=np.zeros_like(m),
                                  ceil_vals=np.ones_like(m), p_ceil=None,
                                  level_count=2, ctx=ctx)
        out[f"{model}_kernel"] = ctx.kernel.weights
        out[f"{model}_reward"] = np.array([ctx.reward, ctx.mse, ctx.cssim_scalar])
        out[f"{model}_reward_map"] = ctx.reward_map
        out[f"{model}_delta_flip"] = metrics.delta_map(ctx, 1.0 - m)
        out[f"{model}_le"] = rl.le_signal(sample)
    out["ssim_window"] = metrics._window_weights(11, 1.5)
    # 64x64 case with the sampling step (rl.make_sample draw order)
    c2 = f32(synth.contone(64, 64, seed=6))
    p2 = f32(Rng(9).uniforms(64 * 64).reshape(64, 64))
    s = rl.make_sample(p2, c2, None, Rng(10), metrics.MetricConfig(
        hvs=hvs.HvsConfig(model="gaussian")))
    out["s64_c"], out["s64_p"], out["s64_m"] = c2, p2, s.m
    out["s64_reward"] = np.array([s.ctx.reward])
    out["s64_le"] = rl.le_signal(s)
    save("reward.npz", **out)


def gen_spectral():
    out = {}
    for n in (4, 32, 256):
        part = spectral.ring_partition((n, n))
        out[f"ring{n}_counts"] = part.counts
        out[f"ring{n}_radii"] = part.radii
        out[f"ring{n}_sha"] = np.frombuffer(
            hashlib.sha256(part.ring_index.astype("<i8").tobytes()).digest(),
            dtype=np.uint8)
    part = spectral.ring_partition((2, 4))
    out["ring2x4_counts"] = part.counts
    r = Rng(12)
    x = f32(0.5 + 0.01 * r.gaussians(32 * 32).reshape(32, 32))
    out["x32"] = x
    out["x32_loss"] = np.array([spectral.anisotropy_loss(x)])
    out["x32_grad"] = spectral.anisotropy_loss_backward(x)
    x2 = f32(r.uniforms(256 * 256).reshape(256, 256))
    out["x256"] = x2.astype(np.float32)
    out["x256_loss"] = np.array([spectral.anisotropy_loss(x2)])
    g2 = spectral.anisotropy_loss_backward(x2)
    out["x256_grad_probe"] = probes(g2.size) @ g2.ravel()
    out["x256_grad_norm"] = np.array([np.linalg.norm(g2)])
    out["x256_grad_crop"] = g2[:16, :16]
    h = (r.uniforms(32 * 32).reshape(32, 32) < 0.3).astype(np.float64)
    cur = spectral.rapsd(spectral.periodogram(h))
    out["h32"], out["h32_power"], out["h32_anis"] = h, cur.power, cur.anisotropy
    out["h32_dc"] = np.array([cur.dc_power])
    save("spectral.npz", **out)


def gen_train():
    out = {}
    # (a) mini config, whole step; (b) full arch, small crop
    for tag, (ch, nb, bs, crop, ba) in {"mini": (8, 2, 2, 24, 2),
                                        "full": (32, 16, 2, 32, 1)}.items():
        cfg = rl.TrainConfig(iterations=10, batch_size=bs, crop_size=crop,
                             channels=ch, blocks=nb, anisotropy_batch_size=ba,
                             hvs_model="gaussian")
        ds = [f32(synth.contone(48, 40, seed=20 + i)) for i in range(3)]
        rng = Rng(cfg.seed)
        net = nn.PolicyNetwork(channels=ch, blocks=nb)
        adam = nn.Adam(net.params())
        net.init_params(rng)
        p0 = flat_params(net)
        state0 = rng.state_words()
        diag = rl.train_step(net, adam, ds, cfg, rng, 0)
        g = flat_grads(net)
        p1 = flat_params(net)
        out[f"{tag}_ds"] = np.stack(ds)
        out[f"{tag}_state0"] = np.array(state0, dtype=np.uint64)
        out[f"{tag}_state1"] = np.array(rng.state_words(), dtype=np.uint64)
        out[f"{tag}_diag"] = np.array([diag["reward"], diag["l_as"],
                                       diag["bin_gap"], diag["lr"]])
        out[f"{tag}_p0_probe"] = probes(p0.size) @ p0
        out[f"{tag}_grad_probe"] = probes(g.size) @ g
        out[f"{tag}_grad_norms"] = np.array(
            [np.linalg.norm(q.grad) for q in net.params()])
        out[f"{tag}_dparam_probe"] = probes(p1.size) @ (p1 - p0)
        out[f"{tag}_dparam_norms"] = np.array(
            [np.linalg.norm(a) for a in np.split(p1 - p0, np.cumsum(
                [q.value.size for q in net.params()])[:-1])])
        if tag == "mini":
            out["mini_grad"], out["mini_p1"] = g, p1
    save("train.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["rng", "forward", "backward", "reward",
                             "spectral", "train"]
    for w in which:
        t0 = time.time()
        globals()[f"gen_{w}"]()
        print(f"{w}: {time.time() - t0:.1f}s")
