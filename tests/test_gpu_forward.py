"""GPU parity of the inference hot path (K1) against the reference oracle.

Tolerance (BASELINE.json north_star): probabilities within 1e-3 absolute of
the reference; halftones bit-exact except where the reference probability
lies within 1e-3 of the 0.5 threshold.  The fp32 SIMT path (impl=1) is held
to 2e-5.  Tiling / batching / row-window sharding of the fused kernel must
be BITWISE invariant (every pixel sees the same operation sequence).
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

P_TOL = 1e-3       # north_star: probabilities within 1e-3 absolute
BAND = 1e-3        # threshold exemption band


def _net(std, ch=32, nb=16, seed=0):
    from paper_2304_12152_b200.imagecore import Rng
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = PolicyNetwork(ch, nb)
    net.init_params(Rng(seed), std=std)
    return net


def _check(p, h, p_ref, tol):
    p_ref = np.asarray(p_ref, np.float64)
    err = np.abs(p - p_ref)
    assert err.max() <= tol, f"max|dp| = {err.max():.3e}"
    h_ref = (p_ref >= 0.5)
    outside = np.abs(p_ref - 0.5) >= BAND
    assert np.array_equal(h[outside].astype(bool), h_ref[outside])
    return float(err.max()), float(1.0 - outside.mean())


@pytest.mark.parametrize("impl", [0, 1])
@pytest.mark.parametrize("std", [0.01, 0.05])
def test_config1_256(impl, std):
    from paper_2304_12152_b200 import rl
    g = golden("forward.npz")
    net = _net(std)
    h, p = rl.halftone(net, g["cfg1_c"], g["cfg1_z"], impl=impl)
    err, band = _check(p, h, g[f"cfg1_p_std{std}"], P_TOL if impl == 0 else 2e-5)
    print(f"impl={impl} std={std}: max|dp|={err:.3e} band={band:.4f}")


@pytest.mark.parametrize("impl", [0, 1])
@pytest.mark.parametrize("shape", ["1x1", "3x5", "7x2", "37x131"])
def test_ragged_shapes(impl, shape):
    from paper_2304_12152_b200 import rl
    g = golden("forward.npz")
    net = _net(0.05)
    h, p = rl.halftone(net, g[f"rag_{shape}_c"], g[f"rag_{shape}_z"], impl=impl)
    _check(p, h, g[f"rag_{shape}_p"], P_TOL if impl == 0 else 2e-5)


@pytest.mark.parametrize("impl", [0, 1])
@pytest.mark.parametrize("std", [0.01, 0.05])
def test_small_full_arch(impl, std):
    from paper_2304_12152_b200 import rl
    g = golden("forward.npz")
    h, p = rl.halftone(_net(std), g["small_c"], g["small_z"], impl=impl)
    _check(p, h, g[f"small_p_std{std}"], P_TOL if impl == 0 else 2e-5)


def test_mini_arch_simt():
    from paper_2304_12152_b200 import rl
    g = golden("forward.npz")
    h, p = rl.halftone(_net(0.05, 8, 2), g["small_c"], g["small_z"])  # C=8 -> SIMT
    _check(p, h, g["small_p_mini"], 2e-5)


def test_batch_equals_single_bitwise():
    import torch
    from paper_2304_12152_b200 import rl, synth
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_f32
    net = _net(0.05)
    cs = synth.config_batch(3, 70, 90, seed=3, step_frac=0.34)
    zs = np.stack([gaussian_noise_map_f32(Rng(10 + i), 90, 70) for i in range(3)])
    hb, pb = rl.halftone(net, cs, zs)
    for i in range(3):
        hi, pi = rl.halftone(net, cs[i], zs[i])
        assert np.array_equal(pi, pb[i]) and np.array_equal(hi, hb[i])


def test_host_batch_pipeline_equals_oneshot():
    """rl.halftone on a host batch of >= 4 images runs chunked through two
    streams (rl._halftone_host_batch); it equals the one-shot path bitwise
    for float64 / float32 numpy, reversed-stride views and CPU tensors, with
    a ragged last chunk, and a chunk that overflows fp16 is redone in float64
    like the one-shot path."""
    import torch
    from paper_2304_12152_b200 import rl, synth
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_f32
    net = _net(0.05)
    B = 11                                        # chunks of 2, the last of 1
    cs = synth.config_batch(B, 40, 52, seed=5, step_frac=0.3).astype(np.float64)
    zs = np.stack([gaussian_noise_map_f32(Rng(30 + i), 52, 40) for i in range(B)])
    h1, p1 = rl._halftone_oneshot(net, cs, zs, None)
    for c, z, rev in ((cs, zs, False), (cs.astype(np.float32), zs, False), (cs[::-1], zs[::-1], True),
                      (torch.from_numpy(cs), torch.from_numpy(zs), False)):
        h, p = rl.halftone(net, c, z)
        assert h.dtype == np.float64 and p.dtype == np.float64 and h.shape == (B, 40, 52)
        if rev:
            h, p = h[::-1], p[::-1]
        assert np.array_equal(p, p1) and np.array_equal(h, h1)
    big = _net(0.1)                               # activations leave fp16's range
    cs4, zs4 = cs[:5, :24, :20], zs[:5, :24, :20]
    hb, pb = rl.halftone(big, cs4, zs4)
    ho, po = rl._halftone_oneshot(big, cs4, zs4, None)
    assert np.array_equal(pb, po) and np.array_equal(hb, ho)


def test_row_window_sharding_bitwise():
    """Config-4 style row strips with the 34-row receptive-field halo."""
    import torch
    from paper_2304_12152_b200 import synth
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_f32
    net = _net(0.05)
    H, W = 200, 150
    c = torch.from_numpy(synth.contone(H, W, seed=9)).cuda()
    z = torch.from_numpy(gaussian_noise_map_f32(Rng(4), W, H)).cuda()
    full = torch.empty((1, H, W), device="cuda")
    net.halftone_device(c[None], z[None], p_out=full)
    halo = 34
    parts = []
    for r0, r1 in ((0, 70), (70, 151), (151, 200)):
        i0, i1 = max(0, r0 - halo), min(H, r1 + halo)
        out = torch.empty((1, r1 - r0, W), device="cuda")
        net.halftone_device(c[None, i0:i1].contiguous(), z[None, i0:i1].contiguous(), p_out=out,
                            rows=(H, i0, r0, r1 - r0))
        parts.append(out)
    stitched = torch.cat(parts, dim=1)
    assert torch.equal(stitched, full)


@pytest.mark.parametrize("impl", [0, 1])
@pytest.mark.parametrize("B,H,W", [(1, 33, 77), (3, 20, 130), (5, 17, 256), (2, 9, 1)])
def test_pbm_payload_matches_packbits(impl, B, H, W):
    """The PBM P4 payload (imagecore.py:289-297) written by the fused kernel's
    epilogue (impl 0: bits OR-reduced per word straight from the logits; a
    word can span two strips' CTAs) or packed from h (impl 1) equals
    np.packbits(1 - h) -- for payloads that are whole words (written in
    place) and ragged ones (padded scratch + copy), with and without h."""
    import torch
    from paper_2304_12152_b200 import synth
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_f32
    net = _net(0.05)
    c = torch.from_numpy(np.stack([synth.contone(H, W, seed=2 + i) for i in range(B)])).cuda()
    z = torch.from_numpy(np.stack([gaussian_noise_map_f32(Rng(2 + i), W, H) for i in range(B)])).cuda()
    h = torch.empty((B, H, W), dtype=torch.uint8, device="cuda")
    pbm = torch.full((B, H, (W + 7) // 8), 0xAB, dtype=torch.uint8, device="cuda")
    net.halftone_device(c, z, h_out=h, pbm_out=pbm, impl=impl, check=True)
    want = np.packbits((1 - h.cpu().numpy()).astype(np.uint8), axis=2)     # imagecore.py:293-294
    assert np.array_equal(pbm.cpu().numpy(), want)
    pbm2 = torch.full_like(pbm, 0x5C)
    net.halftone_device(c, z, pbm_out=pbm2, impl=impl, check=True)     # payload only
    assert torch.equal(pbm2, pbm)
    # a window of rows (row-strip sharding), odd offset
    if H > 4:
        rows = (H, 1, 2, H - 3)
        pw = torch.zeros((B, H - 3, (W + 7) // 8), dtype=torch.uint8, device="cuda")
        hw = torch.empty((B, H - 3, W), dtype=torch.uint8, device="cuda")
        net.halftone_device(c[:, 1:], z[:, 1:], h_out=hw, pbm_out=pw, rows=rows, impl=impl, check=True)
        assert np.array_equal(pw.cpu().numpy(),
                              np.packbits((1 - hw.cpu().numpy()).astype(np.uint8), axis=2))


def test_nonfinite_logits_raise():
    from paper_2304_12152_b200 import rl
    net = _net(0.05)
    net.conv_out.bias.value[0] = np.inf
    with pytest.raises(FloatingPointError):
        rl.halftone(net, np.full((8, 8), 0.5), np.zeros((8, 8)))


def test_infer_halftone_uses_reference_noise_draws():
    from oracle import htoracle as O
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.imagecore import Rng
    net = _net(0.05)
    c = np.linspace(0, 1, 24 * 20).reshape(24, 20)
    h, p = rl.infer_halftone(net, c, Rng(17))
    params = O.init_params(O.Rng(0), 32, 16, 2, 0.05)
    z = O.gaussian_noise_map(O.Rng(17), 20, 24)
    _, p_ref = O.halftone(params, c.astype(np.float32), z.astype(np.float32))
    _check(p, h, p_ref, P_TOL)


def test_device_api_without_sync_reuses_packed_weights():
    """Parameter edits on the host are picked up before the next forward."""
    from paper_2304_12152_b200 import rl
    net = _net(0.05)
    c, z = np.full((16, 16), 0.3), np.zeros((16, 16))
    _, p1 = rl.halftone(net, c, z)
    net.conv_out.bias.value[0] += 1.0
    _, p2 = rl.halftone(net, c, z)
    assert np.all(p2 > p1)


@pytest.mark.parametrize("nb", [0, 1, 2, 3, 5])
def test_fused_pass_plans_for_other_depths(nb):
    """Every pass-plan shape of the fused kernel (conv_in-only, conv_out-only,
    odd block counts) against the reference oracle on the same net (and the
    fp32 SIMT path against it at 2e-5)."""
    from oracle import htoracle as O
    from paper_2304_12152_b200 import rl, synth
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_f32
    net = _net(0.05, 32, nb, seed=nb)
    c = synth.contone(45, 300, seed=nb)
    z = gaussian_noise_map_f32(Rng(nb), 300, 45)
    params = O.init_params(O.Rng(nb), 32, nb, 2, 0.05)
    _, p_ref = O.halftone(params, c.astype(np.float64), z.astype(np.float64))
    h0, p0 = rl.halftone(net, c, z, impl=0)
    h1, p1 = rl.halftone(net, c, z, impl=1)
    _check(p0, h0, p_ref, P_TOL)
    _check(p1, h1, p_ref, 2e-5)


def test_two_networks_on_two_streams_concurrently():
    """Two networks halftoning at the same time on two streams of one GPU
    (each pass's biases travel with its launch, so neither sees the other's):
    the results equal each network's result run alone, bitwise."""
    import torch
    from paper_2304_12152_b200 import synth
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_f32
    nets = [_net(0.05, seed=1), _net(0.05, seed=2)]
    for n in nets:
        n.conv_out.bias.value[0] = 0.3 * (1 if n is nets[0] else -1)
        for blk in n.res:
            blk.conv2.bias.value[:] = 0.01 * (1 if n is nets[0] else -1)
    c = torch.from_numpy(np.stack([synth.contone(256, 256, seed=s) for s in range(8)])).cuda()
    z = torch.from_numpy(np.stack([gaussian_noise_map_f32(Rng(s), 256, 256) for s in range(8)])).cuda()
    alone = []
    for n in nets:
        p = torch.empty_like(c)
        n.halftone_device(c, z, p_out=p, check=True)
        alone.append(p.clone())
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in nets]
    outs = [torch.empty_like(c) for _ in nets]
    wss = [None, None]
    for rep in range(4):
        for k, (n, s) in enumerate(zip(nets, streams)):
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                wss[k] = n.halftone_device(c, z, p_out=outs[k], workspace=wss[k], stream=s)
        torch.cuda.synchronize()
        for k in range(2):
            assert torch.equal(outs[k], alone[k]), f"network {k}, repetition {rep}"
    assert not torch.equal(alone[0], alone[1])


def test_engine_draws_noise_on_device_in_infer_halftone_order():
    """rl.HalftoneEngine(c, rng): image i's noise is the i-th
    gaussian_noise_map of the stream (as B calls of infer_halftone)."""
    import torch
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_device
    net = _net(0.05)
    B, H, W = 3, 40, 52
    r = Rng(8)
    c = torch.from_numpy(r.uniforms(B * H * W).reshape(B, H, W).astype(np.float32)).pin_memory()
    zr = Rng(5)
    z = torch.stack([gaussian_noise_map_device(zr, W, H).cpu() for _ in range(B)]).pin_memory()
    eng = rl.HalftoneEngine(net, B, H, W, chunks=2, output="h")
    o1 = torch.empty(eng.out_shape(), dtype=torch.uint8).pin_memory()
    o2 = torch.empty(eng.out_shape(), dtype=torch.uint8).pin_memory()
    eng(c, z, o1)
    rng = Rng(5)
    eng(c, rng, o2)
    assert torch.equal(o1, o2)
    assert rng.state_words() == zr.state_words()
    assert eng.h2d_bytes(device_noise=True) * 2 == eng.h2d_bytes()


def test_zero_second_convs_make_blocks_identity_bitwise():
    """Reference property (test_nn.py `test_zero_second_conv_is_identity`):
    a residual block whose second conv is zero is the identity.  So a
    16-block network with every conv2 zeroed must give, bit for bit, the
    0-block network with the same conv_in / conv_out -- through every pass of
    the fused kernel (fp32 residual stream carried exactly), at 8 x 512^2."""
    import torch
    from paper_2304_12152_b200 import synth
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_f32
    from paper_2304_12152_b200.nn import PolicyNetwork
    net = _net(0.05)
    for blk in net.res:
        blk.conv2.weight.value[...] = 0.0
        blk.conv2.bias.value[...] = 0.0
    net0 = PolicyNetwork(32, 0)
    for a, b in ((net0.conv_in, net.conv_in), (net0.conv_out, net.conv_out)):
        a.weight.value[...] = b.weight.value
        a.bias.value[...] = b.bias.value
    B, H, W = 8, 512, 512
    c = torch.from_numpy(np.stack([synth.contone(H, W, seed=70 + i) for i in range(B)]).astype(np.float32)).cuda()
    z = torch.from_numpy(np.stack([gaussian_noise_map_f32(Rng(80 + i), W, H) for i in range(B)])).cuda()
    p16 = torch.empty((B, H, W), dtype=torch.float32, device="cuda")
    p0 = torch.empty_like(p16)
    net.halftone_device(c, z, p_out=p16)
    net0.halftone_device(c, z, p_out=p0)
    assert torch.equal(p16, p0)


@pytest.mark.parametrize("noise", ["host", "device"])
def test_engine_streamed_batches_equal_sequential_calls(noise):
    """HalftoneEngine.submit/wait with batches in flight (device buffers
    reused in stream order) gives exactly the per-call results; with device
    noise the RNG stream is consumed batch after batch as sequential calls
    would."""
    import torch
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.imagecore import Rng
    net = _net(0.05)
    B, H, W, n = 5, 33, 70, 4
    r = Rng(3)
    cs = [torch.from_numpy(r.uniforms(B * H * W).reshape(B, H, W).astype(np.float32)).pin_memory()
          for _ in range(n)]
    zs = [torch.from_numpy(r.gaussians_f32(B * H * W).reshape(B, H, W)).pin_memory() for _ in range(n)]
    eng = rl.HalftoneEngine(net, B, H, W, chunks=3, output="h")
    seq, rs = [], Rng(11)
    for i in range(n):
        o = torch.empty(eng.out_shape(), dtype=torch.uint8).pin_memory()
        seq.append(eng(cs[i], zs[i] if noise == "host" else rs, o).clone())
    outs = [torch.empty(eng.out_shape(), dtype=torch.uint8).pin_memory() for _ in range(n)]
    rs2 = Rng(11)
    tickets = [eng.submit(cs[i], zs[i] if noise == "host" else rs2, outs[i]) for i in range(n)]
    for t in tickets:
        eng.wait(t)
    for i in range(n):
        assert torch.equal(outs[i], seq[i]), i
    if noise == "device":
        assert rs2.state_words() == rs.state_words()


@pytest.mark.parametrize("output", ["h", "pbm", "p"])
def test_engine_graph_mode_equals_streamed_path(output):
    """HalftoneEngine(graph=True): the call replays one captured CUDA graph
    (H2D, the nine K1 passes, D2H) and gives exactly the streamed path's
    result; new host buffers or an edited parameter force a recapture, and a
    non-finite logit still raises."""
    import torch
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.imagecore import Rng
    net = _net(0.05)
    B, H, W = 2, 40, 72
    r = Rng(5)
    mk = lambda f: torch.from_numpy(f(B * H * W).reshape(B, H, W).astype(np.float32)).pin_memory()
    c, z = mk(r.uniforms), mk(r.gaussians_f32)
    ref_eng = rl.HalftoneEngine(net, B, H, W, chunks=1, output=output, depth=1)
    eng = rl.HalftoneEngine(net, B, H, W, output=output, depth=1, graph=True)
    dt = ref_eng.out.dtype
    ref = ref_eng(c, z, torch.empty(ref_eng.out_shape(), dtype=dt).pin_memory()).clone()
    o = torch.empty(eng.out_shape(), dtype=dt).pin_memory()
    for _ in range(3):
        o.zero_()
        assert torch.equal(eng(c, z, o), ref)
    g0 = eng._graph
    c.copy_(mk(r.uniforms))                      # same buffers, new contents: same graph
    ref = ref_eng(c, z, torch.empty_like(ref)).clone()
    assert torch.equal(eng(c, z, o), ref) and eng._graph is g0
    net.conv_out.bias.value[0] += 0.5            # edited parameter: recaptured
    ref = ref_eng(c, z, torch.empty_like(ref)).clone()
    assert torch.equal(eng(c, z, o), ref) and eng._graph is not g0
    o2 = torch.empty_like(o)                     # other host buffers: recaptured
    assert torch.equal(eng(c, z, o2), ref)
    c[0, 3, 5] = float("nan")
    with pytest.raises(FloatingPointError):
        eng(c, z, o2)


@pytest.mark.parametrize("case", ["trained_2k", "std0.1"])
def test_config1_beyond_random_init(case):
    """K1 parity with weights that are not the std-0.01 init: the network
    after 2000 iterations of this package's own train_loop (bare HTNN file,
    tests/golden/make_trained_checkpoint.py) and a std-0.1 random init, on
    BASELINE config 1 (256x256) against the oracle's float64 forward.  At
    std 0.1 the activations reach ~1e5 after 16 blocks, beyond fp16's range
    (and beyond what fp32 resolves near the logits' zero crossings): the fused
    kernel flags the overflow and rl.halftone redoes the image in float64 on
    the device, the reference's precision."""
    from oracle import htoracle as O
    from paper_2304_12152_b200 import rl
    from paper_2304_12152_b200.checkpoint import network_from_checkpoint
    from conftest import GOLDEN
    import os
    g = golden("forward.npz")
    if case == "trained_2k":
        net, _ = network_from_checkpoint(os.path.join(GOLDEN, "trained_c32b16_2k.htnn"))
    else:
        net = _net(0.1)
    params = [q.value.copy() for q in net.params()]
    c, z = g["cfg1_c"], g["cfg1_z"]
    _, p_ref = O.halftone(params, c.astype(np.float64), z.astype(np.float64))
    h, p = rl.halftone(net, c, z)
    err, band = _check(p, h, p_ref, P_TOL)
    print(f"{case}: max|dp| = {err:.2e}, band fraction {band:.4f}, "
          f"p range [{p_ref.min():.3f}, {p_ref.max():.3f}]")


def test_host_parameter_edits_reach_the_device():
    """Parameter.value arrays are views of one host buffer (one memory
    compare per use); in-place edits, edits through other views and a
    rebound .value array all reach the kernels."""
    from paper_2304_12152_b200 import rl, synth
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_f32
    net = _net(0.05, nb=2)
    c = synth.contone(20, 24, seed=4)
    z = gaussian_noise_map_f32(Rng(4), 24, 20)
    _, p0 = rl.halftone(net, c, z)
    net.conv_out.bias.value[0] += 0.5                      # in place
    _, p1 = rl.halftone(net, c, z)
    assert np.all(p1 > p0)
    net.conv_out.bias.value.reshape(-1)[0] -= 0.5          # through another view
    _, p2 = rl.halftone(net, c, z)
    assert np.array_equal(p2, p0)
    net.conv_out.bias.value = np.array([1.0])              # rebound
    _, p3 = rl.halftone(net, c, z)
    assert np.all(p3 > p0)
    net.conv_out.bias.value = np.array([0.0])
    _, p4 = rl.halftone(net, c, z)
    assert np.array_equal(p4, p0)


def test_fp16_overflow_redo_covers_every_output():
    """The float64 redo (activations beyond fp16's range) fills p, h, the
    PBM payload and multitone levels like the fused kernel would, on a
    row window and on a side stream."""
    import torch
    from oracle import htoracle as O
    from paper_2304_12152_b200 import synth
    from paper_2304_12152_b200.imagecore import Rng, gaussian_noise_map_f32
    net = _net(0.1)
    H, W = 40, 50
    c = torch.from_numpy(np.stack([synth.contone(H, W, seed=s) for s in (1, 2)])).cuda()
    z = torch.from_numpy(np.stack([gaussian_noise_map_f32(Rng(s), W, H) for s in (1, 2)])).cuda()
    params = [q.value.copy() for q in net.params()]
    p_ref = np.stack([O.halftone(params, c[i].double().cpu().numpy()[5:], z[i].double().cpu().numpy()[5:])[1]
                      for i in range(2)])
    rows = (H, 5, 7, H - 12)            # input rows 5.., output rows 7..7+H-12 (window-relative 2..)
    ci, zi = c[:, 5:].contiguous(), z[:, 5:].contiguous()
    s = torch.cuda.Stream()
    p = torch.empty((2, H - 12, W), device="cuda")
    h = torch.empty((2, H - 12, W), dtype=torch.uint8, device="cuda")
    pbm = torch.empty((2, H - 12, (W + 7) // 8), dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(s):
        net.halftone_device(ci, zi, p_out=p, h_out=h, pbm_out=pbm, rows=rows, check=True, stream=s)
    s.synchronize()
    want = p_ref[:, 2:2 + H - 12]
    assert np.max(np.abs(p.cpu().numpy() - want)) < 1e-6
    hh = h.cpu().numpy()
    assert np.array_equal(pbm.cpu().numpy(), np.packbits((1 - hh).astype(np.uint8), axis=2))
    q = torch.empty_like(h)
    net.halftone_device(ci, zi, h_out=q, rows=rows, check=True, levels=4)
    levels = np.rint(O.quantize_multitone(want, 4) * 3).astype(np.uint8)   # multitone.py:61-67
    assert np.array_equal(q.cpu().numpy(), levels)
