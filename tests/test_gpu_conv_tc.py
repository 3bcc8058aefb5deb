"""The tcgen05 training convolutions (csrc/conv_tc2.cu: scaled fp16 pairs, the
default where the shape allows TMA staging; csrc/conv_tc.cu: split bf16)
against the fp32 SIMT kernel and a float64 reference, one conv at a time,
every epilogue option."""

import numpy as np
import pytest

from paper_2304_12152_b200.imagecore import Rng

pytestmark = pytest.mark.gpu


def _conv64(x, w):
    """float64 cross-correlation with zero padding (nn.py:46-60)."""
    B, C, H, W = x.shape
    xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)))
    out = np.zeros((B, w.shape[0], H, W))
    for ky in range(3):
        for kx in range(3):
            out += np.einsum("bchw,oc->bohw", xp[:, :, ky:ky + H, kx:kx + W], w[:, :, ky, kx])
    return out


def _run(impl, x, w, bias=None, mask=None, resid=None, relu=0):
    import torch
    from paper_2304_12152_b200 import _lib
    t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa
    xd, wd, bd, md, rd = t(x), t(w), t(bias), t(mask), t(resid)
    out = torch.empty_like(xd)
    B, C, H, W = x.shape
    _lib.call("ht_conv3x3_32", _lib.ptr(xd), B, H, W, _lib.ptr(wd), _lib.ptr(bd), _lib.ptr(md),
              _lib.ptr(rd), _lib.ptr(out), relu, impl, _lib.stream_ptr())
    torch.cuda.synchronize()
    return out.double().cpu().numpy()


# (W % 4 == 0 and W + 1 >= 128 take the TMA-staged input path: strips that
# straddle two images, box starts at every 16-B phase)
@pytest.mark.parametrize("B,H,W", [(1, 5, 6), (2, 20, 24), (3, 40, 52), (1, 7, 300), (2, 130, 67),
                                   (3, 9, 128), (3, 6, 132), (4, 5, 136), (2, 11, 256),
                                   # many short segments per CTA (issuer / worker phase
                                   # tracking across strips), single-row images
                                   (8, 3, 128), (5, 2, 252), (4, 1, 128)])
@pytest.mark.parametrize("mode", ["plain", "bias_relu", "mask", "resid"])
@pytest.mark.parametrize("impl", [0, 2, 3])
def test_conv_tc_matches_reference(B, H, W, mode, impl):
    r = Rng(B * 1000 + H * 10 + W)
    x = r.gaussians(B * 32 * H * W).reshape(B, 32, H, W).astype(np.float32).astype(np.float64)
    w = (r.gaussians(32 * 32 * 9).reshape(32, 32, 3, 3) * 0.1).astype(np.float32).astype(np.float64)
    kw = {}
    ref = _conv64(x, w)
    if mode == "bias_relu":
        b = r.gaussians(32).astype(np.float32).astype(np.float64)
        kw = dict(bias=b, relu=1)
        ref = np.maximum(ref + b[None, :, None, None], 0.0)
    elif mode == "mask":
        m = (r.uniforms(x.size).reshape(x.shape) - 0.5).astype(np.float32).astype(np.float64)
        kw = dict(mask=m)
        ref = np.where(m > 0, ref, 0.0)
    elif mode == "resid":
        rs = r.gaussians(x.size).reshape(x.shape).astype(np.float32).astype(np.float64)
        kw = dict(resid=rs)
        ref = ref + rs
    tc = _run(impl, x, w, **kw)
    simt = _run(1, x, w, **kw)
    scale = np.abs(_conv64(np.abs(x), np.abs(w))).max()
    assert np.max(np.abs(simt - ref)) <= 1e-5 * scale
    # split bf16 / scaled fp16 pairs with short accumulation chains: ~1e-7 of
    # scale (SIMT ~2e-7)
    assert np.max(np.abs(tc - ref)) <= 1e-6 * scale, np.unravel_index(np.argmax(np.abs(tc - ref)), ref.shape)


@pytest.mark.parametrize("xscale,wscale", [(1.0, 1.0), (1e-9, 1.0), (1e6, 1e-3), (1e-12, 1e-3)])
def test_conv_tc2_row_scales(xscale, wscale):
    """The fp16-pair kernel scales every input row by its own power of two:
    inputs far outside fp16's range (the backward pass's 1e-9 gradients) and
    rows whose magnitudes differ by 1e12 keep the fp32-class error per row."""
    B, H, W = 3, 24, 256
    r = Rng(77)
    x = r.gaussians(B * 32 * H * W).reshape(B, 32, H, W)
    rowmag = 10.0 ** r.uniforms(B * H).reshape(B, 1, H, 1) * 1e-6 ** r.uniforms(B * H).reshape(B, 1, H, 1)
    x = (x * rowmag * xscale).astype(np.float32).astype(np.float64)
    w = (r.gaussians(32 * 32 * 9).reshape(32, 32, 3, 3) * 0.1 * wscale).astype(np.float32).astype(np.float64)
    ref = _conv64(x, w)
    tc = _run(3, x, w)
    # error bound per output row: the scale of the three input rows it reads
    sc = _conv64(np.abs(x), np.abs(w))
    rows = np.abs(x).max(axis=(1, 3))                         # (B, H)
    rp = np.pad(rows, ((0, 0), (1, 1)))
    near = np.maximum(np.maximum(rp[:, :-2], rp[:, 1:-1]), rp[:, 2:])
    bound = 1e-6 * np.maximum(sc.max(axis=(1, 3)), near * np.abs(w).sum(axis=(1, 2, 3)).max())
    err = np.abs(tc - ref).max(axis=(1, 3))
    assert np.all(np.isfinite(tc))
    assert np.all(err <= bound), float((err / bound).max())


@pytest.mark.parametrize("B,H,W", [(3, 9, 128), (5, 2, 252), (1, 7, 300), (2, 11, 256)])
@pytest.mark.parametrize("mode", ["plain", "mask", "resid"])
def test_conv_tc2_cta_pairs_bitwise(B, H, W, mode):
    """The fp16-pair conv on CTA pairs (tcgen05.mma.cta_group::2, M = 256,
    each CTA holding half of every weight window; ht_set_conv_pair(1)) gives
    bitwise the one-CTA-per-strip results, odd strip counts included."""
    from paper_2304_12152_b200 import _lib
    r = Rng(B * 7 + H * 3 + W)
    x = r.gaussians(B * 32 * H * W).reshape(B, 32, H, W).astype(np.float32).astype(np.float64)
    w = (r.gaussians(32 * 32 * 9).reshape(32, 32, 3, 3) * 0.1).astype(np.float32).astype(np.float64)
    b = r.gaussians(32).astype(np.float32).astype(np.float64)
    e = r.gaussians(x.size).reshape(x.shape).astype(np.float32).astype(np.float64)
    kw = dict(bias=b, relu=1)
    if mode == "mask":
        kw["mask"] = e
    elif mode == "resid":
        kw["resid"] = e
    single = _run(3, x, w, **kw)
    _lib.call("ht_set_conv_pair", 1)
    try:
        pair = _run(3, x, w, **kw)
    finally:
        _lib.call("ht_set_conv_pair", 0)
    assert np.array_equal(pair, single)


@pytest.mark.parametrize("mode", ["plain", "resid", "mask"])
def test_conv_tc2_back_to_back_deterministic(mode):
    """Back-to-back launches (each a programmatic dependent of the previous:
    its prologue overlaps that launch's tail) on fixed inputs give bitwise
    identical outputs -- no race between the roles' barriers, the staging
    rings and the overlapped prologues."""
    import torch
    from paper_2304_12152_b200 import _lib
    torch.manual_seed(1)
    B, H, W = 6, 96, 256
    x = torch.randn(B, 32, H, W, device="cuda")
    w = torch.randn(32, 32, 3, 3, device="cuda") * 0.05
    bias = torch.randn(32, device="cuda")
    e = torch.randn_like(x)
    m = _lib.ptr(e) if mode == "mask" else None
    r = _lib.ptr(e) if mode == "resid" else None
    outs = [torch.empty_like(x) for _ in range(24)]
    for o in outs:
        _lib.call("ht_conv3x3_32", _lib.ptr(x), B, H, W, _lib.ptr(w), _lib.ptr(bias), m, r, _lib.ptr(o), 1, 0,
                  _lib.stream_ptr())
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
