"""Weight / bias gradient of the 32 -> 32 training convs on tcgen05
(csrc/wgrad_tc.cu) against an fp64 restatement of Conv2d.backward's dW, db
(reference nn.py:62-77) and against the fp32 SIMT kernel, through the C-ABI."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ref(x, dout):
    """dW[co, ci, ky, kx] = sum_{b,y,x} dout[b,co,y,x] * xpad[b,ci,y+ky,x+kx], db = sum dout."""
    B, _, H, W = x.shape
    xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)))
    dw = np.zeros((32, 32, 3, 3))
    for ky in range(3):
        for kx in range(3):
            dw[:, :, ky, kx] = np.einsum("bchw,bdhw->cd", dout, xp[:, :, ky:ky + H, kx:kx + W], optimize=True)
    return dw, dout.sum(axis=(0, 2, 3))


def _run(x, dout, impl, parts, dw0=None):
    import torch
    from paper_2304_12152_b200 import _lib
    B, _, H, W = x.shape
    xd = torch.from_numpy(x.astype(np.float32)).cuda()
    dd = torch.from_numpy(dout.astype(np.float32)).cuda()
    dw = torch.zeros(32 * 32 * 9, dtype=torch.float64, device="cuda") if dw0 is None else \
        torch.from_numpy(dw0.ravel().copy()).cuda()
    db = torch.zeros(32, dtype=torch.float64, device="cuda")
    _lib.call("ht_wgrad3x3_32", C.c_void_p(xd.data_ptr()), C.c_void_p(dd.data_ptr()), B, H, W,
              C.c_void_p(dw.data_ptr()), C.c_void_p(db.data_ptr()), impl, parts, None)
    torch.cuda.synchronize()
    return dw.cpu().numpy().reshape(32, 32, 3, 3), db.cpu().numpy()


def _inputs(B, H, W, seed):
    r = np.random.default_rng(seed)
    x = r.standard_normal((B, 32, H, W)).astype(np.float32).astype(np.float64)
    d = (r.standard_normal((B, 32, H, W)) * 1e-2).astype(np.float32).astype(np.float64)
    return x, d


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("B,H,W", [(1, 4, 32), (2, 9, 45), (1, 33, 70), (3, 16, 64), (1, 1, 1), (1, 5, 3)])
def test_wgrad_vs_fp64(B, H, W):
    x, d = _inputs(B, H, W, 100 * H + W)
    dw_ref, db_ref = _ref(x, d)
    for parts, tol in ((3, 1e-6), (2, 2e-5)):
        dw, db = _run(x, d, 0, parts)
        assert _rel(dw, dw_ref) < tol, (parts, _rel(dw, dw_ref))
        assert np.max(np.abs(db - db_ref)) <= 1e-6 * max(1.0, np.max(np.abs(db_ref)))
    dw1, db1 = _run(x, d, 1, 3)
    assert _rel(dw1, dw_ref) < 1e-6


def test_wgrad_accumulates_and_cancels():
    """+= semantics (the caller sums over samples) and a gradient with heavy
    cancellation (dout of mean ~0 against an x with a large constant part)."""
    B, H, W = 2, 20, 37
    x, d = _inputs(B, H, W, 5)
    x = x + 10.0
    dw_ref, db_ref = _ref(x, d)
    base = np.full((32, 32, 3, 3), 0.25)
    dw, _ = _run(x, d, 0, 3, dw0=base)
    assert _rel(dw - base, dw_ref) < 1e-5
    dw2, _ = _run(x, d, 0, 2)
    assert _rel(dw2, dw_ref) < 1e-4


def test_wgrad_large_vs_fp64_and_simt():
    """8 and 20 x 256^2 (config-5 crop size): both implementations against
    fp64.  The tensor-core error stays flat as the batch grows (its TMEM
    accumulation chains are restarted every few tiles and summed with fp32
    adds; measured 1.8e-6 at both sizes) while SIMT's per-thread fp32 sums
    grow (7.7e-7 -> 1.2e-6); both far inside the 1e-4 gradient bar."""
    errs = {}
    for B in (8, 20):
        x, d = _inputs(B, 256, 256, 9)
        dw_ref, db_ref = _ref(x, d)
        dw0, db0 = _run(x, d, 0, 3)
        dw2, _ = _run(x, d, 0, 2)
        dw1, _ = _run(x, d, 1, 3)
        errs[B] = (_rel(dw0, dw_ref), _rel(dw2, dw_ref), _rel(dw1, dw_ref))
        assert errs[B][0] < 4e-6 and errs[B][1] < 1.5e-5 and errs[B][2] < 1e-4, errs
        assert np.max(np.abs(db0 - db_ref)) < 1e-5 * np.max(np.abs(db_ref))
    assert errs[20][0] < 1.3 * errs[8][0], errs
