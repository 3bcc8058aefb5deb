"""HTNN checkpoint files (reference nn.py:200-300 and its
tests test_nn.py:236-320).  Pinned against files written by the reference's
own save_checkpoint (tests/golden/make_checkpoint_golden.py)."""

import os

import numpy as np
import pytest

from paper_2304_12152_b200.imagecore import Rng
from paper_2304_12152_b200.nn import (Adam, CheckpointError, PolicyNetwork, load_checkpoint,
                                      network_from_checkpoint, read_checkpoint, save_checkpoint)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _flat(bufs):
    return np.concatenate([b.ravel() for b in bufs])


def _pair(seed=21):
    net = PolicyNetwork(channels=4, blocks=2, in_channels=2)
    net.init_params(Rng(seed), std=0.3)
    adam = Adam(net.params())
    r = Rng(seed + 1)
    adam.t = 3
    for m, v in zip(adam.m, adam.v):
        m[...] = r.gaussians(m.size).reshape(m.shape)
        v[...] = np.abs(r.gaussians(v.size)).reshape(v.shape)
    return net, adam


def test_reads_reference_written_file():
    ref = np.load(os.path.join(GOLD, "ckpt_ref.npz"))
    meta, values, m, v = read_checkpoint(os.path.join(GOLD, "ckpt_ref.htnn"))
    assert meta == {"in_channels": 2, "channels": 4, "blocks": 2, "iteration": 5,
                    "adam_t": int(ref["adam_t"]), "rng_state": tuple(int(w) for w in ref["rng_state"])}
    assert np.array_equal(_flat(values), ref["values"])
    assert np.array_equal(_flat(m), ref["m"]) and np.array_equal(_flat(v), ref["v"])
    shapes = [p.value.shape for p in PolicyNetwork(4, 2).params()]
    assert [a.shape for a in values] == shapes


def test_writes_reference_bytes(tmp_path):
    """Re-saving the decoded reference file reproduces it byte for byte."""
    net, meta = network_from_checkpoint(os.path.join(GOLD, "ckpt_ref.htnn"))
    adam = Adam(net.params())
    load_checkpoint(os.path.join(GOLD, "ckpt_ref.htnn"), net, adam)
    out = tmp_path / "re.htnn"
    save_checkpoint(out, net, adam, iteration=meta["iteration"], rng_state=meta["rng_state"])
    assert out.read_bytes() == open(os.path.join(GOLD, "ckpt_ref.htnn"), "rb").read()
    bare = tmp_path / "bare.htnn"
    save_checkpoint(bare, net)
    assert bare.read_bytes() == open(os.path.join(GOLD, "ckpt_ref_bare.htnn"), "rb").read()


def test_roundtrip_is_bitwise(tmp_path):
    net, adam = _pair()
    path = tmp_path / "ck.htnn"
    save_checkpoint(path, net, adam, iteration=7, rng_state=(1, 2, 3, 4))
    meta, values, m, v = read_checkpoint(path)
    assert meta == {"in_channels": 2, "channels": 4, "blocks": 2, "iteration": 7, "adam_t": 3,
                    "rng_state": (1, 2, 3, 4)}
    assert np.array_equal(_flat(values), net.flat_values())
    assert np.array_equal(_flat(m), _flat(adam.m)) and np.array_equal(_flat(v), _flat(adam.v))
    fresh = PolicyNetwork(channels=4, blocks=2)
    fresh_adam = Adam(fresh.params())
    got = load_checkpoint(path, fresh, fresh_adam)
    assert got["iteration"] == 7 and fresh_adam.t == 3
    assert np.array_equal(fresh.flat_values(), net.flat_values())
    assert np.array_equal(_flat(fresh_adam.m), _flat(adam.m))


def test_bare_params_file(tmp_path):
    net, _ = _pair()
    path = tmp_path / "bare.htnn"
    save_checkpoint(path, net)
    _, _, m, v = read_checkpoint(path)
    assert m is None and v is None
    fresh = PolicyNetwork(channels=4, blocks=2)
    load_checkpoint(path, fresh)
    with pytest.raises(CheckpointError):
        load_checkpoint(path, fresh, Adam(fresh.params()))


def test_arch_mismatch(tmp_path):
    net, _ = _pair()
    path = tmp_path / "ck.htnn"
    save_checkpoint(path, net)
    with pytest.raises(CheckpointError):
        load_checkpoint(path, PolicyNetwork(channels=4, blocks=1))


def test_corrupt_files(tmp_path):
    raw = open(os.path.join(GOLD, "ckpt_ref_bare.htnn"), "rb").read()
    cases = {"short": raw[:20], "trunc": raw[:-16], "magic": b"XTNN" + raw[4:],
             "version": raw[:4] + (2).to_bytes(4, "little") + raw[8:], "ragged": raw + b"\0\0\0"}
    for name, blob in cases.items():
        path = tmp_path / f"{name}.htnn"
        path.write_bytes(blob)
        with pytest.raises(CheckpointError):
            read_checkpoint(path)
    assert issubclass(CheckpointError, ValueError)


@pytest.mark.gpu
def test_checkpoint_drives_fused_kernel(tmp_path):
    """A loaded file reaches the device path: the fused kernel's output follows
    the file's weights (checked against the oracle on those weights)."""
    import torch
    from oracle import htoracle as O
    from paper_2304_12152_b200 import rl
    src = PolicyNetwork(32, 2)
    src.init_params(Rng(41), std=0.05)
    path = tmp_path / "w.htnn"
    save_checkpoint(path, src)
    net = PolicyNetwork(32, 2)
    net.init_params(Rng(0), std=0.01)
    r = Rng(3)
    c = r.uniforms(48 * 40).reshape(48, 40).astype(np.float32)
    z = r.gaussians(48 * 40).reshape(48, 40).astype(np.float32)
    before = rl.halftone(net, c, z)[1]
    load_checkpoint(path, net)
    h, p = rl.halftone(net, c, z)
    ref = O.policy_forward([pp.value for pp in src.params()],
                           np.stack((c, z)).astype(np.float64)[None])[0, 0]
    assert np.max(np.abs(p - ref)) <= 1e-3
    assert np.max(np.abs(before - ref)) > 1e-3      # the weights really changed
    assert torch.cuda.is_available()


@pytest.mark.gpu
def test_resumed_training_matches_unsplit(tmp_path):
    """rl.train_loop: 2 iterations == 1 iteration + checkpoint + resume."""
    from paper_2304_12152_b200 import rl
    cfg = rl.TrainConfig(iterations=2, batch_size=2, crop_size=16, anisotropy_batch_size=1,
                         channels=8, blocks=1, hvs_size=5, seed=9)
    r = Rng(2)
    dataset = [r.uniforms(24 * 24).reshape(24, 24), np.full((24, 24), 0.4)]
    full_net, full_adam, full_rng = rl.train_loop(cfg, dataset)
    path = tmp_path / "mid.htnn"

    def stop_after_first(t, diag, net, adam, rng):
        if t == 0:
            save_checkpoint(path, net, adam, iteration=1, rng_state=rng.state_words())

    rl.train_loop(rl.TrainConfig(**{**cfg.__dict__, "iterations": 1}), dataset, on_iteration=stop_after_first)
    res_net, res_adam, res_rng = rl.train_loop(cfg, dataset, resume_path=path)
    assert list(res_rng.state_words()) == list(full_rng.state_words())
    assert res_adam.t == full_adam.t == 2
    a, b = res_net.flat_values(), full_net.flat_values()
    assert np.max(np.abs(a - b)) <= 1e-12 * max(1.0, np.abs(b).max())
