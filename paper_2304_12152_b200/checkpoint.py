"""HTNN checkpoint files: trained weights -> the fused
device path.

Same on-disk format as the reference (`nn.py:200-300`), so files move freely
between htlab and this package:

    header  little-endian  magic "HTNN" | u32 version (1) | u32 in_channels |
            u32 channels | u32 blocks | u64 iteration | u64 adam step |
            4 x u64 RNG state words                               (72 bytes)
    body    every parameter tensor in `PolicyNetwork.params()` order as <f8,
            optionally followed by Adam's m then v blobs (same order).

Loading writes the host `Parameter.value` arrays in place; the device copy
and its packed fp16 UMMA tiles are rebuilt on next use (`PolicyNetwork.sync`),
and Adam's device moments are re-uploaded from the restored host lists.
"""

import struct

import numpy as np

MAGIC = b"HTNN"
VERSION = 1
_HEAD = struct.Struct("<4s4I2Q4Q")


class CheckpointError(ValueError):
    """Malformed file or architecture mismatch (nn.py:219-220)."""


def _layout(in_channels, channels, blocks):
    from .nn import PolicyNetwork
    shapes = [p.value.shape for p in PolicyNetwork(channels, blocks, in_channels).params()]
    return shapes, [int(np.prod(s)) for s in shapes]


def save_checkpoint(path, net, adam=None, iteration=0, rng_state=(0, 0, 0, 0)):
    """nn.py:209-217.  Device-resident Adam moments are pulled first."""
    if adam is not None:
        adam.pull_state()
    blobs = [p.value for p in net.params()]
    if adam is not None:
        blobs += list(adam.m) + list(adam.v)
    head = _HEAD.pack(MAGIC, VERSION, net.in_channels, net.channels, net.blocks, int(iteration),
                      int(adam.t) if adam is not None else 0, *[int(w) for w in rng_state])
    with open(path, "wb") as fh:
        fh.write(head)
        for b in blobs:
            fh.write(np.ascontiguousarray(b, dtype="<f8").tobytes())


def read_checkpoint(path):
    """nn.py:223-268: (meta, values, m, v); m and v are None for a bare file."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _HEAD.size:
        raise CheckpointError("file shorter than checkpoint header")
    magic, ver, in_ch, ch, nb, iteration, adam_t, *words = _HEAD.unpack_from(raw)
    if magic != MAGIC:
        raise CheckpointError(f"bad magic {magic!r}")
    if ver != VERSION:
        raise CheckpointError(f"unsupported version {ver}")
    shapes, sizes = _layout(in_ch, ch, nb)
    n = sum(sizes)
    if (len(raw) - _HEAD.size) % 8:
        raise CheckpointError("body is not a whole number of float64 values")
    body = np.frombuffer(raw, dtype="<f8", offset=_HEAD.size)
    if body.size not in (n, 3 * n):
        raise CheckpointError(f"blob length {body.size} does not match arch "
                              f"(C={ch}, B={nb}): expected {n} or {3 * n}")
    meta = {"in_channels": in_ch, "channels": ch, "blocks": nb, "iteration": iteration,
            "adam_t": adam_t, "rng_state": tuple(words)}

    def tensors(vec):
        offs = np.cumsum([0] + sizes)
        return [vec[offs[i]:offs[i + 1]].reshape(s).copy() for i, s in enumerate(shapes)]

    values = tensors(body[:n])
    if body.size == 3 * n:
        return meta, values, tensors(body[n:2 * n]), tensors(body[2 * n:])
    return meta, values, None, None


def load_checkpoint(path, net, adam=None):
    """nn.py:271-291: restore into an existing net (and Adam); returns meta."""
    meta, values, m, v = read_checkpoint(path)
    if (meta["in_channels"], meta["channels"], meta["blocks"]) != (net.in_channels, net.channels,
                                                                   net.blocks):
        raise CheckpointError(f"arch mismatch: file C={meta['channels']} B={meta['blocks']} "
                              f"vs net C={net.channels} B={net.blocks}")
    for p, val in zip(net.params(), values):
        p.value[...] = val
    if adam is not None:
        if m is None:
            raise CheckpointError("checkpoint carries no optimizer state")
        adam.t = meta["adam_t"]
        for dst, src in zip(adam.m, m):
            dst[...] = src
        for dst, src in zip(adam.v, v):
            dst[...] = src
        adam.invalidate_device_state()
    return meta


def network_from_checkpoint(path):
    """nn.py:294-300: a fresh net with the file's architecture and weights."""
    from .nn import PolicyNetwork
    meta, values, _, _ = read_checkpoint(path)
    net = PolicyNetwork(channels=meta["channels"], blocks=meta["blocks"],
                        in_channels=meta["in_channels"])
    for p, val in zip(net.params(), values):
        p.value[...] = val
    return net, meta
