"""Multi-GPU plumbing for the halftoning hot path (one process per GPU).

Inference shards with no collective on the data path:
  * by image   -- config 2/3: rank r halftones images [lo, hi) of the batch;
  * by row strip -- config 4: rank r owns output rows [o0, o1) of a page and
    reads input rows [o0 - 34, o1 + 34) clipped to the page.  34 is the
    receptive-field radius of the 34 stacked 3x3 convs, and the fused kernel
    zero-pads only at true image edges, so stitched strips are bitwise equal
    to the unsharded result (tests/test_gpu_forward.py).
Training is data parallel: every rank consumes the full host RNG stream,
computes its shard of the batch, and gradients plus the three diagnostic
sums are all-reduced once per step (rl.train_step).
"""

from dataclasses import dataclass

RECEPTIVE_RADIUS = 34   # 34 stacked 3x3 convs (nn.py:109-116)


def shard_range(n, rank, world):
    """Contiguous shard [lo, hi) of n items for `rank` (shard sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


@dataclass(frozen=True)
class RowStrip:
    """Rows a rank reads (input window) and writes (output rows) of a page."""
    in_row0: int
    in_rows: int
    out_row0: int
    out_rows: int

    def as_kernel_rows(self, height):
        """(H, in_row0, out_row0, out_rows) for PolicyNetwork.halftone_device."""
        return (height, self.in_row0, self.out_row0, self.out_rows)


def receptive_radius(blocks):
    """Receptive-field radius of a PolicyNetwork with `blocks` residual
    blocks: 2*blocks + 2 stacked 3x3 convs (34 for the paper network)."""
    return 2 * blocks + 2


def row_strip(height, rank, world, halo=RECEPTIVE_RADIUS):
    """Row strip of `rank` for a page of `height` rows split over `world`
    ranks (halo = the network's receptive_radius)."""
    o0, o1 = shard_range(height, rank, world)
    i0, i1 = max(0, o0 - halo), min(height, o1 + halo)
    return RowStrip(i0, i1 - i0, o0, o1 - o0)


def dist_info(group=None):
    import torch
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        return torch.distributed.get_rank(group), torch.distributed.get_world_size(group)
    return 0, 1


def allreduce_sum_(*tensors, group=None):
    """In-place SUM all-reduce of gradient / statistics tensors (no-op for one rank)."""
    import torch
    _, world = dist_info(group)
    if world == 1:
        return tensors
    for t in tensors:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM, group=group)
    return tensors


def halftone_shard(net, contones, noises, group=None, **kw):
    """Halftone this rank's image shard of a (B, H, W) batch (numpy / CPU
    arrays); returns (lo, hi, h) with h the uint8 halftones of images [lo, hi)."""
    from .rl import halftone_batch
    rank, world = dist_info(group)
    lo, hi = shard_range(len(contones), rank, world)
    if hi == lo:
        return lo, hi, None
    return lo, hi, halftone_batch(net, contones[lo:hi], noises[lo:hi], **kw)


def halftone_page_strip(net, page, noise, group=None, output="h"):
    """Halftone this rank's row strip of one page (H, W) (config 4).

    Returns (strip, out) with out the (out_rows, W) uint8 halftone rows."""
    import numpy as np
    import torch
    rank, world = dist_info(group)
    H, W = page.shape
    st = row_strip(H, rank, world, halo=receptive_radius(net.blocks))
    dev = net.device
    c = torch.from_numpy(np.ascontiguousarray(page[st.in_row0:st.in_row0 + st.in_rows],
                                              dtype=np.float32)).to(dev)[None]
    z = torch.from_numpy(np.ascontiguousarray(noise[st.in_row0:st.in_row0 + st.in_rows],
                                              dtype=np.float32)).to(dev)[None]
    h = torch.empty((1, st.out_rows, W), dtype=torch.uint8, device=dev)
    net.halftone_device(c, z, h_out=h, rows=st.as_kernel_rows(H), check=True)
    return st, h[0].cpu().numpy()


class PageEngine:
    """Streams pages of one size (H, W) through this rank's row strip
    (config 4): host contone + noise pages (float32, pinned for asynchronous
    copies) in, the strip's uint8 halftone rows (1 = white) out.  Each
    submitted page runs H2D -> fused forward -> D2H on the stream of one of
    `depth` device-buffer sets, so page i+1's copies overlap page i's
    kernels; wait() blocks until a page's rows are in its out_host."""

    def __init__(self, net, H, W, group=None, depth=2):
        import torch
        from . import _lib
        _lib.require_cuda()
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.net, self.H, self.W = net, H, W
        rank, world = dist_info(group)
        self.strip = st = row_strip(H, rank, world, halo=receptive_radius(net.blocks))
        dev = net.device
        self.dev = dev
        self._sets = [{"stream": torch.cuda.Stream(dev, priority=-1),
                       "c": torch.empty((1, st.in_rows, W), dtype=torch.float32, device=dev),
                       "z": torch.empty((1, st.in_rows, W), dtype=torch.float32, device=dev),
                       "h": torch.empty((1, st.out_rows, W), dtype=torch.uint8, device=dev),
                       "ws": None} for _ in range(depth)]
        self._next = 0
        net.sync()

    def out_shape(self):
        return (self.strip.out_rows, self.W)

    def h2d_bytes(self):
        return 2 * self.strip.in_rows * self.W * 4

    def d2h_bytes(self):
        return self.strip.out_rows * self.W

    def submit(self, page, noise, out_host):
        """Enqueue one page: page / noise (H, W) float32 CPU tensors (pinned
        for overlap), out_host (out_rows, W) uint8 CPU tensor; returns a
        ticket for wait().  Inputs must stay unchanged and out_host unread
        until then."""
        import numpy as np
        import torch
        st, s = self.strip, self._sets[self._next % len(self._sets)]
        if tuple(page.shape) != (self.H, self.W) or tuple(noise.shape) != (self.H, self.W):
            raise ValueError(f"page and noise must be ({self.H}, {self.W})")
        if not isinstance(out_host, torch.Tensor) or tuple(out_host.shape) != self.out_shape() \
                or out_host.dtype != torch.uint8 or out_host.device.type != "cpu":
            raise ValueError(f"out_host must be a CPU uint8 tensor of shape {self.out_shape()}")
        # numpy inputs work too (pageable: their copies do not overlap)
        page = torch.from_numpy(np.ascontiguousarray(page, dtype=np.float32)) if isinstance(page, np.ndarray) else page
        noise = torch.from_numpy(np.ascontiguousarray(noise, dtype=np.float32)) if isinstance(noise, np.ndarray) else noise
        self._next += 1
        stream = s["stream"]
        stream.wait_stream(torch.cuda.current_stream(self.dev))
        r0, r1 = st.in_row0, st.in_row0 + st.in_rows
        with torch.cuda.stream(stream):
            s["c"][0].copy_(page[r0:r1], non_blocking=True)
            s["z"][0].copy_(noise[r0:r1], non_blocking=True)
            s["ws"] = self.net.halftone_device(s["c"], s["z"], h_out=s["h"], rows=st.as_kernel_rows(self.H),
                                               workspace=s["ws"], stream=stream)
            out_host.copy_(s["h"][0], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        return (ev, s)

    def wait(self, ticket):
        """Block until a submitted page's rows are in its out_host.  Raises
        FloatingPointError if the fused kernel saw a non-finite logit."""
        import torch
        from . import _lib
        ev, s = ticket
        torch.cuda.current_stream(self.dev).wait_event(ev)
        ev.synchronize()
        _lib.call("ht_halftone_check", _lib.ptr(s["ws"]), _lib.stream_ptr(s["stream"]))
