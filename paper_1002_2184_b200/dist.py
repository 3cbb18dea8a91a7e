"""Multi-GPU plumbing for the Fast Haar path.

One process per GPU over torch.distributed (NCCL on B200, gloo in the CPU tests).  The transform
partitions into independent units (reading R1: pairs (x[2k], x[2k+1]) make every 2^L-aligned
block independent), so sharding needs no halo exchange:

* batched signals / images (c2, c4): rank r owns units [r*U/N, (r+1)*U/N) of the fixed global
  batch U (strong scaling: BASELINE c4 splits its 256 images across 1/2/4/8 GPUs; c2 its 4096
  signals), no collective on the data path; `unit_shard` keeps the opt-in weak-scaling split;
* one large image (c5): rank r owns rows [r*h/N, (r+1)*h/N), a multiple of 2^L rows; its band
  output equals rows [r*h/N >> j, (r+1)*h/N >> j) of every global level-j band.  The coarsest LL
  of all bands is all-gathered (the only exchange; 64 KiB for c5).

Only host arithmetic and the collective live here; the packing is the library's
fhwt_pack_ll_2d kernel on GPU (callers pass the packed tensor).  PeerLLGather is the opt-in
alternative that fuses the pack with the gather (fhwt_pack_ll_2d_peers stores into every peer's
symmetric-memory buffer over NVLink).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def unit_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Strong scaling: (first unit, count) of `rank`'s contiguous share of `total` independent units
    (images / signals).  Equal shares; the first total % world ranks take one unit more."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if total < world:
        raise ValueError(f"{total} units do not give each of {world} ranks one")
    q, r = divmod(total, world)
    first = rank * q + min(rank, r)
    return first, q + (1 if rank < r else 0)


def unit_shard(units_per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling (opt-in): (first unit, count) owned by `rank` of a global batch world*units."""
    return rank * units_per_rank, units_per_rank


def row_band(h: int, world: int, rank: int, levels: int) -> tuple[int, int]:
    """Rows [r0, r1) of an h-row image owned by `rank` (strong split into 2^levels-aligned bands)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if h % world:
        raise ValueError(f"h={h} does not split into {world} equal bands")
    rows = h // world
    if rows % (1 << levels):
        raise ValueError(f"band of {rows} rows is not a multiple of 2^{levels}: bands would need a halo")
    return rank * rows, (rank + 1) * rows


def band_rows(r0: int, r1: int, level: int) -> tuple[int, int]:
    """Rows of the global level-`level` bands that a band [r0, r1) produces."""
    return r0 >> level, r1 >> level


def segment_1d(n: int, world: int, rank: int, levels: int) -> tuple[int, int]:
    """One very long 1-D signal split into `world` contiguous segments of 2^levels-aligned length
    (§8(f) f2): samples [s0, s1) owned by `rank`.  Segments transform independently (reading R1)."""
    return row_band(n, world, rank, levels)


def segment_bands_1d(s0: int, s1: int, n: int, levels: int) -> dict:
    """Where a segment's local Mallat output [a_J | d_J | ... | d_1] (length s1 - s0) lands in the
    global Mallat layout of the n-sample signal: {band: (local_start, global_start, length)}."""
    seg = s1 - s0
    out = {"a": (0, s0 >> levels, seg >> levels)}
    for j in range(1, levels + 1):
        out[f"d{j}"] = (seg >> j, (n >> j) + (s0 >> j), seg >> j)
    return out


def gather_coarse_ll(ll_local: torch.Tensor, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather the packed coarsest LL of every rank's row band, concatenated along rows
    (rank order = row order).  NCCL: all_gather_into_tensor on the device (NVLink); other backends
    (gloo, CPU tests): all_gather through host memory."""
    world = dist.get_world_size(group)
    shape = (world * ll_local.shape[0],) + tuple(ll_local.shape[1:])
    if out is None:
        out = torch.empty(shape, dtype=ll_local.dtype, device=ll_local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, ll_local.contiguous(), group=group)
        return out
    src = ll_local.detach().to("cpu").contiguous()
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src, group=group)
    out.copy_(torch.cat(parts, dim=0))
    return out


def max_over_ranks(values, device=None, group=None):
    """Device-timed quantities are reported as the max over ranks (a float or a list of floats)."""
    scalar = not isinstance(values, (list, tuple))
    vals = [float(values)] if scalar else [float(v) for v in values]
    if dist.get_backend(group) != "nccl":
        device = "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    res = [float(v) for v in t.tolist()]
    return res[0] if scalar else res


class PeerLLGather:
    """The coarsest-LL all-gather of row-band sharding, fused with the pack over peer memory
    (NVLink P2P): every rank stores its band's LL straight into each peer's symmetric buffer
    (fhwt_pack_ll_2d_peers, one kernel), then one device-side cross-rank barrier (torch symmetric
    memory) on the same stream makes the stores visible.  The result is laid out as
    gather_coarse_ll's (rank order = row order).  Needs CUDA devices with peer access (one node,
    NVLink / NVSwitch).

    Two buffer slots alternate between calls: call k writes slot k % 2 on every rank, so a rank
    may still read call k-1's result (stream-ordered before its call k+1) while faster peers
    already store call k.  Call k+1 reuses the slot of call k-1, which every rank finished reading
    before it entered call k's barrier (reads are consumed before the next call on the stream)."""

    def __init__(self, rows_per_rank: int, cols: int, group=None, device=None):
        import torch.distributed._symmetric_memory as symm_mem
        group = group or dist.group.WORLD
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.rows, self.cols = rows_per_rank, cols
        device = device or torch.device("cuda", torch.cuda.current_device())
        self._mem = symm_mem.empty((2, self.world * rows_per_rank, cols), dtype=torch.float32, device=device)
        self.handle = symm_mem.rendezvous(self._mem, group.group_name)
        slot = self.world * rows_per_rank * cols * 4
        # per slot: a device array of every peer's slot base address (the kernel's peer table)
        self._peers = [torch.tensor([int(p) + k * slot for p in self.handle.buffer_ptrs], dtype=torch.int64,
                                    device=device) for k in range(2)]
        self._calls = 0

    @property
    def buf(self) -> torch.Tensor:
        """The slot of the latest call's result."""
        return self._mem[(self._calls - 1) % 2]

    def __call__(self, coeffs: torch.Tensor, levels: int, stream=None) -> torch.Tensor:
        """Gather on `stream` (default: the current stream).  The returned slot stays valid until
        the call after next; read it on `stream` (or after synchronising with it): the slot
        reuse argument above assumes the result is consumed in stream order."""
        from . import pack_ll_2d_peers
        # one 2-D band per rank: a leading batch > 1 would make the kernel store past the rank's slot
        if (coeffs.dim() < 2 or coeffs.shape[-2] >> levels != self.rows or coeffs.shape[-1] >> levels != self.cols
                or coeffs.numel() != (self.rows << levels) * (self.cols << levels)):
            raise ValueError("coefficient band does not match the gather buffer")
        k = self._calls % 2
        stream = stream or torch.cuda.current_stream(self._mem.device)
        with torch.cuda.stream(stream):   # the barrier kernel runs on torch's current stream
            pack_ll_2d_peers(coeffs, levels, self._peers[k].data_ptr(), self.handle.rank, self.handle.world_size,
                             stream=stream)
            self.handle.barrier(channel=0)
        self._calls += 1
        return self._mem[k]
