"""Multi-GPU plumbing for the sketched path.

One process per GPU (torchrun), NCCL over NVLink through torch.distributed.
Nonzeros are sharded in contiguous mode-0 slabs of the lexsorted COO (equal
nnz, split at i_0 boundaries).  Every sketch of the path is a sum over stored
entries, so each rank sketches its shard and the partial sketches are summed
with one all-reduce per sketch (TensorSketch right-hand sides, RRF stage 1,
fitness cross terms, gathered fibres, ||T||^2); the small dense algebra is
replicated -- identical inputs and deterministic kernels give bitwise
identical replicas on every rank.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(slice_counts, world):
    """Split mode-0 slices into `world` contiguous groups of ~equal nonzeros.

    slice_counts[i] = nonzeros with i_0 == i.  Returns a list of
    (i0_lo, i0_hi, e_lo, e_hi) with nnz offsets into the lexsorted order."""
    counts = np.asarray(slice_counts, dtype=np.int64)
    world = int(world)
    if world < 1:
        raise ValueError("world size must be >= 1")
    cum = np.concatenate([[0], np.cumsum(counts)])
    total = int(cum[-1])
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        i = int(np.searchsorted(cum, target, side="left"))
        # choose the slice boundary closest to the target, never going back
        if i > 0 and abs(cum[i - 1] - target) <= abs(cum[min(i, len(cum) - 1)] - target):
            i -= 1
        cuts.append(max(i, cuts[-1]))
    cuts.append(len(counts))
    return [(cuts[r], cuts[r + 1], int(cum[cuts[r]]), int(cum[cuts[r + 1]])) for r in range(world)]


class Comm:
    """Sum all-reduce over the default process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._sibling = None

    def sibling(self):
        """A second communicator over the same ranks (created once, by every
        rank at the same point of the program) for collectives issued from
        another CUDA stream -- the per-sweep fitness all-reduce runs beside the
        next sweep's collectives, and operations of one NCCL communicator must
        not run concurrently on two streams."""
        if self._sibling is None:
            self._sibling = Comm(self.dist.new_group(ranks=list(range(self.world)))) \
                if self.world > 1 else self
        return self._sibling

    def allreduce(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def allgather(self, t):
        """Concatenation of every rank's equally-shaped 1-D tensor `t`, rank order."""
        if self.world == 1:
            return t
        import torch
        t = t.contiguous()
        if self.dist.get_backend(self.group) == "nccl":
            out = torch.empty(self.world * t.numel(), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t, group=self.group)
            return out
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t, group=self.group)
        return torch.cat(parts)

    def split(self, lo, hi):
        """This rank's contiguous share of the integer range [lo, hi)."""
        n = hi - lo
        return lo + n * self.rank // self.world, lo + n * (self.rank + 1) // self.world

    def row_chunk(self, s):
        """Rows per rank of an s-row matrix split for reduce-scatter/all-gather
        (equal chunks; the last rank's chunk is padded)."""
        return -(-s // self.world)

    def row_slab(self, s):
        """[lo, hi) rows of an s-row matrix owned by this rank."""
        c = self.row_chunk(s)
        return min(self.rank * c, s), min((self.rank + 1) * c, s)

    def reduce_scatter_rows(self, t):
        """Sum over ranks of the (s, ...) tensor t, returning this rank's row slab
        (row_slab(s)) -- half the traffic of an all-reduce, and every rank keeps
        only its part."""
        import torch
        s = t.shape[0]
        c = self.row_chunk(s)
        if self.world == 1:
            return t
        flat = t.reshape(s, -1)
        if c * self.world != s:
            flat = torch.cat([flat, flat.new_zeros((c * self.world - s, flat.shape[1]))])
        out = flat.new_empty((c, flat.shape[1]))
        if self.dist.get_backend(self.group) == "nccl":
            self.dist.reduce_scatter_tensor(out, flat.contiguous(), op=self.dist.ReduceOp.SUM,
                                            group=self.group)
        else:  # gloo has no reduce-scatter: all-reduce and keep the slab
            full = flat.contiguous().clone()
            self.dist.all_reduce(full, op=self.dist.ReduceOp.SUM, group=self.group)
            out.copy_(full[self.rank * c:(self.rank + 1) * c])
        lo, hi = self.row_slab(s)
        return out[:hi - lo].reshape((hi - lo,) + tuple(t.shape[1:]))

    def allgather_rows(self, t, s):
        """Inverse of the row split: every rank's (row_slab) rows -> the full
        (s, ...) tensor on all ranks."""
        import torch
        if self.world == 1:
            return t
        c = self.row_chunk(s)
        flat = t.reshape(t.shape[0], -1)
        if flat.shape[0] < c:
            flat = torch.cat([flat, flat.new_zeros((c - flat.shape[0], flat.shape[1]))])
        full = self.allgather(flat.contiguous().reshape(-1)).reshape(self.world * c, -1)[:s]
        return full.reshape((s,) + tuple(t.shape[1:]))


def shard_device_coo(coords, vals, shape, world, rank):
    """Rank `rank`'s mode-0 slab of a lexsorted (N, nnz) device COO."""
    import torch
    counts = torch.bincount(coords[0].long(), minlength=shape[0]).cpu().numpy()
    lo_i, hi_i, lo, hi = shard_bounds(counts, world)[rank]
    return coords[:, lo:hi].contiguous(), vals[lo:hi].contiguous(), (lo_i, hi_i)
