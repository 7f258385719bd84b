"""Single-box partitioner: views sharded across ranks (one process per GPU).

north_star item (4).  The reference has no multi-device path (SURVEY.md
section 0, gap 3); this module adds it around the unchanged single-GPU pair:

* forward: rank r projects views [a_r, b_r) of the full (replicated) volume
  -- no communication at all;
* back:    rank r back-projects its views into a full-size partial volume,
  then ONE reduce-scatter (sum, fp32) over NCCL / NVLink leaves each rank the
  z-slab it owns of A^T y (``back``), or an all-reduce leaves every rank the
  whole volume (``back_replicated``).

Because the sum over views is split into per-rank partial sums, the N-GPU
back projection equals the 1-GPU result up to fp32 summation order;
``virtual_back`` reproduces exactly the N-rank arithmetic on one device
(partials summed in rank order) for testing.

The projector is injected (``backend``) so the same sharding logic runs on
the CUDA plans in production and on any CPU callable in the gloo tests.
"""

from __future__ import annotations

import math
from dataclasses import dataclass


def view_ranges(nv: int, world: int):
    """Balanced contiguous view shards [(a, b)] for ranks 0..world-1."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    base, extra = divmod(nv, world)
    out, a = [], 0
    for r in range(world):
        b = a + base + (1 if r < extra else 0)
        out.append((a, b))
        a = b
    return out


def slab_size(nz: int, world: int) -> int:
    """z-slab owned per rank after the reduce-scatter (nz padded up)."""
    return math.ceil(nz / world)


@dataclass
class CudaBackend:
    """Device backend: the SF plans of one rank's view shard."""

    pair: object  # ProjectorPair over the shard's views
    device_index: int

    def forward(self, x, out=None):
        return self.pair.plan(self.device_index).forward(x, out=out)

    def back(self, y, out=None):
        return self.pair.plan(self.device_index).back(y, out=out)


class ViewShardedProjector:
    """One rank's share of an N-way view-sharded SF pair."""

    def __init__(self, pair, rank: int, world: int, device=None, group=None, backend=None):
        from .operator import ProjectorPair

        self.full = pair
        self.rank, self.world, self.group = rank, world, group
        nv = pair.geometry.numViews
        if world > nv:
            raise ValueError(f"cannot shard {nv} views over {world} ranks")
        self.ranges = view_ranges(nv, world)
        a, b = self.ranges[rank]
        self.views = (a, b)
        self.shard = ProjectorPair(pair.model, pair.geometry.with_views(range(a, b)), pair.volumeSpec)
        self.device = device
        if backend is None:
            backend = CudaBackend(self.shard, device.index if device is not None else 0)
        self.backend = backend
        nz = pair.volumeSpec.numZ
        self.slab = slab_size(nz, world)
        self.nz_pad = self.slab * world

    # -- forward: no communication -------------------------------------------
    def forward(self, x):
        """x [B, nz, ny, nx] (replicated) -> this rank's views [B, nv_r, nr, nc]."""
        return self.backend.forward(x)

    # -- back: partial volume + reduce-scatter ---------------------------------
    def _partial(self, y_local):
        import torch

        B = y_local.shape[0]
        spec = self.full.volumeSpec
        part = torch.zeros((B, self.nz_pad, spec.numY, spec.numX), dtype=torch.float32,
                           device=y_local.device)
        if B == 1 or self.nz_pad == spec.numZ:
            self.backend.back(y_local, out=part[:, : spec.numZ])  # contiguous view
        else:
            part[:, : spec.numZ] = self.backend.back(y_local)
        return part

    def back(self, y_local):
        """This rank's views -> the z-slab [B, slab, ny, nx] of A^T y it owns
        (slab r covers z in [r*slab, (r+1)*slab), zero-padded past nz)."""
        import torch
        import torch.distributed as dist

        part = self._partial(y_local)
        if self.world == 1:
            return part
        B = part.shape[0]
        # reduce-scatter along z: make the z-slab the leading (scattered) dim
        src = part[0] if B == 1 else part.transpose(0, 1).contiguous()  # [nz_pad, (B,) ny, nx]
        out = torch.empty((self.slab,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
        if dist.get_backend(self.group) == "gloo":
            # gloo has no reduce_scatter: all-reduce then keep our slab (CPU tests only)
            dist.all_reduce(src, group=self.group)
            out.copy_(src[self.rank * self.slab:(self.rank + 1) * self.slab])
        else:
            dist.reduce_scatter_tensor(out, src, group=self.group)
        if B == 1:
            return out[None]
        return out.transpose(0, 1).contiguous()

    def back_replicated(self, y_local):
        """All-reduce variant: every rank gets the whole A^T y [B, nz, ny, nx]."""
        import torch.distributed as dist

        part = self._partial(y_local)
        if self.world > 1:
            dist.all_reduce(part, group=self.group)
        return part[:, : self.full.volumeSpec.numZ]


def virtual_back(pair, y, world: int, backend_factory):
    """Single-device emulation of the N-rank back projection: per-shard
    partial volumes summed in rank order (what the reduce-scatter computes,
    up to NCCL's own reduction order)."""
    import torch

    ranges = view_ranges(pair.geometry.numViews, world)
    total = None
    for a, b in ranges:
        be = backend_factory(pair, a, b)
        part = be.back(y[:, a:b].contiguous())
        total = part.clone() if total is None else total + part
    return total


def gather_slabs(slabs, nz: int):
    """Concatenate per-rank z-slabs (rank order) and drop the padding."""
    import torch

    return torch.cat(list(slabs), dim=1)[:, :nz]
