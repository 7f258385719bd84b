"""Single-box partitioners (one process per GPU): views sharded across ranks
(cone / modular), or z-slabs without any collective (parallel beam).

north_star item (4).  The reference has no multi-device path (SURVEY.md
section 0, gap 3); this module adds it around the unchanged single-GPU pair:

* forward: rank r projects views [a_r, b_r) of the full (replicated) volume
  -- no communication at all;
* back:    rank r back-projects its views into a full-size partial volume and
  the partial volumes are summed so that each rank owns one z-slab of A^T y
  (``back``), or an all-reduce leaves every rank the whole volume
  (``back_replicated``).  On NCCL process groups the SF back projection goes
  through the native fused path (``ctp_sf_back_sharded``, csrc/dist.cu): the
  partial volume is produced in 256-slice z-chunks and each finished chunk is
  reduced to its slab owners on a communication stream while the next chunk
  is back-projected.  Otherwise (gloo tests, Siddon)
  one reduce-scatter follows the whole back projection.

Parallel beam (``ZSlabParallelProjector``): rank r owns detector rows
[r0, r1) in the forward and volume slices [z0, z1) in the back projection,
with a one-slice / one-row halo; no communication.

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
        plan = self.pair.plan(self.device_index)
        return (plan.siddon_forward if self.pair.model == "siddon" else plan.forward)(x, out=out)

    def back(self, y, out=None):
        plan = self.pair.plan(self.device_index)
        return (plan.siddon_back if self.pair.model == "siddon" else plan.back)(y, out=out)


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
        self._dist = None
        self.native = False
        if isinstance(backend, CudaBackend) and pair.model == "sf" and world > 1:
            import torch.distributed as dist

            self.native = dist.is_initialized() and dist.get_backend(group) == "nccl"

    def native_dist(self):
        """The rank's ctp_dist (NCCL communicator of the fused back projection),
        created on first use; the 128-byte id travels over the process group."""
        if self._dist is None:
            from ._native import Dist

            if self.world == 1:
                self._dist = Dist(Dist.make_id(), 1, 0, self.backend.device_index)
            else:
                import torch.distributed as dist

                obj = [Dist.make_id() if self.rank == 0 else None]
                dist.broadcast_object_list(obj, src=0, group=self.group)
                self._dist = Dist(obj[0], self.world, self.rank, self.backend.device_index)
        return self._dist

    def back_native(self, y_local, out=None):
        """Fused back projection + per-z-chunk reductions (csrc/dist.cu): this
        rank's z-slab [B, slab, ny, nx]."""
        plan = self.shard.plan(self.backend.device_index)
        return self.native_dist().back_sharded(plan, y_local.contiguous(), out=out)

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

        if self.native:
            return self.back_native(y_local)
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


# --------------------------------------------------------------------------
# parallel beam: z-slabs, no communication (north_star item 4)
# --------------------------------------------------------------------------
def even_ranges(n: int, world: int):
    """Balanced contiguous [a, b) ranges of 0..n-1 over ``world`` ranks."""
    if world > n:
        raise ValueError(f"cannot split {n} items over {world} ranks")
    return view_ranges(n, world)


def _row_z(det, row_edge: float) -> float:
    """World z of a detector row boundary (parallel beam: vax = +z, t = z)."""
    return (row_edge - det.centerRow) * det.pixelHeight


def rows_of_slices(g, spec, z0: int, z1: int):
    """Detector rows [ra, rb) that slices [z0, z1) can reach (parallel beam:
    rays have no z component, so slice iz only reaches the rows covering
    [z_lo + iz hz, z_lo + (iz + 1) hz]; one row of margin each side)."""
    det = g.detector
    lo, _ = spec.bounds()
    za, zb = lo[2] + z0 * spec.voxelHeight, lo[2] + z1 * spec.voxelHeight
    ra = math.floor(za / det.pixelHeight + det.centerRow + 0.5) - 1
    rb = math.ceil(zb / det.pixelHeight + det.centerRow - 0.5) + 2
    return max(ra, 0), min(rb, det.numRows)


def slices_of_rows(g, spec, r0: int, r1: int):
    """Volume slices [za, zb) that rows [r0, r1) can receive from (one slice
    of margin each side)."""
    det = g.detector
    lo, _ = spec.bounds()
    za_w, zb_w = _row_z(det, r0 - 0.5), _row_z(det, r1 - 0.5)
    za = math.floor((za_w - lo[2]) / spec.voxelHeight) - 1
    zb = math.ceil((zb_w - lo[2]) / spec.voxelHeight) + 1
    return max(za, 0), min(zb, spec.numZ)


def row_subgeometry(g, r0: int, r1: int):
    """The same scanner restricted to detector rows [r0, r1)."""
    from dataclasses import replace

    det = g.detector
    return replace(g, detector=replace(det, numRows=r1 - r0, centerRow=det.centerRow - r0))


class ZSlabParallelProjector:
    """One rank's share of an N-way z-partitioned PARALLEL-beam SF pair.

    Parallel rays have no z component (geometry.py pose table: vax = +z), so
    detector row r only sees the slices covering its z range.  Forward: rank
    r owns detector rows [r0, r1) of every view and projects the slices that
    reach them (its row slab plus a one-slice halo); back: rank r owns volume
    slices [z0, z1) and back-projects the rows that reach them (plus a
    one-row halo).  Outputs are disjoint, inputs are read-only: no
    collective at all.  Each sub-problem is a plan over a row sub-geometry
    and a z-slab VolumeSpec, so only the fp32 rounding of the offsets
    differs from the single-GPU pair (results equal within 1e-6).
    """

    def __init__(self, pair, rank: int, world: int, device=None, backend_factory=None):
        from .chunking import slab_spec
        from .geometry import PARALLEL
        from .operator import ProjectorPair

        g, spec = pair.geometry, pair.volumeSpec
        if g.kind != PARALLEL:
            raise ValueError("z-slab partitioning needs parallel-beam geometry (use ViewShardedProjector)")
        self.full, self.rank, self.world = pair, rank, world
        nr, nz = g.detector.numRows, spec.numZ
        # forward: detector rows of this rank, the slices reaching them
        self.rows = even_ranges(nr, world)[rank]
        self.fwd_slices = slices_of_rows(g, spec, *self.rows)
        a, b = self.fwd_slices
        self.fwd_pair = (ProjectorPair(pair.model, row_subgeometry(g, *self.rows), slab_spec(spec, a, b - a))
                         if b > a else None)
        # back: volume slices of this rank, the rows reaching them
        self.slices = even_ranges(nz, world)[rank]
        self.back_rows = rows_of_slices(g, spec, *self.slices)
        ra, rb = self.back_rows
        z0, z1 = self.slices
        self.back_pair = (ProjectorPair(pair.model, row_subgeometry(g, ra, rb), slab_spec(spec, z0, z1 - z0))
                          if rb > ra else None)
        if backend_factory is None:
            idx = device.index if device is not None else 0
            backend_factory = lambda p: CudaBackend(p, idx)  # noqa: E731
        self._fwd = backend_factory(self.fwd_pair) if self.fwd_pair is not None else None
        self._back = backend_factory(self.back_pair) if self.back_pair is not None else None

    def forward(self, x):
        """x [B, nz, ny, nx] (or just its slices ``fwd_slices``) -> rows
        ``rows`` of every view [B, nv, r1 - r0, nc]."""
        import torch

        g = self.full.geometry
        a, b = self.fwd_slices
        if self._fwd is None:  # no slice reaches these rows
            return torch.zeros((x.shape[0], g.numViews, self.rows[1] - self.rows[0], g.detector.numCols),
                               dtype=torch.float32, device=x.device)
        xs = x[:, a:b] if x.shape[1] == self.full.volumeSpec.numZ else x
        return self._fwd.forward(xs.contiguous())

    def back(self, y):
        """y [B, nv, nr, nc] (or just its rows ``back_rows``) -> slices
        ``slices`` of A^T y [B, z1 - z0, ny, nx]."""
        import torch

        spec = self.full.volumeSpec
        ra, rb = self.back_rows
        if self._back is None:  # these slices project outside the detector
            return torch.zeros((y.shape[0], self.slices[1] - self.slices[0], spec.numY, spec.numX),
                               dtype=torch.float32, device=y.device)
        ys = y[:, :, ra:rb] if y.shape[2] == self.full.geometry.detector.numRows else y
        return self._back.back(ys.contiguous())
