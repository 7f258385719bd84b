"""View-chunked streaming between host memory and the device.

The reference bounds memory by processing one batch element at a time
(operator.py:59-75) and keeps "one copy of the projection data and volume
data".  Here the host<->device traffic of a host-resident call
is split into view chunks so copies overlap the kernels:

* forward  (host volume -> host sinogram): the volume goes up once, then
  chunk k of views is projected on the compute stream while chunk k-1 is
  copied down on a copy stream into pinned host memory;
* back     (host sinogram -> host volume): chunk k+1 of views is copied up on
  the copy stream while chunk k is back-projected into the resident volume
  with CTP_FLAG_ACCUMULATE; the volume comes down once at the end.

Every chunk is a plan over ``Geometry.with_views`` of a contiguous view
range, so the arithmetic per view is identical to the unchunked call
(forward: bitwise; back: the per-voxel view sum is split into chunk partial
sums, i.e. a different fp32 summation order).

z-slabs (``zslab_apply``) bound the device working set by the volume side:
the grid is cut into slabs of ``nzs`` slices (each a plan over a VolumeSpec
with the slab's numZ / offsetZ).  Forward: slab k+1 is uploaded while slab k is
projected and accumulated into the resident sinogram (CTP_FLAG_ACCUMULATE).
Back: slab k is back-projected from the resident sinogram while slab k-1 is
copied down.  Only one slab of the volume is on the device at a time (two
while overlapping).
"""

from __future__ import annotations

import math
import os

from . import _native

#: target bytes of sinogram per chunk (host<->device granularity)
CHUNK_BYTES = int(os.environ.get("CTPROJ_CHUNK_BYTES", str(256 << 20)))


def _torch():
    import torch

    return torch


def view_chunks(nv: int, view_bytes: int, chunk_bytes: int = CHUNK_BYTES):
    """Contiguous [a, b) view ranges of about ``chunk_bytes`` each.  Chunks of
    32 views or more are whole multiples of 32: the back kernel sets up 32
    views per lane-parallel pass, so a ragged chunk would idle lanes."""
    per = max(1, min(nv, chunk_bytes // max(1, view_bytes)))
    if 32 <= per < nv:
        per = per // 32 * 32
    else:
        n = math.ceil(nv / per)
        per = math.ceil(nv / n)
    return [(a, min(nv, a + per)) for a in range(0, nv, per)]


def chunk_plans(plan: "_native.Plan", ranges):
    g, spec, dev = plan.geometry, plan.spec, plan.device.index
    if len(ranges) == 1:
        return [plan]
    return [_native.get_plan(g.with_views(range(a, b)), spec, dev) for a, b in ranges]


#: at most this many view chunks per call: each chunk is one kernel launch, and
#: a back-projection launch re-reads and re-writes the accumulated volume
MAX_CHUNKS = int(os.environ.get("CTPROJ_MAX_CHUNKS", "8"))


def host_apply(plan: "_native.Plan", host, direction: int, chunk_bytes: int | None = None):
    """Apply A (direction 0) / A^T (1) to a host f32 tensor [B, ...]; returns
    a pinned host tensor.  The whole batch moves together (so batched paths
    such as the fan-beam kernels apply); views are chunked by bytes
    (``CHUNK_BYTES``, or more per chunk so there are at most ``MAX_CHUNKS``)."""
    torch = _torch()
    dev = plan.device
    B = int(host.shape[0])
    nv, nr, nc = plan.sino_shape
    view_bytes = B * nr * nc * 4
    if chunk_bytes is None:
        chunk_bytes = max(CHUNK_BYTES, math.ceil(nv * view_bytes / MAX_CHUNKS))
    ranges = view_chunks(nv, view_bytes, chunk_bytes)
    plans = chunk_plans(plan, ranges)
    compute = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    src = host if host.is_pinned() else host.pin_memory()
    # one device buffer for the whole sinogram (chunks are slices of it when
    # B == 1, where a view range is contiguous): no per-chunk allocations, so
    # repeated calls reuse the same caching-allocator blocks
    whole = B == 1
    with torch.cuda.device(dev):
        if direction == 0:
            out = torch.empty((B,) + tuple(plan.sino_shape), dtype=torch.float32, pin_memory=True)
            xd = src.to(dev, non_blocking=True)
            yall = torch.empty((B,) + tuple(plan.sino_shape), dtype=torch.float32, device=dev) if whole else None
            for (a, e), p in zip(ranges, plans):
                yd = p.forward(xd, out=yall[:, a:e]) if whole else p.forward(xd)
                ev = torch.cuda.Event()
                ev.record(compute)
                copy.wait_event(ev)
                with torch.cuda.stream(copy):
                    if len(ranges) == 1:
                        out.copy_(yd, non_blocking=True)
                    else:
                        out[:, a:e].copy_(yd, non_blocking=True)
                    if not whole:
                        yd.record_stream(copy)
            compute.wait_stream(copy)
            compute.synchronize()
            return out
        out_d = torch.empty((B,) + tuple(plan.vol_shape), dtype=torch.float32, device=dev)
        yall = torch.empty((B,) + tuple(plan.sino_shape), dtype=torch.float32, device=dev) if whole else None
        for k, ((a, e), p) in enumerate(zip(ranges, plans)):
            with torch.cuda.stream(copy):
                part = src if len(ranges) == 1 else src[:, a:e]
                if whole:
                    yd = yall[:, a:e]
                    yd.copy_(part, non_blocking=True)
                else:
                    yd = part.to(dev, non_blocking=True).contiguous()
            ev = torch.cuda.Event()
            ev.record(copy)
            compute.wait_event(ev)
            if not whole:
                yd.record_stream(compute)
            p.back(yd, out=out_d, accumulate=k > 0)
        out = torch.empty((B,) + tuple(plan.vol_shape), dtype=torch.float32, pin_memory=True)
        out.copy_(out_d, non_blocking=True)
        compute.synchronize()
        return out


def slab_spec(spec, z_first: int, nzs: int):
    """VolumeSpec of slices [z_first, z_first + nzs) of ``spec``."""
    from .geometry import VolumeSpec

    lo = spec.offsetZ - spec.numZ * spec.voxelHeight / 2.0
    center = lo + (z_first + nzs / 2.0) * spec.voxelHeight
    return VolumeSpec(numX=spec.numX, numY=spec.numY, numZ=nzs, voxelWidth=spec.voxelWidth,
                      voxelHeight=spec.voxelHeight, offsetX=spec.offsetX, offsetY=spec.offsetY,
                      offsetZ=center)


def zslab_ranges(nz: int, nzs: int):
    return [(a, min(nz, a + nzs)) for a in range(0, nz, nzs)]


def zslab_apply(plan: "_native.Plan", host, direction: int, nzs: int):
    """Host tensor in -> pinned host tensor out, streaming the volume in
    z-slabs of ``nzs`` slices (see module docstring)."""
    torch = _torch()
    dev = plan.device
    g, spec = plan.geometry, plan.spec
    B = int(host.shape[0])
    ranges = zslab_ranges(spec.numZ, nzs)
    plans = [_native.get_plan(g, slab_spec(spec, a, b - a), dev.index) for a, b in ranges]
    compute = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    src = host if host.is_pinned() else host.pin_memory()
    with torch.cuda.device(dev):
        if direction == 0:
            yd = torch.zeros((B,) + tuple(g.shape), dtype=torch.float32, device=dev)
            for b in range(B):
                for k, ((a, e), p) in enumerate(zip(ranges, plans)):
                    with torch.cuda.stream(copy):
                        xs = src[b:b + 1, a:e].to(dev, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy)
                    compute.wait_event(ev)
                    xs.record_stream(compute)
                    p.forward(xs, out=yd[b:b + 1], accumulate=True)
            out = torch.empty((B,) + tuple(g.shape), dtype=torch.float32, pin_memory=True)
            out.copy_(yd, non_blocking=True)
            compute.synchronize()
            return out
        yd = src.to(dev, non_blocking=True)
        out = torch.empty((B,) + tuple(spec.shape), dtype=torch.float32, pin_memory=True)
        for b in range(B):
            for (a, e), p in zip(ranges, plans):
                xs = p.back(yd[b:b + 1])
                ev = torch.cuda.Event()
                ev.record(compute)
                copy.wait_event(ev)
                with torch.cuda.stream(copy):
                    out[b, a:e].copy_(xs[0], non_blocking=True)
                    xs.record_stream(copy)
        compute.wait_stream(copy)
        compute.synchronize()
        return out
