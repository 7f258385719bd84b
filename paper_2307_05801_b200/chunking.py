"""Streaming between host memory and the device: view chunks x z-slabs.

The reference bounds memory by processing one batch element at a time
(operator.py:59-66) and keeps "one copy of the projection data and volume
data".  Here a host-resident call is cut into blocks of
(z-slab of the volume) x (view chunk of the sinogram), each an ordinary plan
over ``slab_spec`` / ``Geometry.with_views``, so the device only ever holds
two slabs, two view chunks and one kernel workspace -- whatever the sizes of
the volume and the sinogram (north_star item 3):

* forward (host volume -> host sinogram): for each view chunk, the slabs are
  uploaded in turn (copy stream, double-buffered) and projected into the
  chunk with CTP_FLAG_ACCUMULATE; the finished chunk is copied down on a
  second copy stream while the next chunk is projected.  With one slab the
  volume goes up once;
* back (host sinogram -> host volume): for each slab, the view chunks are
  uploaded in turn and back-projected into the slab with CTP_FLAG_ACCUMULATE;
  the finished slab is copied down while the next slab is computed.  With one
  view chunk the sinogram goes up once.

Every device buffer is a slot of a two-entry ring; an upload into a slot waits
for the event of the kernel that last read it, a kernel writing a slot waits
for the download that last read it, so the streams never race on recycled
memory (the caching allocator may hand out blocks still in use on
another stream).

``plan_blocks`` picks the sizes from a device budget: CTPROJ_DEVICE_BUDGET
(bytes) if set, else 80% of the free device memory; CTPROJ_ZSLAB forces a
slab size, CTPROJ_CHUNK_BYTES / CTPROJ_MAX_CHUNKS (/ CTPROJ_MAX_CHUNKS_FWD for
the forward) tune the view chunks, CTPROJ_FWD_STREAMS the forward's compute
streams.
Forward with one slab is bitwise identical to one resident call; slabs and
back chunks only change the fp32 summation order (tested < 1e-6).
"""

from __future__ import annotations

import math
import os

from . import _native
from .errors import CudaRuntimeError

#: target bytes of sinogram per view chunk (host<->device granularity)
CHUNK_BYTES = int(os.environ.get("CTPROJ_CHUNK_BYTES", str(256 << 20)))
#: at most about this many view chunks per call when everything fits: each
#: chunk is one launch (a launch tail, a re-transposed volume, a back
#: projection's read-modify-write of its slab) while fewer chunks expose more
#: of the first upload / last download; measured on C3 (tools/e2e_chunks.py,
#: with ``taper``; median fwd + back call ms): MAX_CHUNKS 1: 476, 2: 445,
#: 3: 441, 4: 463, 6: 470
MAX_CHUNKS = int(os.environ.get("CTPROJ_MAX_CHUNKS", "3"))
#: the forward's own cap: its chunks alternate on two compute streams
#: (FWD_STREAMS), so a chunk's launch tails (~3 ms per tile-parity launch on
#: C3: a task is one view x 4 columns x 768 rows) overlap the next chunk's
#: start; measured on C3 (tools/e2e_ab.py, median forward call ms): 3 chunks
#: 258.4 with one or two streams, 6 chunks 278.3 on one stream, 252.6 on two,
#: 8 chunks 255.3 on two
MAX_CHUNKS_FWD = int(os.environ.get("CTPROJ_MAX_CHUNKS_FWD", "6"))
#: compute streams the forward's view chunks alternate on (volume resident)
FWD_STREAMS = int(os.environ.get("CTPROJ_FWD_STREAMS", "2"))


_FWD_STREAM = {}  # device index -> the forward's second compute stream


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


def device_budget(device) -> int:
    """Bytes a streamed call may hold on ``device``."""
    forced = int(os.environ.get("CTPROJ_DEVICE_BUDGET", "0"))
    if forced > 0:
        return forced
    torch = _torch()
    return int(0.8 * torch.cuda.mem_get_info(device)[0])


def block_bytes(g, spec, batch: int, nzs: int, nvc: int) -> int:
    """Device bytes a streamed call holds for slabs of ``nzs`` slices and view
    chunks of ``nvc`` views: two slab slots + two chunk slots + the larger
    kernel workspace (a transposed copy of the launch's input, ctp_sf_*)."""
    xs = 4 * batch * spec.numX * spec.numY * nzs
    yc = 4 * batch * nvc * g.detector.numRows * g.detector.numCols
    return 2 * xs + 2 * yc + max(xs, yc)


def plan_blocks(g, spec, batch: int, budget: int, direction: int = 1):
    """(nzs, view ranges) for a streamed call within ``budget`` bytes: the
    whole volume with up to MAX_CHUNKS view chunks (or 32-view chunks) when
    that fits; otherwise z-slabs with the largest view chunks that still leave
    room for at least one slice (down to single views)."""
    nv, nz = g.numViews, spec.numZ
    view_bytes = 4 * batch * g.detector.numRows * g.detector.numCols
    slice_bytes = 4 * batch * spec.numX * spec.numY
    forced = int(os.environ.get("CTPROJ_ZSLAB", "0"))
    chunk = max(CHUNK_BYTES, math.ceil(nv * view_bytes / (MAX_CHUNKS_FWD if direction == 0 else MAX_CHUNKS)))
    options = []
    for nvc_cap in (chunk // view_bytes, 32, 1):
        ranges = view_chunks(nv, view_bytes, max(1, nvc_cap) * view_bytes)
        nvc = max(b - a for a, b in ranges)
        if forced > 0:
            nzs = min(forced, nz)
        else:
            room = budget - 3 * nvc * view_bytes  # 2 chunk slots + (at most) a chunk workspace
            nzs = min(nz, room // (3 * slice_bytes)) if room > 0 else 0
        if nzs >= 1 and (forced > 0 or block_bytes(g, spec, batch, nzs, nvc) <= budget):
            options.append((int(nzs), ranges))
    if forced > 0 and options:
        return options[0]
    # whole volume with chunks of >= 32 views (the back kernel sets up 32 views
    # per pass); then the largest chunks that leave room for some slabs
    for nzs, ranges in options:
        if nzs == nz and (len(ranges) == 1 or ranges[0][1] - ranges[0][0] >= 32):
            return nzs, ranges
    if options:
        return options[0]
    raise CudaRuntimeError(
        f"cannot stream within {budget / 2**30:.2f} GiB: one z-slice ({slice_bytes} B) and one view "
        f"({view_bytes} B) per block need {block_bytes(g, spec, batch, 1, 1)} B")


def taper(ranges, direction: int, first: int = 32):
    """Split the chunk whose transfer is exposed -- the back projection's
    first upload (direction 1), the forward projection's last download (0) --
    so that only ``first`` views' worth of it waits: [a, e) -> [a, a + first),
    [a + first, e) (mirrored for the forward) when e - a >= 2 first.  The rest
    of the split chunk moves while the small one computes (a view transfers
    several times faster than it projects)."""
    rs = list(ranges)
    if len(rs) < 2:
        return rs
    if direction == 1:
        a, e = rs[0]
        return [(a, a + first), (a + first, e)] + rs[1:] if e - a >= 2 * first else rs
    a, e = rs[-1]
    return rs[:-1] + [(a, e - first), (e - first, e)] if e - a >= 2 * first else rs


def _flat(buf, shape):
    """Contiguous view of the first prod(shape) elements of a flat buffer."""
    n = 1
    for s in shape:
        n *= int(s)
    return buf[:n].view(shape)


def stream_apply(plan: "_native.Plan", host, direction: int, nzs: int | None = None, ranges=None):
    """Apply A (direction 0) / A^T (1) of ``plan`` to a host f32 tensor
    [B, ...] block by block (z-slabs of ``nzs`` slices x view ``ranges``);
    returns a pinned host tensor."""
    torch = _torch()
    dev = plan.device
    g, spec = plan.geometry, plan.spec
    B = int(host.shape[0])
    nz, ny, nx = spec.shape
    nv, nr, nc = g.shape
    if nzs is None or ranges is None:
        nzs0, ranges0 = plan_blocks(g, spec, B, device_budget(dev), direction)
        nzs = nzs0 if nzs is None else nzs
        ranges = ranges0 if ranges is None else ranges
    zr = zslab_ranges(nz, min(nzs, nz))
    if len(zr) == 1:
        ranges = taper(ranges, direction)
    one_slab, one_chunk = len(zr) == 1, len(ranges) == 1
    plans = {}

    def sub(zi, vi):
        key = (zi, vi)
        if key not in plans:
            if one_slab and one_chunk:
                plans[key] = plan
            else:
                (z0, z1), (a, e) = zr[zi], ranges[vi]
                gg = g if one_chunk else g.with_views(range(a, e))
                ss = spec if one_slab else slab_spec(spec, z0, z1 - z0)
                plans[key] = _native.get_plan(gg, ss, dev.index)
        return plans[key]

    compute = torch.cuda.current_stream(dev)
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    src = host if host.is_pinned() else host.pin_memory()
    nzs_max = max(z1 - z0 for z0, z1 in zr)
    nvc_max = max(e - a for a, e in ranges)

    def upload(dst, zi_or_vi, slab):
        """dst (device) <- the host block; per batch element when strided."""
        with torch.cuda.stream(h2d):
            if slab:
                z0, z1 = zr[zi_or_vi]
                part = src if one_slab else src[:, z0:z1]
            else:
                a, e = ranges[zi_or_vi]
                part = src if one_chunk else src[:, a:e]
            if B == 1 or part.is_contiguous():
                dst.copy_(part, non_blocking=True)
            else:
                for b in range(B):
                    dst[b].copy_(part[b], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(h2d)
        compute.wait_event(ev)

    def download(out, block, sl, after=None):
        ev = torch.cuda.Event()
        ev.record(compute if after is None else after)
        d2h.wait_event(ev)
        with torch.cuda.stream(d2h):
            dst = out if sl is None else out[:, sl[0]:sl[1]]
            if B == 1 or dst.is_contiguous():
                dst.copy_(block, non_blocking=True)
            else:
                for b in range(B):
                    dst[b].copy_(block[b], non_blocking=True)
        done = torch.cuda.Event()
        done.record(d2h)
        return done

    with torch.cuda.device(dev):
        if direction == 0:
            out = torch.empty((B, nv, nr, nc), dtype=torch.float32, pin_memory=True)
            yring = [torch.empty(B * nvc_max * nr * nc, dtype=torch.float32, device=dev) for _ in range(2)]
            y_free = [None, None]  # download that last read the slot
            # with the whole volume resident, consecutive view chunks run on
            # alternating compute streams: their outputs are disjoint and the
            # volume is read-only, so one chunk's launch tails overlap the
            # next chunk's start (FWD_STREAMS = 1: one stream)
            cstreams = [compute]
            if one_slab:
                xd = torch.empty((B, nz, ny, nx), dtype=torch.float32, device=dev)
                upload(xd, 0, True)
                if FWD_STREAMS > 1 and len(ranges) > 1:
                    # one persistent stream per device: the caching allocator
                    # keeps freed blocks per stream, so a fresh stream per call
                    # would re-allocate the chunks' workspaces every call
                    if dev.index not in _FWD_STREAM:
                        _FWD_STREAM[dev.index] = torch.cuda.Stream(dev)
                    cstreams.append(_FWD_STREAM[dev.index])
                    cstreams[1].wait_stream(compute)
            else:
                xring = [torch.empty(B * nzs_max * ny * nx, dtype=torch.float32, device=dev) for _ in range(2)]
                x_free = [None, None]  # kernel that last read the slot
            step = 0
            for vi, (a, e) in enumerate(ranges):
                k = vi % 2
                cs = cstreams[vi % len(cstreams)]
                ys = _flat(yring[k], (B, e - a, nr, nc))
                if y_free[k] is not None:
                    cs.wait_event(y_free[k])
                for zi, (z0, z1) in enumerate(zr):
                    if one_slab:
                        xs = xd
                    else:
                        s = step % 2
                        if x_free[s] is not None:
                            h2d.wait_event(x_free[s])
                        xs = _flat(xring[s], (B, z1 - z0, ny, nx))
                        upload(xs, zi, True)
                    if cs is compute:
                        sub(zi, vi).forward(xs, out=ys, accumulate=zi > 0)
                    else:
                        with torch.cuda.stream(cs):
                            sub(zi, vi).forward(xs, out=ys, accumulate=zi > 0)
                    if not one_slab:
                        x_free[s] = torch.cuda.Event()
                        x_free[s].record(compute)
                        step += 1
                y_free[k] = download(out, ys, None if one_chunk else (a, e), after=cs)
            for cs in cstreams[1:]:
                compute.wait_stream(cs)
            compute.wait_stream(d2h)
            compute.synchronize()
            return out
        out = torch.empty((B, nz, ny, nx), dtype=torch.float32, pin_memory=True)
        xring = [torch.empty(B * nzs_max * ny * nx, dtype=torch.float32, device=dev) for _ in range(2)]
        x_free = [None, None]
        if one_chunk:
            yd = torch.empty((B, nv, nr, nc), dtype=torch.float32, device=dev)
            upload(yd, 0, False)
        else:
            yring = [torch.empty(B * nvc_max * nr * nc, dtype=torch.float32, device=dev) for _ in range(2)]
            y_free = [None, None]
        step = 0
        for zi, (z0, z1) in enumerate(zr):
            k = zi % 2
            xs = _flat(xring[k], (B, z1 - z0, ny, nx))
            if x_free[k] is not None:
                compute.wait_event(x_free[k])
            for vi, (a, e) in enumerate(ranges):
                if one_chunk:
                    ys = yd
                else:
                    s = step % 2
                    if y_free[s] is not None:
                        h2d.wait_event(y_free[s])
                    ys = _flat(yring[s], (B, e - a, nr, nc))
                    upload(ys, vi, False)
                sub(zi, vi).back(ys, out=xs, accumulate=vi > 0)
                if not one_chunk:
                    y_free[s] = torch.cuda.Event()
                    y_free[s].record(compute)
                    step += 1
            x_free[k] = download(out, xs, None if one_slab else (z0, z1))
        compute.wait_stream(d2h)
        compute.synchronize()
        return out


def host_apply(plan: "_native.Plan", host, direction: int, chunk_bytes: int | None = None):
    """Whole volume resident, views in chunks of about ``chunk_bytes``
    (default: CHUNK_BYTES, or more so there are at most MAX_CHUNKS)."""
    B = int(host.shape[0])
    nv, nr, nc = plan.sino_shape
    view_bytes = B * nr * nc * 4
    if chunk_bytes is None:
        chunk_bytes = max(CHUNK_BYTES, math.ceil(nv * view_bytes / MAX_CHUNKS))
    return stream_apply(plan, host, direction, plan.spec.numZ, view_chunks(nv, view_bytes, chunk_bytes))


def zslab_apply(plan: "_native.Plan", host, direction: int, nzs: int):
    """z-slabs of ``nzs`` slices, views in the default chunks."""
    B = int(host.shape[0])
    nv, nr, nc = plan.sino_shape
    view_bytes = B * nr * nc * 4
    chunk_bytes = max(CHUNK_BYTES, math.ceil(nv * view_bytes / MAX_CHUNKS))
    return stream_apply(plan, host, direction, nzs, view_chunks(nv, view_bytes, chunk_bytes))
