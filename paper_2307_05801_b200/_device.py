"""Device dispatch shared by sf.py / operator.py / the torch binding.

``run_batched`` applies A (direction 0) or A^T (direction 1) to a batch
through the cached ``_native.Plan``:

* CUDA tensor in  -> CUDA tensor out, on the input's device, stream-ordered
  on torch's current stream (no host synchronisation);
* CPU tensor / numpy in -> the same type out.  Inputs are staged through
  pinned memory and copied in view- or slice-chunks by ``Streamer``
  (chunked H2D / compute / D2H overlap, see chunking.py).

There is no CPU arithmetic path: a machine without a GPU gets a
``NativeLibraryError`` / ``CudaRuntimeError``, never silent CPU results.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import CudaRuntimeError, SpecMismatchError
from .geometry import Geometry, VolumeSpec


def _torch():
    import torch

    return torch


def default_device_index() -> int:
    torch = _torch()
    if not torch.cuda.is_available():
        raise CudaRuntimeError("no CUDA device is visible; this build has no CPU fallback")
    return torch.cuda.current_device()


def plan_for(g: Geometry, spec: VolumeSpec, device_index: int | None = None) -> "_native.Plan":
    if device_index is None:
        device_index = default_device_index()
    return _native.get_plan(g, spec, device_index)


def run_batched(g: Geometry, spec: VolumeSpec, batch, direction: int, out=None, model: str = "sf"):
    """Apply A / A^T of ``model`` ("sf" or "siddon") to ``batch``
    ([B, *in_shape]); returns [B, *out_shape]."""
    torch = _torch()
    in_shape = spec.shape if direction == 0 else g.shape
    if tuple(batch.shape[1:]) != tuple(in_shape):
        raise SpecMismatchError(f"batch must have shape (B, {', '.join(map(str, in_shape))}), "
                                f"got {tuple(batch.shape)}")
    if model == "siddon":
        return _run_siddon(g, spec, batch, direction, out)
    if isinstance(batch, torch.Tensor) and batch.is_cuda:
        plan = plan_for(g, spec, batch.device.index)
        x = batch if batch.dtype == torch.float32 else batch.to(torch.float32)
        x = x.contiguous()
        with torch.cuda.device(batch.device):
            return plan.forward(x, out=out) if direction == 0 else plan.back(x, out=out)
    # host input: numpy array or CPU tensor
    from .chunking import host_apply, zslab_apply

    plan = plan_for(g, spec)
    as_numpy = not isinstance(batch, torch.Tensor)
    host = torch.from_numpy(np.ascontiguousarray(batch, dtype=np.float32)) if as_numpy else batch
    host = host.to(torch.float32).contiguous()
    nzs = zslab_slices(g, spec, int(host.shape[0]), plan.device)
    if 0 < nzs < spec.numZ:
        res = zslab_apply(plan, host, direction, nzs)
    else:
        res = host_apply(plan, host, direction)
    return res.numpy() if as_numpy else res


def _run_siddon(g: Geometry, spec: VolumeSpec, batch, direction: int, out=None):
    """Siddon pair: CUDA tensors stay on the device; host arrays / CPU tensors
    go up through pinned memory, are projected in one launch, and come back
    as the same kind (no view chunking: this model is not the hot path)."""
    torch = _torch()
    if isinstance(batch, torch.Tensor) and batch.is_cuda:
        plan = plan_for(g, spec, batch.device.index)
        x = batch if batch.dtype == torch.float32 else batch.to(torch.float32)
        x = x.contiguous()
        with torch.cuda.device(batch.device):
            return plan.siddon_forward(x, out=out) if direction == 0 else plan.siddon_back(x, out=out)
    plan = plan_for(g, spec)
    as_numpy = not isinstance(batch, torch.Tensor)
    host = torch.from_numpy(np.ascontiguousarray(batch, dtype=np.float32)) if as_numpy else batch
    host = host.to(torch.float32).contiguous()
    with torch.cuda.device(plan.device):
        xd = host.pin_memory().to(plan.device, non_blocking=True)
        res = plan.siddon_forward(xd) if direction == 0 else plan.siddon_back(xd)
        res = res.cpu()
    return res.numpy() if as_numpy else res


def zslab_slices(g: Geometry, spec: VolumeSpec, batch: int, device) -> int:
    """z-slab size for host-resident calls: CTPROJ_ZSLAB if set, else 0 (no
    slabbing) when volume + sinogram + workspaces fit in 80% of the free
    device memory, else the largest slab that does (north_star item 3)."""
    import os

    torch = _torch()
    forced = int(os.environ.get("CTPROJ_ZSLAB", "0"))
    if forced > 0:
        return forced
    vol = 4 * batch * spec.num_voxels
    sino = 4 * batch * int(np.prod(g.shape))
    free = torch.cuda.mem_get_info(device)[0]
    budget = 0.8 * free
    if 2 * vol + 2 * sino <= budget:
        return 0
    per_slice = 2 * vol / spec.numZ
    room = budget - 2 * sino
    if room <= per_slice:
        raise CudaRuntimeError(
            f"sinogram of {sino / 2**30:.1f} GiB does not fit next to one z-slice on the device")
    return max(1, int(room // per_slice))
