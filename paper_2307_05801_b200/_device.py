"""Device dispatch shared by sf.py / operator.py / the torch binding.

``run_batched`` applies A (direction 0) or A^T (direction 1) to a batch
through the cached ``_native.Plan``:

* CUDA tensor in  -> CUDA tensor out, on the input's device, stream-ordered
  on torch's current stream (no host synchronisation);
* CPU tensor / numpy in -> the same type out.  Inputs are staged through
  pinned memory and streamed block by block (view chunks x z-slabs sized to
  the device budget, chunked H2D / compute / D2H overlap, see chunking.py),
  so neither the whole volume nor the whole sinogram has to fit on the GPU.

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
    from .chunking import device_budget, plan_blocks, stream_apply

    plan = plan_for(g, spec)
    as_numpy = not isinstance(batch, torch.Tensor)
    host = torch.from_numpy(np.ascontiguousarray(batch, dtype=np.float32)) if as_numpy else batch
    host = host.to(torch.float32).contiguous()
    nzs, ranges = plan_blocks(g, spec, int(host.shape[0]), device_budget(plan.device), direction)
    res = stream_apply(plan, host, direction, nzs, ranges)
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
