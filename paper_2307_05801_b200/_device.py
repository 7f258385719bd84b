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


def run_batched(g: Geometry, spec: VolumeSpec, batch, direction: int, out=None):
    """Apply A / A^T to ``batch`` ([B, *in_shape]); returns [B, *out_shape]."""
    torch = _torch()
    in_shape = spec.shape if direction == 0 else g.shape
    if tuple(batch.shape[1:]) != tuple(in_shape):
        raise SpecMismatchError(f"batch must have shape (B, {', '.join(map(str, in_shape))}), "
                                f"got {tuple(batch.shape)}")
    if isinstance(batch, torch.Tensor) and batch.is_cuda:
        plan = plan_for(g, spec, batch.device.index)
        x = batch if batch.dtype == torch.float32 else batch.to(torch.float32)
        x = x.contiguous()
        with torch.cuda.device(batch.device):
            return plan.forward(x, out=out) if direction == 0 else plan.back(x, out=out)
    # host input: numpy array or CPU tensor
    from .chunking import host_apply

    plan = plan_for(g, spec)
    as_numpy = not isinstance(batch, torch.Tensor)
    host = torch.from_numpy(np.ascontiguousarray(batch, dtype=np.float32)) if as_numpy else batch
    res = host_apply(plan, host.to(torch.float32).contiguous(), direction)
    return res.numpy() if as_numpy else res
