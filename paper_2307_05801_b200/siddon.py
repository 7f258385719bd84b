"""Siddon projector pair on B200 (pkg/src/ctproj/siddon.py).

Ray-driven exact line lengths: the forward integrates each detector pixel's
centre ray through the grid (merged plane crossings, each interval
attributed to the voxel holding its midpoint); the back projector gathers,
per voxel, the exact ray/box clip length times y over the rays inside the
voxel's corner-projection window.  Both run in float64 in the CUDA kernels
of ``csrc/siddon_kernels.cu`` through the C-ABI (``ctp_siddon_forward`` /
``ctp_siddon_back``), restating the reference's float64 arithmetic in the
same order; every geometry kind, modular included, is supported.
"""

from __future__ import annotations

from . import _device
from .datamodel import ProjectionSet, Volume
from .geometry import Geometry, VolumeSpec

MODEL = "siddon"


def siddon_forward(x: Volume, g: Geometry) -> ProjectionSet:
    """y[sample] = sum over hit voxels of length * value (siddon.py:18-23)."""
    y = _device.run_batched(g, x.spec, x.values[None], direction=0, model=MODEL)
    return ProjectionSet(g, y[0])


def siddon_backproject(y: ProjectionSet, spec: VolumeSpec) -> Volume:
    """Matched transpose of siddon_forward for the same geometry (siddon.py:26-31)."""
    x = _device.run_batched(y.geometry, spec, y.values[None], direction=1, model=MODEL)
    return Volume(spec, x[0])
