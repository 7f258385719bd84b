"""Multi-GPU path on the device: the fused back projection + per-z-chunk NCCL
reductions (ctp_sf_back_sharded, csrc/dist.cu) and the NCCL view sharding.

* world = 1 runs on any GPU box: a one-rank communicator turns every
  reduction into a copy, so the fused path must equal the plain back
  projection bit for bit (same kernel blocks, z-chunk by z-chunk);
* world = torch.cuda.device_count() > 1 spawns one NCCL process per GPU and
  compares the gathered z-slabs with the single-GPU back projection
  (skipped on one GPU).
"""

import json
import os
import socket

import numpy as np
import pytest
import torch

import paper_2307_05801_b200 as ct
from paper_2307_05801_b200 import errors, partition

from conftest import REARRANGE_TOL, rel_l2

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)
# 300 slices: two back z-chunks (256 + 44), tall enough for both forward bands
GEO = dict(geometry="cone", numX=40, numY=36, numZ=300, voxelWidth=0.6667, voxelHeight=0.6667,
           numRows=320, numCols=72, pixelHeight=1.0, pixelWidth=1.0, sod=1000.0, sdd=1500.0,
           numAngles=24, angularRange=360.0)


def _pair(cfg=GEO):
    g, spec = ct.parse_config(json.dumps(cfg))
    return ct.ProjectorPair(ct.SF, g, spec)


@pytest.mark.parametrize("batch", [1, 2])
def test_fused_back_world1_equals_back(batch):
    P = _pair()
    sh = partition.ViewShardedProjector(P, 0, 1, device=DEV)
    y = torch.rand((batch,) + P.geometry.shape, device=DEV, generator=torch.Generator(DEV).manual_seed(3))
    ref = P.plan(0).back(y)
    got = sh.back_native(y)
    torch.cuda.synchronize()
    assert got.shape == (batch,) + P.volumeSpec.shape
    assert torch.equal(got, ref)
    # repeated calls reuse the communicator and events and stay bitwise stable
    assert torch.equal(sh.back_native(y), ref)


def test_fused_back_rejects_bad_inputs():
    P = _pair()
    sh = partition.ViewShardedProjector(P, 0, 1, device=DEV)
    y = torch.rand((1,) + P.geometry.shape, device=DEV)
    with pytest.raises(errors.InvalidValueError):
        sh.back_native(y.double())
    with pytest.raises(ct.SpecMismatchError):
        sh.back_native(y[:, :5])


def _worker(rank, world, port, cfg, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    import torch.distributed as dist

    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    g, spec = ct.parse_config(json.dumps(cfg))
    P = ct.ProjectorPair(ct.SF, g, spec)
    sh = partition.ViewShardedProjector(P, rank, world, device=dev)
    assert sh.native
    a, b = sh.views
    gen = torch.Generator(dev).manual_seed(11)
    y = torch.rand((1,) + g.shape, device=dev, generator=gen)  # same full sinogram on every rank
    slab = sh.back(y[:, a:b].contiguous())
    q.put((rank, slab.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_view_sharded_back_matches_single_gpu():
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs for NCCL ranks (one process per GPU)")
    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, n, port, GEO, q)) for r in range(n)]
    for p in procs:
        p.start()
    slabs = dict(q.get(timeout=600) for _ in range(n))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    P = _pair()
    y = torch.rand((1,) + P.geometry.shape, device=DEV, generator=torch.Generator(DEV).manual_seed(11))
    ref = P.plan(0).back(y)[0].cpu().numpy()
    got = np.concatenate([slabs[r][0] for r in range(n)], axis=0)[: P.volumeSpec.numZ]
    assert rel_l2(got, ref) <= REARRANGE_TOL
