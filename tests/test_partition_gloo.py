"""Multi-rank partitioner (paper_2307_05801_b200/partition.py) on CPU.

Two processes over gloo on 127.0.0.1 run the SAME sharding code the NCCL
path runs, with the CPU oracle injected as the per-rank projector backend:
views are split across ranks, forward needs no communication, back ends with
the z-slab reduce-scatter (gloo: all-reduce + slice).  The gathered result
must equal the single-process projection.
"""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_05801_b200 import partition

CFG = dict(geometry="cone", numX=10, numY=9, numZ=7, voxelWidth=1.2, voxelHeight=1.1,
           numRows=9, numCols=14, pixelHeight=1.6, pixelWidth=1.5, sod=40.0, sdd=80.0,
           angles=[360.0 * i / 11 for i in range(11)])


class OracleBackend:
    """Per-rank backend computing with the CPU oracle (test-only)."""

    def __init__(self, cfg):
        from oracle import oracle

        self.o, self.cfg = oracle, cfg

    def forward(self, x, out=None):
        y = np.stack([self.o.sf_forward(self.cfg, xb.numpy()) for xb in x])
        return torch.from_numpy(y)

    def back(self, y, out=None):
        v = torch.from_numpy(np.stack([self.o.sf_back(self.cfg, yb.numpy()) for yb in y]))
        if out is not None:
            out.copy_(v)
            return out
        return v


def _shard_cfg(cfg, a, b):
    from oracle import oracle

    return oracle.with_views(cfg, list(range(a, b)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, x, y, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2307_05801_b200 as ct

        g, spec = ct.parse_config(json.dumps(cfg))
        P = ct.ProjectorPair(ct.SF, g, spec)
        ranges = partition.view_ranges(g.numViews, world)
        a, b = ranges[rank]
        sp = partition.ViewShardedProjector(P, rank, world,
                                            backend=OracleBackend(_shard_cfg(cfg, a, b)))
        yl = sp.forward(torch.from_numpy(x)[None])
        slab = sp.back(torch.from_numpy(y[a:b])[None].contiguous())
        full = sp.back_replicated(torch.from_numpy(y[a:b])[None].contiguous())
        q.put((rank, a, b, yl.numpy(), slab.numpy(), full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_view_sharded_pair_matches_single_process(world, oracle_mod):
    rng = np.random.default_rng(0)
    vshape, sshape = oracle_mod.shapes(CFG)
    x = rng.random(vshape, dtype=np.float32)
    y = rng.random(sshape, dtype=np.float32)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CFG, x, y, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_f = oracle_mod.sf_forward(CFG, x)
    ref_b = oracle_mod.sf_back(CFG, y)
    # forward: shards are disjoint view ranges, no communication -> bitwise
    fwd = np.concatenate([r[3][0] for r in res], axis=0)
    np.testing.assert_array_equal(fwd, ref_f)
    # back: reduce-scatter of per-rank partial volumes along z
    slabs = [torch.from_numpy(r[4]) for r in res]
    back = partition.gather_slabs(slabs, vshape[0]).numpy()[0]
    np.testing.assert_allclose(back, ref_b, rtol=2e-6, atol=2e-6 * np.abs(ref_b).max())
    for r in res:  # all-reduce variant: every rank holds the whole volume
        np.testing.assert_allclose(r[5][0], ref_b, rtol=2e-6, atol=2e-6 * np.abs(ref_b).max())


def test_view_ranges_balanced():
    assert partition.view_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert partition.view_ranges(720, 8)[-1] == (630, 720)
    assert partition.slab_size(512, 3) == 171
    with pytest.raises(ValueError):
        partition.view_ranges(4, 0)


def test_virtual_back_equals_sum_of_shards(oracle_mod):
    import paper_2307_05801_b200 as ct

    g, spec = ct.parse_config(json.dumps(CFG))
    P = ct.ProjectorPair(ct.SF, g, spec)
    y = torch.from_numpy(np.random.default_rng(3).random(g.shape, dtype=np.float32))[None]
    tot = partition.virtual_back(P, y, 4, lambda pair, a, b: OracleBackend(_shard_cfg(CFG, a, b)))
    ref = oracle_mod.sf_back(CFG, y[0].numpy())
    np.testing.assert_allclose(tot[0].numpy(), ref, rtol=2e-6, atol=2e-6 * np.abs(ref).max())


# ---- parallel beam: z-slab partitioning, no collective ---------------------
PCFG = dict(geometry="parallel", numX=9, numY=8, numZ=13, voxelWidth=1.1, voxelHeight=0.9,
            offsetZ=0.7, numRows=15, numCols=14, pixelHeight=1.0, pixelWidth=1.2,
            angles=[180.0 * i / 7 + 3.0 for i in range(7)])


def _pair_cfg(pair):
    from paper_2307_05801_b200 import geometry as geo

    return json.loads(geo.config_text(pair.geometry, pair.volumeSpec))


def _zslab_worker(rank, world, port, cfg, x, y, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2307_05801_b200 as ct

        g, spec = ct.parse_config(json.dumps(cfg))
        P = ct.ProjectorPair(ct.SF, g, spec)
        zp = partition.ZSlabParallelProjector(P, rank, world,
                                              backend_factory=lambda p: OracleBackend(_pair_cfg(p)))
        yl = zp.forward(torch.from_numpy(x)[None])
        xl = zp.back(torch.from_numpy(y)[None])
        dist.barrier()  # nothing is exchanged; the ranks only meet here
        q.put((rank, zp.rows, zp.slices, yl.numpy(), xl.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_zslab_parallel_pair_matches_single_process(world, oracle_mod):
    rng = np.random.default_rng(5)
    vshape, sshape = oracle_mod.shapes(PCFG)
    x = rng.random(vshape, dtype=np.float32)
    y = rng.random(sshape, dtype=np.float32)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_zslab_worker, args=(r, world, port, PCFG, x, y, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_f = oracle_mod.sf_forward(PCFG, x)
    ref_b = oracle_mod.sf_back(PCFG, y)
    # forward: each rank owns detector rows; concatenated along rows
    assert [r[1] for r in res] == partition.even_ranges(sshape[1], world)
    fwd = np.concatenate([r[3][0] for r in res], axis=1)
    np.testing.assert_allclose(fwd, ref_f, rtol=1e-9, atol=1e-9 * np.abs(ref_f).max())
    # back: each rank owns volume slices; concatenated along z
    back = np.concatenate([r[4][0] for r in res], axis=0)
    np.testing.assert_allclose(back, ref_b, rtol=1e-9, atol=1e-9 * np.abs(ref_b).max())


def test_zslab_ranges_cover_the_reach(oracle_mod):
    """Every slice a row receives from lies in that rank's slice range (and
    vice versa), checked against the oracle's own explicit matrix."""
    import paper_2307_05801_b200 as ct

    g, spec = ct.parse_config(json.dumps(PCFG))
    vshape, sshape = oracle_mod.shapes(PCFG)
    nz, nr = vshape[0], sshape[1]
    reach = np.zeros((nr, nz), dtype=bool)  # row r receives from slice iz
    for iz in range(nz):
        x = np.zeros(vshape, dtype=np.float32)
        x[iz] = 1.0
        reach[:, iz] = np.abs(oracle_mod.sf_forward(PCFG, x)).sum(axis=(0, 2)) > 0
    for world in (1, 2, 4, 5):
        for r0, r1 in partition.even_ranges(nr, world):
            a, b = partition.slices_of_rows(g, spec, r0, r1)
            assert not reach[r0:r1, :a].any() and not reach[r0:r1, b:].any()
        for z0, z1 in partition.even_ranges(nz, world):
            ra, rb = partition.rows_of_slices(g, spec, z0, z1)
            assert not reach[:ra, z0:z1].any() and not reach[rb:, z0:z1].any()


def test_zslab_rejects_cone():
    import paper_2307_05801_b200 as ct

    g, spec = ct.parse_config(json.dumps(CFG))
    with pytest.raises(ValueError):
        partition.ZSlabParallelProjector(ct.ProjectorPair(ct.SF, g, spec), 0, 2,
                                         backend_factory=lambda p: None)
