#!/usr/bin/env python
"""bench.py -- fwd+back SF projector GUPS (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Workload (BASELINE.json configs[2], the metric's config): cone-beam flat
panel, 512^3 voxels of 0.6667 mm, 720 views over 360 deg, 768^2 detector of
1.0 mm, sod 1000 / sdd 1500 mm; U[0,1) f32 volume (PCG64 seed 0) and
sinogram (seed 1), synthetic.  One step = one SF forward projection of the
whole volume + one SF back projection of a whole sinogram (what an autograd
forward+backward of ``Projector`` costs).

    GUPS = 2 * nx*ny*nz * nv / t_step / 1e9     (voxel-view updates per second)

N > 1: one process per GPU.  Without a torchrun environment, ``--gpus N``
re-launches itself under ``python -m torch.distributed.run --nproc-per-node N``
(127.0.0.1, a free port, NCCL_DEBUG=INFO so the N-rank communicator shows in
the log); with one it checks WORLD_SIZE == N.  Views are sharded over ranks;
the forward has no communication, the back projection is fused with per-z-
chunk NCCL reductions to the z-slab owners (csrc/dist.cu, overlapped with the
remaining back projection).  Total work is fixed, so "scaling" is "strong";
time = max over ranks; per-rank times and the exposed reduction time are
reported under "dist".

Inputs (512 MiB volume, 1.58 GiB sinogram) exceed the 126 MB L2, so no L2
flush is needed between timed iterations.  ``--impl reference`` times the
reference algorithm on the host cores (the C restatement in oracle/, as the
reference itself is Python/numba and cannot travel to the GPU box).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c3": dict(geometry="cone", numX=512, numY=512, numZ=512, voxelWidth=0.6667,
               voxelHeight=0.6667, numRows=768, numCols=768, pixelHeight=1.0, pixelWidth=1.0,
               sod=1000.0, sdd=1500.0, numAngles=720, angularRange=360.0),
    "c2": dict(geometry="cone", numX=512, numY=512, numZ=1, voxelWidth=0.6667,
               voxelHeight=1.0, numRows=1, numCols=768, pixelHeight=1.0, pixelWidth=1.0,
               sod=1000.0, sdd=1500.0, numAngles=720, angularRange=360.0),
    "c5": dict(geometry="cone", numX=1024, numY=1024, numZ=1024, voxelWidth=0.3333,
               voxelHeight=0.3333, numRows=1536, numCols=1536, pixelHeight=0.5, pixelWidth=0.5,
               sod=1000.0, sdd=1500.0, numAngles=1440, angularRange=360.0),
    "c1": dict(geometry="parallel", numX=128, numY=128, numZ=128, voxelWidth=1.0,
               voxelHeight=1.0, numRows=128, numCols=128, pixelHeight=1.0, pixelWidth=1.0,
               numAngles=180, angularRange=180.0),
}
WORKLOAD_NAME = {
    "c3": "cone-beam flat 512^3 x 720 views, 768^2 det, fwd+back (BASELINE configs[2])",
    "c1": "parallel-beam 128^3 x 180 views, 128^2 det, fwd+back (BASELINE configs[0])",
    "c2": "fan-beam (cone-flat, 1 row, 1 slice) 512^2 x batch 64 x 720 views, 768 cols (BASELINE configs[1])",
    "c5": "cone-beam flat 1024^3 x 1440 views, 1536^2 det, fwd+back (BASELINE configs[4])",
}
METRIC = "fwd+back projector GUPS, cone-beam 512³ × 720 views"
METRICS = {"c3": METRIC, "c1": "fwd+back projector GUPS, parallel-beam 128³ × 180 views",
           "c2": "fwd+back projector GUPS, fan-beam 512² × batch 64 × 720 views",
           "c5": "fwd+back projector GUPS, cone-beam 1024³ × 1440 views"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, device_index: int, period: float = 0.1):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            pass
        self._period = period
        self._t = threading.Thread(target=self._run, daemon=True)

    _REASONS = {
        0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    }

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self._REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self._period)

    def __enter__(self):
        if self._ok:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_sample(cfg: dict, budget_s: float = 20.0):
    """Time the CPU oracle (reference algorithm, all host threads) on a bounded
    view subset of cfg; returns (GUPS, threads, description)."""
    import numpy as np

    from oracle import oracle

    oracle.build()
    threads = oracle.max_threads()
    shape_v, shape_s = oracle.shapes(cfg)
    nv = shape_s[0]
    nvox = int(np.prod(shape_v))
    x = np.random.default_rng(0).random(shape_v, dtype=np.float32)
    # probe one view, then size the sample to the budget
    one = oracle.with_views(cfg, [0])
    t0 = time.perf_counter()
    oracle.sf_forward(one, x)
    y1 = np.random.default_rng(1).random((1,) + tuple(shape_s[1:]), dtype=np.float32)
    oracle.sf_back(one, y1)
    t1 = time.perf_counter() - t0
    # the reference forward parallelises over views (prange, _kernels.py:655): use a
    # multiple of the thread count so every core works, as in the full workload
    k = int(max(1, budget_s * threads / max(t1, 1e-3)))
    k = max(threads, (k // threads) * threads)
    k = min(nv, k)
    idx = [int(round(i * nv / k)) % nv for i in range(k)]
    sub = oracle.with_views(cfg, idx)
    y = np.random.default_rng(1).random((k,) + tuple(shape_s[1:]), dtype=np.float32)
    t0 = time.perf_counter()
    oracle.sf_forward(sub, x)
    tf = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.sf_back(sub, y)
    tb = time.perf_counter() - t0
    gups = 2.0 * nvox * k / (tf + tb) / 1e9
    desc = (f"{k} of {nv} views (evenly spaced) of the same geometry, full volume, fwd "
            f"{tf:.2f}s + back {tb:.2f}s; f64 C restatement (oracle/sf_oracle.c), OpenMP")
    return gups, threads, desc


def run_reference(args, cfg):
    world, rank, local = _dist_env()
    if rank != 0:
        return
    import numpy as np

    from oracle import oracle

    oracle.build()
    threads = oracle.max_threads()
    shape_v, shape_s = oracle.shapes(cfg)
    nv = shape_s[0]
    nvox = int(np.prod(shape_v))
    x = np.random.default_rng(0).random(shape_v, dtype=np.float32)
    # one view per host thread per step: the reference forward parallelises over
    # views (_kernels.py:655) and the back over voxel columns (_kernels.py:676)
    views_per_step = max(1, int(os.environ.get("BENCH_REF_VIEWS", str(threads))))
    y = np.random.default_rng(1).random((views_per_step,) + tuple(shape_s[1:]), dtype=np.float32)
    times = []
    for step in range(args.warmup + args.steps):
        idx = [((step * 97) + i * (nv // views_per_step)) % nv for i in range(views_per_step)]
        sub = oracle.with_views(cfg, idx)
        t0 = time.perf_counter()
        oracle.sf_forward(sub, x)
        oracle.sf_back(sub, y)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    t = sum(times)
    value = 2.0 * nvox * views_per_step * len(times) / t / 1e9
    sample = (f"each step = fwd+back of {views_per_step} of {nv} views (full 512^3 volume), "
              "f64 C restatement of the reference kernels (oracle/sf_oracle.c), OpenMP over "
              "host cores; the reference itself is Python/numba and does not travel to the box")
    line = {
        "impl": "reference", "metric": METRICS[args.config], "value": value, "unit": "GUPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * t / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic U[0,1) (PCG64 seeds 0/1)",
        "config": {"workload": WORKLOAD_NAME[args.config], "sample": "view subset per step"},
        "cpu_baseline": {"value": value, "unit": "GUPS", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def _spawn_or_check(args):
    """--gpus N > 1 outside torchrun: re-run this command under torchrun with N
    local ranks; inside torchrun: WORLD_SIZE must equal N."""
    if args.impl == "reference":
        return  # rank 0 alone runs the host baseline; no ranks needed
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        import socket
        import subprocess

        import torch

        n = torch.cuda.device_count()
        if n < args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but only {n} CUDA device(s) visible"}), flush=True)
            raise SystemExit(2)
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd, env=env))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch with --nproc-per-node {args.gpus}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=15)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--batch", type=int, default=0, help="batch size (default: 64 for c2, else 1)")
    ap.add_argument("--views", type=int, default=0,
                    help="profiling only: restrict to the first N views (not a bench number)")
    args = ap.parse_args()
    _spawn_or_check(args)
    cfg = dict(CONFIGS[args.config])
    if args.views:
        cfg["numAngles"] = args.views
        cfg["angularRange"] = cfg["angularRange"] * args.views / CONFIGS[args.config]["numAngles"]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2307_05801_b200 as ct
    from paper_2307_05801_b200 import partition

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    g, spec = ct.parse_config(json.dumps(cfg))
    P = ct.ProjectorPair(ct.SF, g, spec)
    sharded = partition.ViewShardedProjector(P, rank, world, device=dev)
    a, b = sharded.views
    nv_local = b - a
    nvox = spec.num_voxels
    nr, nc = g.detector.numRows, g.detector.numCols

    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    B = args.batch or (64 if args.config == "c2" else 1)
    x = torch.rand((B,) + spec.shape, device=dev, generator=gen)
    gen.manual_seed(1 + rank)
    y = torch.rand((B, nv_local, nr, nc), device=dev, generator=gen)
    plan = sharded.shard.plan(local)
    sino_out = torch.empty((B, nv_local, nr, nc), device=dev)

    slab_out = None
    if world > 1:
        slab_out = torch.empty((B, sharded.slab) + spec.shape[1:], device=dev)

    def step(time_kernel=False):
        plan.forward(x, out=sino_out, time_kernel=time_kernel)
        if world == 1:
            return plan.back(y, time_kernel=time_kernel)
        # fused back projection + per-z-chunk NCCL reductions (csrc/dist.cu)
        return sharded.back_native(y, out=slab_out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    fwd_ms, back_ms = [], []
    stream = torch.cuda.current_stream(dev)
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eb = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        for i in range(args.steps):
            plan.forward(x, out=sino_out, time_kernel=True)
            eb[i][0].record(stream)
            if world == 1:
                plan.back(y, time_kernel=True)
            else:
                sharded.back_native(y, out=slab_out)
            eb[i][1].record(stream)
            fwd_ms.append(plan.kernel_time_ms(0))
            if world == 1:
                back_ms.append(plan.kernel_time_ms(1))
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    t_ms = e0.elapsed_time(e1)
    t_max = t_ms
    dist_info = None
    if world > 1:
        tt = torch.tensor([t_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
        fused_ms = statistics.mean(a.elapsed_time(b) for a, b in eb)
        # the same back projection without the reductions (untimed): what the
        # fused call's communication adds on the critical path
        part = torch.empty((B,) + spec.shape, device=dev)
        for _ in range(args.steps):
            plan.back(y, out=part, time_kernel=True)
            back_ms.append(plan.kernel_time_ms(1))
        per_rank = [None] * world
        dist.all_gather_object(per_rank, {"rank": rank, "step_ms": t_ms / args.steps, "views": [a, b],
                                          "fwd_kernel_ms": statistics.mean(fwd_ms),
                                          "back_fused_ms": fused_ms,
                                          "back_kernel_ms": statistics.mean(back_ms)})
        dist_info = {"ranks": per_rank,
                     "reduce_exposed_ms": max(r["back_fused_ms"] - r["back_kernel_ms"] for r in per_rank),
                     "reduce_bytes_per_rank": 4 * B * nvox,
                     "collective": "ncclReduce per (z-chunk of 256 slices, owner), grouped, on a comm stream"}
    total_updates = 2.0 * B * nvox * g.numViews * args.steps
    value = total_updates / (t_max / 1e3) / 1e9

    # roofline of the dominant kernel: algorithmic bytes per
    # launch = 4 B per voxel-view update + 4 B per output element
    peak, peak_kind = _peaks()
    f_ms, b_ms = statistics.mean(fwd_ms), statistics.mean(back_ms)
    upd = B * nvox * nv_local
    # the kernels that ran (csrc/sf_forward3d.cu, csrc/sf_back3d.cu; the round-1
    # per-row kernels of csrc/sf_kernels.cu only under CTP_*_LEGACY)
    fname = "sf_forward_kernel" if os.environ.get("CTP_FWD_LEGACY") else "sf_forward3d_kernel"
    bname = "sf_back_kernel" if os.environ.get("CTP_BACK_LEGACY") else "sf_back3d_kernel"
    kern = {
        fname: {"ms": f_ms, "bytes": 4.0 * upd + 4.0 * B * nv_local * nr * nc},
        bname: {"ms": b_ms, "bytes": 4.0 * upd + 4.0 * B * nvox},
    }
    for k in kern.values():
        k["gbs"] = k["bytes"] / (k["ms"] / 1e3) / 1e9
        k["frac"] = k["gbs"] / peak
        k["gups"] = upd / (k["ms"] / 1e3) / 1e9
    dom = max(kern, key=lambda n: kern[n]["ms"])
    traffic = None
    prof = {}
    try:
        # DRAM bytes per launch, warp instructions per update and issue activity
        # from the committed `ncu --set full` capture of the same kernel on C3
        # (tools/summarize_profiles.py; a view subset is scaled to all views)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            prof = json.load(f)
        t = prof.get(dom)
        if t and args.config == "c3" and B == 1 and world == 1:
            traffic = t["dram_bytes_per_launch"]
    except Exception:
        pass
    for k, v in kern.items():
        t = prof.get(k) if args.config == "c3" and B == 1 else None
        if t and "inst_per_update" in t:
            v["inst_per_update"] = t["inst_per_update"]
            v["issue_active"] = t["issue_active"]

    # e2e: public API with host (pinned) buffers, H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        yh = y.cpu().pin_memory()
        shard_pair = sharded.shard
        # warm: plans, and the pinned-output pool in its steady state (a loop
        # holds the previous step's results while the next step allocates)
        for _ in range(3):
            yo = ct.forward(shard_pair, xh)
            xo = ct.adjoint(shard_pair, yh)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        calls = []
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            ta = time.perf_counter()
            yo = ct.forward(shard_pair, xh)       # host in -> host out
            tb = time.perf_counter()
            xo = ct.adjoint(shard_pair, yh)       # host in -> host out (partial volume)
            calls.append([round((tb - ta) * 1e3, 1), round((time.perf_counter() - tb) * 1e3, 1)])
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([te], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        # the value is the median step's rate (robust to a one-off host stall, e.g. a
        # pinned-pool refill); the mean over all timed steps is reported beside it
        step_s = sorted((a + b) / 1e3 for a, b in calls)
        med = step_s[len(step_s) // 2]
        if world > 1:
            tm = torch.tensor([med], device=dev)
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            med = float(tm.item())
        e2e = {"value": 2.0 * B * nvox * g.numViews / med / 1e9, "unit": "GUPS",
               "value_mean": 2.0 * B * nvox * g.numViews * args.e2e_steps / te / 1e9,
               "h2d_bytes_per_step": int(xh.numel() * 4 + yh.numel() * 4),
               "d2h_bytes_per_step": int(yo.numel() * 4 + xo.numel() * 4),
               "steps": args.e2e_steps, "calls_ms": calls,
               "path": "paper_2307_05801_b200.forward/adjoint on pinned host tensors "
                       "(view-chunked H2D/compute/D2H overlap)"}
        if world > 1:
            e2e["note"] = "per-rank view shard through the public API; back returns the partial volume"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        gups, threads, desc = cpu_sample(cfg)
        cpu = {"value": gups, "unit": "GUPS", "cores": threads, "kind": "port", "sample": desc}

    if rank == 0:
        line = {
            "metric": METRICS[args.config], "value": value, "unit": "GUPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic U[0,1) f32 (seeded)",
            "config": {"workload": WORKLOAD_NAME[args.config],
                       "parallelism": f"views sharded x{world}" + (" + NCCL reduce-scatter" if world > 1 else ""),
                       "l2": "inputs (0.5 GiB volume, 1.58 GiB sinogram) exceed L2; no flush",
                       "voxels": list(spec.shape), "views": g.numViews, "detector": [nr, nc],
                       "batch": B},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["gbs"], "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": kern[dom]["frac"],
                         "traffic": traffic,
                         "algorithmic_bytes_per_launch": kern[dom]["bytes"],
                         "launch_ms": kern[dom]["ms"],
                         # the kernels are issue-bound, not HBM-bound:
                         # ncu warp instructions per voxel-view update and issue-slot activity
                         "inst_per_update": kern[dom].get("inst_per_update"),
                         "issue_active": kern[dom].get("issue_active"),
                         "profile": prof.get(dom, {}).get("capture")},
            "kernels": {k: {kk: round(vv, 4) for kk, vv in v.items()} for k, v in kern.items()},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks.summary(),
            "gpu_launches": 4 * args.steps if world == 1 else (2 + 1 + -(-spec.numZ // 256)) * args.steps,
        }
        if dist_info is not None:
            line["dist"] = dist_info
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
