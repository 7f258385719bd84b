"""A/B probe of the 3D SF kernels: kernel time (library CUDA events) and an
output digest for one config; run it twice (e.g. with CTP_BACK_LEGACY=1) and
compare the saved outputs with --compare.

    python tools/ab_probe.py --config c3 --tag new --out gpurun_out/ab
    CTP_BACK_LEGACY=1 python tools/ab_probe.py --config c3 --tag old --out gpurun_out/ab
    python tools/ab_probe.py --compare gpurun_out/ab/new.npz gpurun_out/ab/old.npz
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--tag", default="run")
    ap.add_argument("--out", default="gpurun_out/ab")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dirs", default="fb")
    ap.add_argument("--compare", nargs=2)
    ap.add_argument("--views", type=int, default=0, help="override numAngles (same angular range)")
    a = ap.parse_args()
    import numpy as np
    if a.compare:
        p, q = np.load(a.compare[0]), np.load(a.compare[1])
        res = {}
        for k in sorted(set(p.files) & set(q.files)):
            x, y = p[k].astype(np.float64), q[k].astype(np.float64)
            res[k] = dict(rel_l2=float(np.linalg.norm(x - y) / np.linalg.norm(y)),
                          max_abs_rel=float(np.abs(x - y).max() / np.abs(y).max()))
        print(json.dumps(res))
        return
    import torch
    import paper_2307_05801_b200 as ct
    from bench import CONFIGS
    cfg = dict(CONFIGS[a.config])
    if a.views:
        cfg["numAngles"] = a.views
    g, spec = ct.parse_config(json.dumps(cfg))
    P = ct.ProjectorPair(ct.SF, g, spec)
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(0)
    x = torch.rand((1,) + spec.shape, device=dev, generator=gen)
    y = torch.rand((1,) + g.shape, device=dev, generator=gen)
    plan = P.plan(0)
    res = {"config": a.config, "tag": a.tag}
    outs = {}
    for d, name, inp, fn in (("f", "fwd", x, plan.forward), ("b", "back", y, plan.back)):
        if d not in a.dirs:
            continue
        o = fn(inp, time_kernel=True)
        torch.cuda.synchronize()
        ms = []
        for _ in range(a.reps):
            fn(inp, out=o, time_kernel=True)
            torch.cuda.synchronize()
            ms.append(plan.kernel_time_ms(0 if d == "f" else 1))
        res[name + "_ms"] = ms
        res[name + "_ms_min"] = min(ms)
        nup = spec.shape[0] * spec.shape[1] * spec.shape[2] * g.shape[0]
        res[name + "_gups"] = nup / min(ms) / 1e6
        o64 = o.double()
        res[name + "_sum"] = float(o64.sum())
        # a strided sample of the output for --compare
        flat = o.reshape(-1)
        idx = torch.arange(0, flat.numel(), 997, device=dev)
        outs[name] = flat[idx].cpu().numpy()
    os.makedirs(a.out, exist_ok=True)
    np.savez(os.path.join(a.out, a.tag + ".npz"), **outs)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
