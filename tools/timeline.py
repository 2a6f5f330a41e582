#!/usr/bin/env python
"""GPU timeline of one decomposition (CUPTI kernel records through torch.profiler):
per-step busy time, idle gaps between kernels and the kernels on either side of the
largest gaps.  Diagnostics only (no bench number comes from a profiled run).

    python tools/timeline.py --config c3 [--steps 2] [--warmup 3] [--top 25] [--json out.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--json", default=None)
    ap.add_argument("--list", default=None, help="write the last step's records (start µs, duration µs, name) here")
    args = ap.parse_args()

    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_1703_06065_b200 import bcur as B
    from paper_1703_06065_b200.configs import CONFIGS, spectrum

    cfg = CONFIGS[args.config]
    ctx = B.Context(0)
    m, n, s = cfg["m"], cfg["n"], cfg["s"]
    dt = np.float32 if cfg["dtype"] == "f32" else np.float64
    if cfg["kind"] == "lowrank":
        dm = B.DeviceMatrix.generate("lowrank", dt, m, n, seed=cfg["seed"], sigma=spectrum(cfg["spectrum"], cfg["rank"]),
                                     noise=cfg["noise"], ctx=ctx)
    else:
        dm = B.DeviceMatrix.generate("biometric", dt, m, n, seed=cfg["seed"], ctx=ctx)
    part = B.BlockPartition.equal_blocks(n, s)
    rpart = B.BlockPartition.equal_blocks(m, s)
    for _ in range(args.warmup):
        bench.run_step(B, cfg, dm, part, rpart, ctx)
    ctx.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(args.steps):
            bench.run_step(B, cfg, dm, part, rpart, ctx)
        ctx.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev), key=lambda t: t[0])
    if not ks:
        print("no device records")
        return
    span = ks[-1][1] - ks[0][0]
    busy, gaps = 0.0, []
    cur_s, cur_e, prev = ks[0][0], ks[0][1], ks[0][2]
    for s0, e0, nm in ks[1:]:
        if s0 > cur_e:
            busy += cur_e - cur_s
            gaps.append((s0 - cur_e, prev, nm))
            cur_s = s0
        if e0 > cur_e:
            cur_e, prev = e0, nm
    busy += cur_e - cur_s
    gaps.sort(reverse=True)
    per = args.steps
    out = {"config": args.config, "steps": per, "records": len(ks) / per, "span_ms": span / 1e3 / per,
           "busy_ms": busy / 1e3 / per, "idle_ms": (span - busy) / 1e3 / per,
           "gaps_over_5us": sum(1 for g in gaps if g[0] > 5) / per,
           "top_gaps_us": [(round(g, 1), a[:70], b[:70]) for g, a, b in gaps[: args.top]]}
    print(json.dumps({k: v for k, v in out.items() if k != "top_gaps_us"}))
    for g, a, b in out["top_gaps_us"]:
        print(f"{g:9.1f} us  after {a}\n              before {b}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)
    if args.list:
        # the last step: from its norms pass (the first k_block_sumsq after the midpoint) on
        starts = [i for i, k in enumerate(ks) if "k_block_sumsq" in k[2]]
        i0 = starts[-1] if starts else 0
        t0 = ks[i0][0]
        with open(args.list, "w") as f:
            for s0, e0, nm in ks[i0:]:
                f.write(f"{s0 - t0:10.1f} {e0 - s0:9.1f}  {nm[:140]}\n")


if __name__ == "__main__":
    main()
