#!/usr/bin/env python
"""The paper's roofline experiment (Fig. 5) on B200 -- SURVEY 8(f) N1.

Runs a workload with the paper's unfused decomposition (FD_OPT_KERNEL=3:
fd_pzz, [fd_pyy], fd_pxx, fd_time as separate kernels, plus add_source and the
receiver gather) and with the fused kernel, times every launch with CUDA
events (FD_OPT_PROFILE) and prints one roofline record per kernel:
arithmetic intensity (flops / cache-ideal bytes), achieved GFLOP/s, achieved
GB/s and the efficiency against the measured HBM roof (MEASURED_PEAKS.json,
the B200 analogue of the paper's BabelStream roof).

    python scripts/fig5_roofline.py C3:2 C3:8 C2:2 C2:8 [--steps 50] [--out profiles/fig5_r01.md]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def costs(ndim, r):
    """(flops, cache-ideal bytes) per grid point per kernel (fp32, FMA = 2 flops)."""
    d2 = (1 + 3 * r, 8.0)                       # c0*p, then r x (add + fma); read p, write D
    t = (2 * (ndim - 1) + 4, 4.0 * (4 + ndim))  # (ndim-1) adds + 2 fma; read p, pp, K, D*ndim, write
    fused = (ndim * (3 * r + 2) + 3, 16.0)
    return {"fd_pxx": d2, "fd_pyy": d2, "fd_pzz": d2, "fd_time": t, "fused": fused}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("specs", nargs="+")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import paper_2311_05038_b200 as fd
    from workloads import config
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        src = "measured"
    except Exception:
        peak, src = 6650.0, "fallback"
    lines = ["# Fig. 5 on B200: per-kernel roofline of the paper's decomposition vs the fused kernel", "",
             f"HBM roof: {peak:.0f} GB/s ({src}, MEASURED_PEAKS.json copy bandwidth).  Bytes are the",
             "cache-ideal algorithmic bytes per point; time = CUDA events around each launch.", "",
             "| workload | order | kernel | AI flop/B | time/launch us | GB/s | GFLOP/s | eff. vs roof |",
             "|---|---|---|---|---|---|---|---|"]
    stream = torch.cuda.Stream()
    for spec in args.specs:
        name, order = spec.split(":")
        wl = config(name, order=int(order))
        vel = wl.vel()
        cst = costs(wl.ndim, wl.order // 2)
        step_bytes = {}
        for kernel in (3, 0):
            sim = fd.Simulation(vel, wl.h, wl.dt, wl.order, stream=stream.cuda_stream,
                                options={fd.FD_OPT_KERNEL: kernel, fd.FD_OPT_ASYNC: 1})
            for s in wl.sources:
                sim.add_source(s.idx, s.f, s.t0, s.amp)
            sim.set_receivers(wl.receivers)
            sim.step(5)
            stream.synchronize()
            fd.fd_set_option(sim.ctx, fd.FD_OPT_PROFILE, 1)
            sim.step(args.steps)
            kt = sim.kernel_times()
            spl = sim.info()["steps_per_launch"]
            sim.close()
            for k, (ms, n) in kt.items():
                if k not in cst:
                    continue
                fl, by = cst[k]
                if k == "fused" and spl == 2:      # temporal blocking: two steps, 20 B/pt per launch
                    fl, by = 2 * fl, 20.0
                t = ms / n / 1e3
                gbs = by * wl.npts / t / 1e9
                gfl = fl * wl.npts / t / 1e9
                kname = k if not (k == "fused" and spl == 2) else "fused (2 steps/launch)"
                rec = {"workload": name, "order": wl.order, "kernel": kname, "ai": fl / by, "us": t * 1e6,
                       "gbs": gbs, "gflops": gfl, "eff": gbs / peak, "launches": n}
                print(json.dumps(rec), flush=True)
                lines.append(f"| {name} | {wl.order} | {kname} | {fl / by:.2f} | {t * 1e6:.1f} | {gbs:.0f} | "
                             f"{gfl:.0f} | {gbs / peak:.1%} |")
                step_bytes.setdefault(kernel, 0.0)
                step_bytes[kernel] += t / (spl if k == "fused" else 1)     # time per step
        if 3 in step_bytes and 0 in step_bytes:
            lines.append(f"| {name} | {wl.order} | **time per step: unfused / fused** | | "
                         f"{step_bytes[3] * 1e6:.1f} / {step_bytes[0] * 1e6:.1f} | | | "
                         f"x{step_bytes[3] / step_bytes[0]:.2f} |")
    text = "\n".join(lines) + "\n"
    print(text)
    if args.out:
        open(args.out, "w").write(text)


if __name__ == "__main__":
    main()
