"""Where does the per-launch kernel time of bench.py's profile pass come from?

Times K steps of a workload four ways on one GPU (CUDA events on the
library's stream, after warm-up): CUDA-graph replay (bench's value pass),
plain launches without per-launch events, the profile pass (events around
every launch, bench's roofline pass), and graph replay again (clock/thermal
drift check).  Prints ms per launch for each.

    python scripts/launch_timing.py --config C3 --order 8 --steps 1000
"""
import argparse
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class Poll:
    """NVML every 50 ms: SM / memory clock, power, GPU / memory temperature, reasons."""

    def __init__(self):
        import pynvml as nv
        nv.nvmlInit()
        self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(0)
        self.rows, self.stop = [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)
        self.t.start()

    def run(self):
        nv, h = self.nv, self.h
        while not self.stop.wait(0.05):
            try:
                self.rows.append((time.time(), nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM),
                                  nv.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                  nv.nvmlDeviceGetTemperature(h, nv.NVML_TEMPERATURE_GPU),
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass

    def window(self, t0, t1):
        r = [x for x in self.rows if t0 <= x[0] <= t1]
        if not r:
            return {}
        med = lambda i: sorted(x[i] for x in r)[len(r) // 2]
        reasons = 0
        for x in r:
            reasons |= x[5]
        return {"n": len(r), "sm_mhz": med(1), "mem_mhz": med(2), "power_w_max": max(x[3] for x in r),
                "temp_c": max(x[4] for x in r), "reasons": hex(reasons)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--order", type=int, default=2)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--kplane", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2311_05038_b200 as fd
    from workloads import config

    wl = config(a.config, a.order)
    stream = torch.cuda.Stream()
    out = {}
    poll = Poll()

    def make(graph):
        opts = {fd.FD_OPT_ASYNC: 1, fd.FD_OPT_GRAPH: 1 if graph else 0}
        if a.kplane:
            opts[fd.FD_OPT_KPLANE] = 1
        sim = fd.Simulation(wl.vel(), wl.h, wl.dt, wl.order, stream=stream.cuda_stream, options=opts)
        for s in wl.sources:
            sim.add_source(s.idx, s.f, s.t0, s.amp)
        sim.set_receivers(wl.receivers)
        sim.step(10)
        sim.reserve(4 * a.steps)
        stream.synchronize()
        return sim

    def timed(sim, label, profile=False):
        if profile:
            fd.fd_set_option(sim.ctx, fd.FD_OPT_PROFILE, 1)
            sim.reset_kernel_times()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        l0 = sim.info()["kernel_launches"]
        w0 = time.time()
        e0.record(stream)
        sim.step(a.steps)
        e1.record(stream)
        e1.synchronize()
        w1 = time.time()
        n = sim.info()["kernel_launches"] - l0
        ms = e0.elapsed_time(e1)
        row = {"total_ms": ms, "launches": n, "ms_per_launch": ms / max(n, 1), **poll.window(w0, w1)}
        if profile:
            kt = sim.kernel_times()
            row["event_ms_per_launch"] = kt["fused"][0] / max(kt["fused"][1], 1)
            fd.fd_set_option(sim.ctx, fd.FD_OPT_PROFILE, 0)
        out[label] = row
        print(label, {k: round(v, 4) if isinstance(v, float) else v for k, v in row.items()}, flush=True)
        return row

    g = make(True)
    timed(g, "graph replay")
    p = make(False)
    timed(p, "plain launches")
    timed(p, "profile pass (events per launch)", profile=True)
    timed(g, "graph replay again")
    timed(g, "profile pass on the graph context", profile=True)
    for i in range(6):
        timed(g, f"graph replay, repeat {i}")
    time.sleep(3.0)
    timed(g, "graph replay after 3 s idle")
    g.close()
    p.close()


if __name__ == "__main__":
    main()
