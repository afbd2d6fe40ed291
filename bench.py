#!/usr/bin/env python
"""Benchmark of the fused acoustic FD time step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--order 2]
                    [--impl ours|reference] [--no-cpu-baseline]

A "step" is one leapfrog time step of the whole hot path (source injection,
stencil with band rule, time update, receiver sampling -- all SURVEY.md 8(a)
rows) over the configured grid.  value = grid-point updates per second
(Gpts/s) over all ranks, timed with CUDA events on the stream the kernels run
on, W untimed warm-up steps first, max over ranks.  The per-step working set
(p, p_prev, K: 1.5 GiB for C3) is far larger than the 126 MB L2, so no flush
is needed between steps (stated in config).

Passes: (1) the value -- K steps replayed from CUDA graphs, CUDA events on
the library stream, NVML clocks sampled; the roofline's kernel time is this
region's time / step-kernel launches at N = 1; (2) K more steps with events
around every launch (per-kernel breakdown; the kernel time at N > 1);
(3, N = 1, --sustained S) ~S seconds of graph replay after everything else,
reported as `sustained` with clocks and power (the board's 1 kW cap engages
after ~0.3 s of full load; not the value).  e2e = three complete public-API
runs (model upload, K steps, traces and final field to pinned host memory),
median.  cpu_baseline = the fp64 oracle on a bounded sample, all host cores
and one.  Device memory comes from torch's caching allocator.

Options: --tsteps 1|2 (steps per launch; 0 auto), --kplane (per-plane K for
layered/homogeneous models: not the headline), --sponge W (Cerjan frame),
--transport nccl|peer (N > 1 halo exchange), --strong (N > 1: split the
workload's grid instead of stacking N copies), --no-graph, --no-e2e.

--impl reference times the fp64 CPU oracle (the tier's reference arm) on a
bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_POINT = 16.0   # read p, p_prev, K; write p_next (fp32), DESIGN.md section 5


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu_traffic(workload: str, order: int, suffix: str = ""):
    """DRAM bytes per launch of the step kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        e = d.get(f"{workload}:o{order}{suffix}")
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled (every 50 ms) during the
    timed region by a streaming `nvidia-smi -lms` child process."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._p = None
        self._t = None

    def _reader(self):
        for line in self._p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "50"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._reader, daemon=True)
            self._t.start()
            time.sleep(0.3)   # let the first samples arrive before the timed region
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is not None:
            time.sleep(0.1)
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
            self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(s[0]) for s in self.samples) if v is not None]
        mx = [v for v in (num(s[1]) for s in self.samples) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].strip().lower() == "active"})
        # "under load": samples at or above half the max clock (idle samples excluded)
        load = [v for v in sm if mx and v >= 0.5 * max(mx)] or sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


class NvmlClockSampler(ClockSampler):
    """Same record as ClockSampler, read in-process through NVML every 100 ms
    (no nvidia-smi child process polling the driver during the timed region)."""

    def __init__(self, device: int):
        super().__init__(device)
        self._stop = threading.Event()

    def _poll(self):
        import pynvml as nv
        h = nv.nvmlDeviceGetHandleByIndex(self.device)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
                ("sw_power_cap", 0x4)]
        while True:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for _, b in bits])
            except Exception:
                pass
            if self._stop.wait(0.1):
                break

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
            time.sleep(0.15)
        except Exception:
            self._t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=5)


class PowerSampler:
    """NVML every 50 ms over a pass: SM clock, power, throttle reasons."""

    def __init__(self, device: int):
        self.device, self.rows, self._stop, self._t = device, [], threading.Event(), None

    def _poll(self):
        import pynvml as nv
        h = nv.nvmlDeviceGetHandleByIndex(self.device)
        while not self._stop.wait(0.05):
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "power_w_max": None, "reasons": ["unavailable"]}
        bits = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
                ("sw_power_cap", 0x4)]
        r = 0
        for x in self.rows:
            r |= x[2]
        return {"sm_mhz": float(np.median([x[0] for x in self.rows])), "power_w_max": max(x[1] for x in self.rows),
                "reasons": [n for n, b in bits if r & b], "samples": len(self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("FD_BENCH_SHARE_GPU") == "1":
        local = 0        # test hook: every rank on cuda:0 (peer transport, gloo plumbing)
    return rank, world, local


# ------------------------------------------------------------------ CPU side
def cpu_oracle_sample(wl, budget_s: float = 15.0):
    """Time the fp64 oracle as it stands on the host cores on a bounded sample:
    full-width planes of the workload's grid, steps chosen from a calibration
    step so the sample takes ~budget_s seconds.  Returns (Gpts/s, cores, desc)."""
    import oracle
    oracle.build()
    cores = oracle.max_threads()
    vel = wl.vel()
    src = [(s.idx, s.f, s.t0, s.amp) for s in wl.sources]
    # calibration: 1 step
    t0 = time.perf_counter()
    oracle.run(vel, wl.h, wl.dt, wl.order, 1, src, nthreads=cores)
    t1 = time.perf_counter() - t0
    steps = int(max(2, min(wl.steps, budget_s / max(t1, 1e-3))))
    t0 = time.perf_counter()
    oracle.run(vel, wl.h, wl.dt, wl.order, steps, src, nthreads=cores)
    el = time.perf_counter() - t0
    return wl.npts * steps / el / 1e9, cores, f"{wl.name} full grid {wl.dims}, {steps} steps, {cores} threads"


def cpu_oracle_one_thread(wl, budget_s: float = 3.0):
    """The oracle on ONE host thread (all cores and 1 thread), on a
    slab of full-width planes sized from a calibration step to ~budget_s."""
    import oracle
    from workloads import velocity
    plane = int(np.prod(wl.dims[1:]))
    nz_s = max(4 * wl.order + 1, min(wl.dims[0], int(2e6 // plane) + 1))
    dims_s = (nz_s,) + tuple(wl.dims[1:])
    vel = velocity(wl.model, dims_s, nz_global=wl.dims[0])
    src = [((nz_s // 2,) + tuple(s.idx[1:]), s.f, s.t0, s.amp) for s in wl.sources]
    t0 = time.perf_counter()
    oracle.run(vel, wl.h, wl.dt, wl.order, 1, src, nthreads=1)
    t1 = time.perf_counter() - t0
    steps = int(max(2, min(wl.steps, budget_s / max(t1, 1e-3))))
    t0 = time.perf_counter()
    oracle.run(vel, wl.h, wl.dt, wl.order, steps, src, nthreads=1)
    el = time.perf_counter() - t0
    return nz_s * plane * steps / el / 1e9, f"{dims_s} slab, {steps} steps, 1 thread"


def cpu_info() -> dict:
    """Host CPU as /proc/cpuinfo reports it: model, sockets, physical cores, logical CPUs."""
    model, sockets, cores = "unknown", set(), set()
    try:
        phys = None
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "model name":
                model = v
            elif k == "physical id":
                phys = v
                sockets.add(v)
            elif k == "core id":
                cores.add((phys, v))
    except OSError:
        pass
    return {"cpu_model": model, "sockets": len(sockets) or None, "physical_cores": len(cores) or None,
            "logical_cpus": os.cpu_count()}


def run_reference(args, wl):
    """The tier's reference arm: the fp64 oracle, as it stands, on the host
    cores.  W warm-up steps, then exactly K timed steps in one oracle call on
    a bounded slab of the workload (full-width planes around the source plane),
    the slab sized from a calibration step so the K steps take ~--ref-budget s."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    from workloads import velocity
    oracle.build()
    cores = oracle.max_threads()
    plane = int(np.prod(wl.dims[1:]))

    def sample(nz_s):
        dims_s = (nz_s,) + tuple(wl.dims[1:])
        vel = velocity(wl.model, dims_s, nz_global=wl.dims[0])
        src = [((nz_s // 2,) + tuple(s.idx[1:]), s.f, s.t0, s.amp) for s in wl.sources]
        return dims_s, vel, src

    # calibration: one step on a small slab
    dims_c, vel_c, src_c = sample(max(2 * (wl.order // 2) + 1, min(wl.dims[0], 32)))
    rate = 0.0
    for _ in range(2):                         # the first call also loads the library
        t0 = time.perf_counter()
        oracle.run(vel_c, wl.h, wl.dt, wl.order, 4, src_c, nthreads=cores)
        rate = max(rate, 4 * int(np.prod(dims_c)) / (time.perf_counter() - t0))   # points/s
    nz_s = int(rate * args.ref_budget / max(args.steps, 1) / plane)
    nz_s = max(2 * (wl.order // 2) + 1, min(wl.dims[0], nz_s))
    dims_s, vel, src = sample(nz_s)
    P, Pm, _ = oracle.run(vel, wl.h, wl.dt, wl.order, args.warmup, src, nthreads=cores)
    t0 = time.perf_counter()
    oracle.run(vel, wl.h, wl.dt, wl.order, args.steps, src, P0=P, Pm1=Pm, nthreads=cores)
    el = time.perf_counter() - t0
    npts = int(np.prod(dims_s))
    value = npts * args.steps / el / 1e9
    desc = (f"{wl.name}: {nz_s} of {wl.dims[0]} planes {dims_s}, {args.steps} steps in one oracle call, "
            f"{cores} threads")
    line = {
        "impl": "reference", "metric": "grid-point updates/s (Gpts/s)", "value": value, "unit": "Gpts/s",
        "n_gpus": max(world, args.gpus), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl.name, "grid": list(wl.dims), "order": wl.order, "model": wl.model,
                   "sample_grid": list(dims_s)},
        "cpu_baseline": {"value": value, "unit": "Gpts/s", "cores": cores, "kind": "oracle", "sample": desc,
                         **cpu_info()},
        "e2e": {"value": value, "unit": "Gpts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU side
def _global_dims(wl, world, strong=False):
    """The grid all ranks share: the workload's own (N = 1, or --strong: split
    across the ranks) or N copies stacked along z (weak scaling)."""
    if world == 1 or strong:
        return tuple(wl.dims)
    return (wl.dims[0] * world,) + tuple(wl.dims[1:])


def _velocity(wl, world, strong=False):
    """This rank's fp32 velocity planes (the whole grid at N=1)."""
    from workloads import velocity
    if world == 1:
        return wl.vel(), tuple(wl.dims)
    import torch.distributed as dist
    from paper_2311_05038_b200 import dist as fdd
    gdims = _global_dims(wl, world, strong)
    z0, z1 = fdd.partition(gdims[0], world, dist.get_rank())
    return velocity(wl.model, gdims, z0, z1, nz_global=gdims[0]), gdims


def _make_sim(wl, world, vel, gdims, stream=None, options=None, transport="nccl", sponge=0):
    """This rank's simulation: the whole grid at N=1; at N>1 a z-slab of the
    weak-scaled grid (N copies of the workload's grid stacked along z,
    slab-decomposed, halo exchange inside libfd.so: NCCL send/recv, or the
    step kernels' peer stores with --transport peer)."""
    import paper_2311_05038_b200 as fd
    if world == 1:
        sim = fd.Simulation(vel, wl.h, wl.dt, wl.order, stream=stream, options=options)
    else:
        from paper_2311_05038_b200 import dist as fdd
        sim = fdd.create(vel, gdims, wl.h, wl.dt, wl.order, device=dist_env()[2], stream=stream,
                         options=options, transport=transport, sponge=(sponge, 0.015) if sponge else None)
    if sponge and world == 1:
        sim.set_sponge(sponge, 0.015)        # Cerjan frame (R#18), classic alpha
    for s in wl.sources:
        sim.add_source(s.idx, s.f, s.t0, s.amp)
    sim.set_receivers(wl.receivers)
    return sim


def run_ours(args, wl):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2311_05038_b200 as fd
    from paper_2311_05038_b200 import fd as fdm
    if args.transport != "peer":
        # PyTorch as the device-memory provider (its caching allocator; the peer
        # transport's CUDA IPC mappings need plain cudaMalloc blocks)
        fdm.fd_set_allocator_torch()

    if world > 1:
        import torch.distributed as dist
        if os.environ.get("FD_BENCH_SHARE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    vel, gdims = _velocity(wl, world, args.strong)
    npts_global = int(np.prod(gdims))
    stream = torch.cuda.Stream(device=dev)
    opts = {fd.FD_OPT_ASYNC: 1}
    if args.no_graph:
        opts[fd.FD_OPT_GRAPH] = 0
    opts[fd.FD_OPT_TSTEPS] = args.tsteps
    if args.kplane:
        opts[fd.FD_OPT_KPLANE] = 1
    if args.tb2tile >= 0:
        opts[fd.FD_OPT_TB2TILE] = args.tb2tile
    if args.zchunks > 0:
        opts[fd.FD_OPT_ZCHUNKS] = args.zchunks
    sim = _make_sim(wl, world, vel, gdims, stream=stream.cuda_stream, options=opts, transport=args.transport,
                    sponge=args.sponge)
    sim.step(args.warmup)
    # setup for the timed steps (trace/wavelet tables for both passes, the CUDA
    # graphs to replay) happens here, outside the timed region
    sim.reserve((args.reps + 1) * args.steps)
    stream.synchronize()
    launches0 = sim.info()["kernel_launches"]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    # pass 1 (the value): K steps exactly as a user runs them (CUDA-graph
    # replay), repeated --reps times (each repetition exactly K steps between
    # barriers + synchronize); the value is the median repetition, max over
    # ranks per repetition (min and median of >= 5 repetitions)
    sampler = {"nvml": NvmlClockSampler, "smi": ClockSampler}.get(args.clock_sampler, NvmlClockSampler)
    rep_ms = []
    with sampler(local) as clk:
        for rep in range(args.reps):
            if rep:
                if world > 1:
                    torch.distributed.barrier()
                torch.cuda.synchronize()
            ev0.record(stream)
            sim.step(args.steps)
            ev1.record(stream)
            ev1.synchronize()
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            rep_ms.append(ev0.elapsed_time(ev1))
    launches = int(round((sim.info()["kernel_launches"] - launches0) / args.reps))   # per timed repetition
    if world > 1:
        t = torch.tensor(rep_ms, dtype=torch.float64,
                         device=dev if torch.distributed.get_backend() == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        rep_ms = [float(x) for x in t.cpu().tolist()]
    ms = float(np.median(rep_ms))
    # pass 2 (per-kernel breakdown): K more steps with CUDA events around every
    # launch on the library's stream.  At N = 1 the roofline's kernel time comes
    # from pass 1 itself (its events ÷ the step-kernel launches): the GPU runs
    # pass 2 after ~K steps of full load, when the 1 kW power cap may already
    # have lowered the SM clock (scripts/launch_timing.py)
    fd.fd_set_option(sim.ctx, fd.FD_OPT_PROFILE, 1)
    sim.reset_kernel_times()
    sim.step(args.steps)
    stream.synchronize()
    ktimes = sim.kernel_times()
    fd.fd_set_option(sim.ctx, fd.FD_OPT_PROFILE, 0)
    info = sim.info()
    T = sim.traces()
    finite = bool(np.all(np.isfinite(T)))
    def sustained_pass():
        # pass 3, after everything else (e2e included) so that the power-capped
        # state it measures does not leak into the other numbers: graph replay
        # for ~args.sustained seconds of full load, clocks / power sampled
        out = None
        if args.sustained > 0 and world == 1:
            n3 = max(args.steps, int(args.sustained / max(ms / 1e3 / args.steps, 1e-9)))
            n3 -= n3 % 2
            sim.reserve(n3)
            stream.synchronize()
            with PowerSampler(local) as pw:
                ev0.record(stream)
                sim.step(n3)
                ev1.record(stream)
                ev1.synchronize()
            ms3 = ev0.elapsed_time(ev1)
            out = {"value": wl.npts * n3 / (ms3 / 1e3) / 1e9, "unit": "Gpts/s", "steps": n3,
                   "seconds": ms3 / 1e3, **pw.summary(),
                   "what": "graph replay after the other passes, ~%.0f s of full load (reported, not the value)"
                           % args.sustained}
        if world > 1:
            from paper_2311_05038_b200 import dist as fdd
            fdd.close(sim)
        else:
            sim.close()
        return out

    ms_step = ms / args.steps
    gpts = npts_global * args.steps / (ms / 1e3) / 1e9

    # e2e through the public API with host buffers (pinned): create (H2D of the
    # model, K computed on the device), K steps, traces + final wavefield read
    # back (D2H).  The input arrays exist before the clock starts.
    if args.no_e2e:
        return _emit(args, wl, world, rank, gpts, ms_step, info, launches, clk, finite, None, ktimes,
                     sustained_pass(), rep_ms)
    vel_pin = torch.empty(vel.shape, dtype=torch.float32, pin_memory=True).numpy()
    vel_pin[...] = vel
    out_pin = torch.empty(vel.shape, dtype=torch.float32, pin_memory=True).numpy()
    tr_pin = torch.empty((len(wl.receivers), args.steps), dtype=torch.float32, pin_memory=True).numpy()
    # three complete runs; the reported time is their median (host-side
    # effects -- page-cache state, CPU clocks -- vary run to run)
    runs = []
    for _ in range(3):
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        s2 = _make_sim(wl, world, vel_pin, gdims, transport=args.transport, sponge=args.sponge,
                       options={fd.FD_OPT_KPLANE: 1} if args.kplane else None)
        s2.step(args.steps)
        T2 = s2.traces(out=tr_pin)
        W2 = s2.wavefield(out=out_pin)
        e2e_s = time.perf_counter() - t0     # results are on the host: teardown is not part of the job
        if world > 1:
            from paper_2311_05038_b200 import dist as fdd
            e2e_s = fdd.max_over_ranks(e2e_s)
            fdd.close(s2)                    # collective: no rank frees buffers a neighbour still maps
        else:
            s2.close()
        runs.append(e2e_s)
    e2e_s = sorted(runs)[1]
    h2d = vel_pin.nbytes + 8 * len(wl.receivers) * wl.ndim
    d2h = T2.nbytes + W2.nbytes
    e2e = {"value": npts_global * args.steps / e2e_s / 1e9, "unit": "Gpts/s",
           "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
           "seconds": e2e_s, "seconds_runs": runs, "pinned_host_buffers": True,
           "what": "fd_create (model upload) + fd_step(K) + fd_get_traces + fd_get_wavefield",
           "device_memory": "torch caching allocator (fd_set_allocator)" if args.transport != "peer" else "cudaMalloc"}
    return _emit(args, wl, world, rank, gpts, ms_step, info, launches, clk, finite, e2e, ktimes, sustained_pass(),
                 rep_ms)


def _reps_summary(rep_ms, wl, world, args):
    """The timed repetitions of pass 1 (each exactly K steps; max over ranks)."""
    if not rep_ms:
        return None
    npts = (1 if args.strong else world) * wl.npts
    rate = [npts * args.steps / (m / 1e3) / 1e9 for m in rep_ms]
    return {"n": len(rep_ms), "ms": rep_ms, "value_median": float(np.median(rate)), "value_max": max(rate),
            "value_min": min(rate), "ms_per_step_min": min(rep_ms) / args.steps,
            "ms_per_step_median": float(np.median(rep_ms)) / args.steps,
            "what": "value = the median repetition; each repetition K steps between barrier + synchronize"}


def _l2_note(wl) -> str:
    """Timing rule: inputs larger than L2 (no flush) -- say by how much."""
    ws = 12.0 * wl.npts           # p, p_prev, K (fp32) read per step
    l2 = 126e6
    if ws > l2:
        return "no flush: per-step working set %.3f GB = %.1fx the 126 MB L2" % (ws / 1e9, ws / l2)
    return "working set %.2f MB fits the 126 MB L2 (launch/latency-bound config, not a bandwidth number)" % (ws / 1e6)


def _emit(args, wl, world, rank, gpts, ms_step, info, launches, clk, finite, e2e, ktimes, sustained=None,
          rep_ms=None):
    peak, peak_src = _peaks()
    # dominant kernel: the fused step kernel, one launch per step; its average
    # launch duration from the events around each launch in the timed region
    # 0: each fd_step(n) call is one cluster launch (FD_OPT_RESIDENT, C1-size
    # grids): latency-bound, the fraction below is not a roofline statement
    resident = info.get("steps_per_launch", 1) == 0
    steps_per_launch = int(info.get("steps_per_launch", 1) or 1)
    npass = args.steps // steps_per_launch + args.steps % steps_per_launch
    kms, kn = ktimes.get("fused", (ms_step * args.steps, npass))
    # per pass over the slab: at N > 1 a pass is several launches (boundary
    # regions on the comm stream + the interior); their durations are summed
    k_avg_prof_s = kms / max(npass, 1) / 1e3
    if world == 1:
        # the timed region (pass 1): its CUDA events ÷ the step-kernel launches
        # (includes the graphs' one-thread step-counter kernels, ~0.3 %)
        k_avg_s = ms_step * args.steps / max(npass, 1) / 1e3
        ksrc = "CUDA events around the timed region (pass 1) / step-kernel launches"
    else:
        k_avg_s = k_avg_prof_s
        ksrc = "CUDA events around every launch, a second pass of K steps (summed per pass)"

    # algorithmic bytes per launch: 16 B per point for a one-step launch; a
    # temporal-blocking launch does two steps for 20 B per point; with K per
    # plane (--kplane, FD_OPT_KPLANE active) 4 B less (K is not streamed)
    kz = bool(info.get("kplane"))
    npts_local = int(np.prod([d for d in info["local_dims"][:wl.ndim]]))     # this rank's points
    bytes_per_launch = ((20.0 if steps_per_launch >= 2 else BYTES_PER_POINT) - (4.0 if kz else 0.0)) * npts_local
    achieved = bytes_per_launch / k_avg_s / 1e9
    if world == 1 and steps_per_launch >= 2 and args.steps % steps_per_launch:
        # K not a multiple of the steps per launch: the remainder runs as single
        # steps (16 B per point); the whole region's algorithmic bytes / its time
        nrem = args.steps % steps_per_launch
        total = (args.steps // steps_per_launch) * bytes_per_launch + nrem * (BYTES_PER_POINT - (4.0 if kz else 0.0)) * npts_local
        achieved = total / (ms_step * args.steps / 1e3) / 1e9
    roof = {"bound": "latency" if resident else "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": _ncu_traffic(wl.name, wl.order, (f":tb{steps_per_launch}" if steps_per_launch >= 2 else "")
                                    + (":kz" if kz else "")),
            "peak_source": peak_src,
            "algorithmic_bytes_per_point": bytes_per_launch / npts_local / steps_per_launch,
            "algorithmic_bytes_per_launch": bytes_per_launch, "steps_per_launch": steps_per_launch,
            "points_per_launch": npts_local,
            "kernel": "resident_kernel" if resident else
                      "rs2d_step_kernel" if int(info.get("tb_kind", 0)) == 1 else
                      {(3, 1): "fused_step_kernel", (3, 2): "tb2ws_step_kernel", (2, 1): "tile2d_step_kernel",
                       (2, 2): "tb2d_step_kernel", (2, 3): "tbs2d_step_kernel",
                       (2, 4): "tbs2d_step_kernel"}[(wl.ndim, steps_per_launch)],
            "kernel_ms_per_launch": k_avg_s * 1e3, "launches_per_pass": kn / max(npass, 1),
            "kernel_ms_per_launch_profile_pass": k_avg_prof_s * 1e3,
            "kernel_share_of_step_profile_pass": (kms / max(sum(v[0] for v in ktimes.values()), 1e-12))
            if ktimes else None,
            "kernel_times_ms": {k: v[0] for k, v in ktimes.items()},
            # the Gpts/s ceiling of this kernel's data movement at `peak`, and the
            # value against the one-step-per-launch (16 B/update) ceiling
            "gpts_ceiling": peak / (bytes_per_launch / npts_local / steps_per_launch),
            "value_over_single_step_ceiling": gpts * BYTES_PER_POINT / peak / world,
            "kernel_time_source": ksrc}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, desc = cpu_oracle_sample(wl, args.cpu_budget)
        v1, desc1 = cpu_oracle_one_thread(wl, min(3.0, args.cpu_budget / 5))
        cpu = {"value": v, "unit": "Gpts/s", "cores": cores, "kind": "oracle", "sample": desc,
               "value_1_thread": v1, "sample_1_thread": desc1, **cpu_info()}
    line = {
        "metric": "grid-point updates/s (Gpts/s)", "value": gpts, "unit": "Gpts/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if (args.strong and world > 1) else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": wl.name, "grid": list(wl.dims), "order": wl.order, "model": wl.model,
                   "dt": wl.dt, "h": wl.h, "receivers": len(wl.receivers), "sources": len(wl.sources),
                   "l2": _l2_note(wl),
                   "parallelism": (f"z-slabs x{world} ({'in-kernel peer-store' if args.transport == 'peer' else 'NCCL'}"
                                   f" halo exchange)") if world > 1 else "1 GPU",
                   **({"shared_gpu": True} if os.environ.get("FD_BENCH_SHARE_GPU") == "1" else {}),
                   **({"sponge_cells": args.sponge} if args.sponge else {}),
                   **({"k_storage": "per-plane table (FD_OPT_KPLANE; the model is layered)" if kz else
                       "K field (per-plane table requested, model not plane-constant)"} if args.kplane else {}),
                   "global_grid": list(_global_dims(wl, world, args.strong)),
                   "tile": [info["tile_x"], info["tile_y"]], "zchunks": info["zchunks"], "ctas": info["ctas"],
                   **({"nccl_comm_nranks": info.get("comm_nranks")} if world > 1 else {}),
                   "graph_steps": info.get("graph_steps")},
        "repetitions": _reps_summary(rep_ms, wl, world, args),
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clk.summary(), "traces_finite": finite,
        **({"sustained": sustained} if sustained else {}),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--order", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="plain launches instead of CUDA-graph replay")
    ap.add_argument("--clock-sampler", default="nvml", choices=["nvml", "smi"])
    ap.add_argument("--sponge", type=int, default=0,
                    help="absorbing Cerjan frame of this many cells (fd_set_sponge, alpha 0.015); 0 = band rule only")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer"],
                    help="halo transport at N>1: NCCL send/recv or in-kernel peer stores (CUDA IPC)")
    ap.add_argument("--tsteps", type=int, default=0, choices=[0, 1, 2, 3, 4],
                    help="0 auto (library default), 1 one step per launch, S >= 2 temporal blocking "
                         "(S steps per launch, 20/S B per update; S >= 3: 2D single slab)")
    ap.add_argument("--sustained", type=float, default=2.0,
                    help="seconds of an extra graph-replay pass reported as 'sustained' (power-capped state); 0 = off")
    ap.add_argument("--strong", action="store_true",
                    help="N > 1: split the workload's grid across the ranks (strong scaling, BASELINE configs[3]) "
                         "instead of stacking N copies along z (weak scaling, the default)")
    ap.add_argument("--kplane", action="store_true",
                    help="FD_OPT_KPLANE: K per plane for layered/homogeneous models (12 B per single-step update; "
                         "not the headline)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=90.0, help="seconds of oracle work for --impl reference")
    ap.add_argument("--tb2tile", type=int, default=-1,
                    help="FD_OPT_TB2TILE: pin a two-step kernel configuration (tuning; -1 = auto)")
    ap.add_argument("--zchunks", type=int, default=0,
                    help="FD_OPT_ZCHUNKS: pin the z-chunk count (tuning; 0 = auto)")
    ap.add_argument("--reps", type=int, default=5,
                    help="repetitions of the K timed steps (value = the median repetition; min/median/max reported)")
    ap.add_argument("--launch-check", action="store_true",
                    help="start the N ranks (spawning torchrun when --gpus N > 1 has no WORLD_SIZE), check the "
                         "world size, print one JSON line and exit (no GPU work; tests the launch path)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    args.reps = max(1, args.reps)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        return spawn_ranks(args, sys.argv[1:] if argv is None else list(argv))
    rank, world, _ = dist_env()
    if args.impl == "ours" and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
              f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus", file=sys.stderr)
        return 2
    if args.launch_check:
        return launch_check(args)
    from workloads import config
    wl = config(args.config, order=args.order)
    if args.impl == "reference":
        return run_reference(args, wl)
    return run_ours(args, wl)


def spawn_ranks(args, argv) -> int:
    """`bench.py --gpus N` without torchrun's environment: start N ranks on this
    node (python -m torch.distributed.run, rendezvous on 127.0.0.1), one per GPU,
    with NCCL's init log on (communicator rank counts in stderr).  Refuses when
    the node has fewer than N GPUs (FD_BENCH_SHARE_GPU=1: every rank on cuda:0,
    test hook, not a scaling number)."""
    import socket
    share = os.environ.get("FD_BENCH_SHARE_GPU") == "1"
    if not share:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has {have} "
                  f"(FD_BENCH_SHARE_GPU=1 runs every rank on cuda:0 as a test hook)", file=sys.stderr)
            return 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]
    return subprocess.run(cmd, env=env).returncode


def launch_check(args) -> int:
    """One JSON line from rank 0 after every rank joined the process group (gloo)."""
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        t = [None] * world
        dist.all_gather_object(t, (rank, local))
        dist.barrier()
    else:
        t = [(0, local)]
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "gpus_requested": args.gpus,
                          "ranks": [list(x) for x in t]}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
