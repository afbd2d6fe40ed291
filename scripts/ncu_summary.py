#!/usr/bin/env python
"""Summarise ncu captures (run HERE, no GPU needed) into profiles/.

    python scripts/ncu_summary.py TAG            # reads gpurun_out/prof_TAG_*.ncu-rep
                                                 #   and gpurun_out/launches_TAG_*.csv

Writes profiles/ncu_TAG.md (human summary), merges per-workload DRAM bytes per
launch into profiles/ncu_summary.json (read by bench.py for roofline.traffic),
and copies the launch lists to profiles/.
"""
import csv
import glob
import io
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def to_bytes(v, u):
    return float(v.replace(",", "")) * UNIT.get(u, 1)


def npts_of(workload):
    sys.path.insert(0, ROOT)
    from workloads import config
    return config(workload).npts


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    summ_path = os.path.join(PROF, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    lines = [f"# ncu summary, tag {tag}", "",
             "Captured with `scripts/gpu_profile.sh` (ncu --set full --clock-control none, one steady-state",
             "launch of the fused step kernel; launch lists with gpu__time_duration.sum).  Algorithmic bytes",
             "= 16 B x grid points per launch (DESIGN.md section 5.4).", ""]
    for rep in sorted(glob.glob(os.path.join(OUT, f"prof_{tag}_*.ncu-rep"))):
        m = re.match(rf"prof_{tag}_(C\d)_o(\d)(_tb(\d))?(_kz)?\.ncu-rep", os.path.basename(rep))
        if not m:
            continue
        wl, order, kz = m.group(1), int(m.group(2)), bool(m.group(5))
        spl = int(m.group(4)) if m.group(4) else 1
        d = raw(rep)
        kname = d.get("Kernel Name", ("", ""))[0]
        if spl == 1 and "tb2" in kname:      # the default 3D order-2 path is two steps per launch
            spl = 2
        tb2 = spl >= 2
        rd = to_bytes(*d["dram__bytes_read.sum"])
        wr = to_bytes(*d["dram__bytes_write.sum"])
        npts = npts_of(wl)
        dur = float(d["gpu__time_duration.sum"][0].replace(",", ""))
        dunit = d["gpu__time_duration.sum"][1]
        dur_s = dur * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(dunit, 1e-9)
        alg = ((20.0 if tb2 else 16.0) - (4.0 if kz else 0.0)) * npts    # K per plane: not streamed
        summ[f"{wl}:o{order}{f':tb{spl}' if tb2 else ''}{':kz' if kz else ''}"] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                                  "algorithmic_bytes": alg, "bytes_per_point": (rd + wr) / npts,
                                  "ncu_duration_s": dur_s, "tag": tag}
        lines += [f"## {wl}, order {order}{f' (temporal blocking, {spl} steps per launch)' if tb2 else ''}"
                  f"{' (K per plane, FD_OPT_KPLANE)' if kz else ''}", "",
                  f"* kernel: `{kname[:120]}`",
                  f"* DRAM traffic per launch: {(rd + wr) / 1e9:.3f} GB = {(rd + wr) / npts:.2f} B/pt "
                  f"(algorithmic {alg / npts:.0f} B/pt = {alg / 1e9:.3f} GB)",
                  f"* ncu duration {dur_s * 1e6:.1f} us -> {(rd + wr) / dur_s / 1e9:.0f} GB/s DRAM, "
                  f"{alg / dur_s / 1e9:.0f} GB/s algorithmic", "", "| metric | value |", "|---|---|"]
        for key, name in METRICS:
            if key in d:
                lines.append(f"| {name} (`{key}`) | {d[key][0]} {d[key][1]} |")
        stalls = sorted(((float(v[0].replace(",", "")), k) for k, v in d.items()
                         if k.startswith("smsp__average_warps_issue_stalled") and
                         k.endswith("_per_issue_active.ratio")), reverse=True)[:6]
        lines += ["", "Top stall reasons (warps per issue-active cycle): " +
                  ", ".join(f"{k.split('stalled_')[1].split('_per')[0]} {v:.2f}" for v, k in stalls), ""]
    for f in sorted(glob.glob(os.path.join(OUT, f"launches_{tag}_*.csv"))):
        shutil.copy(f, PROF)
        rows = [r for r in csv.reader(open(f)) if len(r) > 10 and r[0] != "ID"]
        tot = {}
        for r in rows:
            name = r[4].split("(")[0].replace("void ", "")
            tot[name] = tot.get(name, 0.0) + float(r[-1].replace(",", ""))
        allt = sum(tot.values())
        lines += [f"### launch list {os.path.basename(f)}", "", "| kernel | total ns | share |", "|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            lines.append(f"| {k} | {v:.0f} | {v / allt:.1%} |")
        lines.append("")
    json.dump(summ, open(summ_path, "w"), indent=1, sort_keys=True)
    open(os.path.join(PROF, f"ncu_{tag}.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
