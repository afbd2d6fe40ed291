#!/usr/bin/env python
"""Summarise gpurun_out/matrix_TAG.log (scripts/bench_matrix.sh) into
profiles/bench_matrix_TAG.md."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(tag):
    rows, args = [], None
    for line in open(os.path.join(ROOT, "gpurun_out", f"matrix_{tag}.log")):
        if line.startswith("# "):
            args = line[2:].strip()
        elif line.startswith("{"):
            d = json.loads(line)
            r = d["roofline"]
            rows.append((args, d["config"]["workload"], d["config"]["order"], r["kernel"], r["steps_per_launch"],
                         r["algorithmic_bytes_per_point"], d["value"], r["frac"], d["ms_per_step"] * 1e3,
                         d["clocks"]["sm_mhz"], ",".join(d["clocks"]["reasons"]) or "-",
                         (d.get("repetitions") or {}).get("value_max", d["value"])))
    out = [f"# bench.py measurement matrix, {tag}", "",
           "One B200, `scripts/bench_matrix.sh` (value pass of bench.py: CUDA-graph replay of K steps,",
           "CUDA events on the library stream; roofline frac = algorithmic bytes per launch / kernel time",
           "in the timed region / MEASURED_PEAKS hbm_gbs).", "",
           "| bench.py args | workload | order | kernel | steps/launch | alg. B per update | Gpts/s (median of 5) | best rep | roofline frac | us/step | SM MHz | throttle |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for a, w, o, k, spl, b, v, f, us, mhz, why, best in rows:
        out.append(f"| `{a}` | {w} | {o} | `{k}` | {spl} | {b:.1f} | {v:.1f} | {best:.1f} | {f:.3f} | {us:.2f} | {mhz} | {why} |")
    path = os.path.join(ROOT, "profiles", f"bench_matrix_{tag}.md")
    open(path, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r05")
