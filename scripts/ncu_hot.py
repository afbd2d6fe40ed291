"""Top SASS lines of an ncu capture by warp-stall samples (run here, no GPU):
    python scripts/ncu_hot.py gpurun_out/prof_X.ncu-rep [N]
Prints address, samples (all / not issued), executed count and the SASS text,
plus the CUDA source line it maps to (-lineinfo)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ia, isrc, iall, inot, iex = (hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"),
                             hdr.index("Warp Stall Sampling (Not-issued Samples)"), hdr.index("Instructions Executed"))
tot = sum(int(r[iall] or 0) for r in data if len(r) > iall)
print(f"total samples {tot}")
data = [r for r in data if len(r) > iall]
for i, r in sorted(enumerate(data), key=lambda t: -int(t[1][iall] or 0))[:n]:
    print(f"{i:5d} {r[ia][-5:]} {int(r[iall]):7d} {int(r[inot]):7d} {r[iex]:>10s}  {r[isrc].strip()}")
