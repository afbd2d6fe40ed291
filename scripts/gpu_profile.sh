#!/bin/bash
# Run on the GPU box (gpurun): ncu launch list + one full capture of the step
# kernel per workload/order.  Outputs under gpurun_out/ (keep each call under
# gpurun's 64 MiB: a few captures per call via SPECS).  Never wrap a
# multi-rank command in ncu.
#   SPECS="C3:2:1 C3:2:2 C2:2:1" TAG=r03 bash scripts/gpu_profile.sh
#   (workload:order:steps-per-launch[:kz]; 2 = temporal blocking, kz = --kplane)
set -u
mkdir -p gpurun_out
TAG=${TAG:-r03}
SPECS=${SPECS:-"C3:2:2 C3:2:1 C3:8:1"}
for spec in $SPECS; do
  IFS=: read cfg ord ts kz <<< "$spec"
  sfx=""; [ "$ts" -ge 2 ] && sfx="_tb${ts}"
  kzf=""; [ "${kz:-}" = "kz" ] && { sfx="${sfx}_kz"; kzf="--kplane"; }
  # launch list (cold-cache, serialised): compare the step kernel's SHARE of the step
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
      --log-file gpurun_out/launches_${TAG}_${cfg}_o${ord}${sfx}.csv \
      python bench.py --config $cfg --order $ord --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --reps 1 --tsteps $ts $kzf \
      > /dev/null 2>&1
  # full capture of one steady-state launch of the step kernel
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-step_kernel} -s ${KSKIP:-5} -c 1 \
      -o gpurun_out/prof_${TAG}_${cfg}_o${ord}${sfx} -f \
      python bench.py --config $cfg --order $ord --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --reps 1 --tsteps $ts $kzf \
      > /dev/null 2>&1
done
ls -la gpurun_out
