#!/bin/bash
# Run on the GPU box (gpurun): ncu launch list + one full capture of the fused
# kernel per workload/order.  Outputs under gpurun_out/.  Never wrap a
# multi-rank command in ncu.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r01}
for spec in "C3 2" "C3 8" "C2 2" "C2 8"; do
  set -- $spec
  cfg=$1; ord=$2
  # launch list (cold-cache, serialised): compare the fused kernel's SHARE of the step
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
      --log-file gpurun_out/launches_${TAG}_${cfg}_o${ord}.csv \
      python bench.py --config $cfg --order $ord --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_${cfg}_o${ord}.log 2>&1
  # full capture of one steady-state launch of the fused kernel
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 \
      -o gpurun_out/prof_${TAG}_${cfg}_o${ord} -f \
      python bench.py --config $cfg --order $ord --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_${cfg}_o${ord}.log 2>&1
done
# temporal blocking (two steps per launch), 3D order 2 and 4
for ord in 2 4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tb2 -s 3 -c 1 \
      -o gpurun_out/prof_${TAG}_C3_o${ord}_tb2 -f \
      python bench.py --config C3 --order $ord --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --tsteps 2 > gpurun_out/ncu_full_C3_o${ord}_tb2.log 2>&1
done
