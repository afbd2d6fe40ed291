#!/bin/bash
# A few ncu metrics of the step kernel for library variants (gpurun):
#   VARIANTS="default O3D" ARGS="--config C4 --steps 10" TAG=x bash scripts/ncu_quick.sh
set -u
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
for v in ${VARIANTS}; do
  lib=paper_2311_05038_b200/libfd_${v}.so
  [ "$v" = "default" ] && lib=paper_2311_05038_b200/libfd.so
  FD_LIB=$lib timeout 900 ncu --metrics $M --clock-control none -k regex:step_kernel -s 6 -c 3 --csv \
      --log-file gpurun_out/ncuq_${TAG}_${v}.csv \
      python bench.py --no-cpu-baseline --no-e2e --sustained 0 --reps 1 ${ARGS} > /dev/null 2>&1
  echo "== $v"; grep -v "^==" gpurun_out/ncuq_${TAG}_${v}.csv | python -c "
import csv, sys
rows = list(csv.reader(sys.stdin))
h = rows[0]; im, iv, iu = h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
for r in rows[1:]:
    print(r[im], r[iv], r[iu])"
done
