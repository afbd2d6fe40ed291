#!/bin/bash
# compute-sanitizer over every kernel path (run under gpurun): memcheck,
# racecheck, synccheck and initcheck on scripts/sanitize_run.py, plus memcheck
# with the tb2d linear units.  Logs: gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 3 python scripts/sanitize_run.py \
      > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
done
FD_TB2D_LINEAR=1 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 3 python scripts/sanitize_run.py \
    > gpurun_out/sanitize_memcheck_linear.log 2>&1
echo "memcheck(linear) rc=$?" >> gpurun_out/sanitize_summary.txt
cat gpurun_out/sanitize_summary.txt
