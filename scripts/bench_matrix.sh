#!/bin/bash
# Measurement matrix on one GPU (run under gpurun): every BASELINE workload and
# order through bench.py (value pass only), default kernels, --tsteps 1 and
# --kplane variants.  Summarise with: python scripts/bench_matrix.py TAG
TAG=${TAG:-r05}
mkdir -p gpurun_out
out=gpurun_out/matrix_${TAG}.log
: > $out
B="python bench.py --no-cpu-baseline --no-e2e --sustained 0"
for a in "--config C3 --order 2" "--config C3 --order 4" "--config C3 --order 6" "--config C3 --order 8" \
         "--config C3 --order 2 --tsteps 1" "--config C3 --order 2 --kplane" "--config C3 --order 8 --kplane" \
         "--config C2 --order 2 --steps 2000" "--config C2 --order 4 --steps 2000" "--config C2 --order 6 --steps 2000" \
         "--config C2 --order 8 --steps 2000" "--config C2 --order 2 --steps 2000 --tsteps 1" \
         "--config C2 --order 2 --steps 2000 --kplane" "--config C2 --order 8 --steps 2000 --kplane" \
         "--config C1 --order 2 --steps 500" "--config C1 --order 8 --steps 500"; do
  echo "# $a" >> $out
  timeout 300 $B $a >> $out 2>&1
done
