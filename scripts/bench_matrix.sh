#!/bin/bash
# Measurement matrix on one GPU (run under gpurun): every BASELINE workload and
# order through bench.py (value pass only: 5 repetitions of K steps, K short
# enough that the repetitions stay ahead of the 1 kW power cap), default
# kernels, --tsteps and --kplane variants.  Summarise with: python scripts/bench_matrix.py TAG
TAG=${TAG:-r05}
mkdir -p gpurun_out
out=gpurun_out/matrix_${TAG}.log
: > $out
B="python bench.py --no-cpu-baseline --no-e2e --sustained 0"
for a in "--config C3 --order 2 --steps 200" "--config C3 --order 4 --steps 200" "--config C3 --order 6 --steps 200" \
         "--config C3 --order 8 --steps 200" "--config C3 --order 2 --steps 200 --tsteps 1" \
         "--config C3 --order 8 --steps 200 --tsteps 2" \
         "--config C3 --order 2 --steps 200 --kplane" "--config C3 --order 8 --steps 200 --kplane" \
         "--config C2 --order 2 --steps 1000" "--config C2 --order 4 --steps 1000" "--config C2 --order 6 --steps 1000" \
         "--config C2 --order 8 --steps 1000" "--config C2 --order 2 --steps 1000 --tsteps 1" \
         "--config C2 --order 2 --steps 1002 --tsteps 3 --zchunks 9" \
         "--config C2 --order 2 --steps 1000 --kplane" "--config C2 --order 8 --steps 1000 --kplane" \
         "--config C4 --order 2 --steps 40" "--config C4 --order 8 --steps 40" "--config C5:1 --order 2 --steps 60" \
         "--config C1 --order 2 --steps 500" "--config C1 --order 8 --steps 500"; do
  echo "# $a" >> $out
  timeout 300 $B $a >> $out 2>&1
done
