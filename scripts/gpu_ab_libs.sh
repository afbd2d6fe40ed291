# A/B of library builds (gpurun): LIBS="A B" CASES="--order 2;--order 4" TAG=x bash scripts/gpu_ab_libs.sh
set -u
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-e2e --sustained 0 --steps 2000 --warmup 20 --reps 3 --config ${CFG:-C2}"
: > gpurun_out/${TAG}_bench.log
for rep in 1 2; do
IFS=';'
for a in ${CASES}; do
  unset IFS
  for v in ${LIBS}; do
    echo "# lib=$v rep=$rep $a" >> gpurun_out/${TAG}_bench.log
    FD_LIB=paper_2311_05038_b200/libfd_${v}.so timeout 300 $B $a >> gpurun_out/${TAG}_bench.log 2>&1
  done
done
done
python scripts/bench_lines.py gpurun_out/${TAG}_bench.log
