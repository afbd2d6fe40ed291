# rs2d A/B (gpurun): steal on / off over a few tiles
set -u
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-e2e --sustained 0 --steps 2000 --warmup 20 --reps 3 --config C2"
: > gpurun_out/${TAG}_bench.log
IFS=';'
for a in ${CASES}; do
  unset IFS
  for st in 1 0; do
    echo "# steal=$st $a" >> gpurun_out/${TAG}_bench.log
    FD_RS_STEAL=$st timeout 300 $B $a >> gpurun_out/${TAG}_bench.log 2>&1
  done
done
python scripts/bench_lines.py gpurun_out/${TAG}_bench.log
