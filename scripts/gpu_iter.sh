# One GPU iteration on the 2D kernels (gpurun): TAG=x CASES="..." bash scripts/gpu_iter.sh
set -u
mkdir -p gpurun_out
if [ -z "${NOTEST:-}" ]; then
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py -k "${TESTK:-2d or tbs2d or virtual_slabs}" tests/test_gpu_peer.py tests/test_gpu_sponge.py tests/test_gpu_rs2d.py > gpurun_out/${TAG}_pytest.log 2>&1
tail -3 gpurun_out/${TAG}_pytest.log
fi
B="python bench.py --no-cpu-baseline --no-e2e --sustained 0 --steps 2000 --warmup 20 --reps 3"
: > gpurun_out/${TAG}_bench.log
IFS=';'
for a in ${CASES}; do
  unset IFS
  echo "# $a" >> gpurun_out/${TAG}_bench.log
  timeout 300 $B $a >> gpurun_out/${TAG}_bench.log 2>&1
done
unset IFS
python scripts/bench_lines.py gpurun_out/${TAG}_bench.log
if [ -n "${NCU:-}" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:${NCUK:-rs2d_step_kernel} -s 4 -c 1 \
   -o gpurun_out/prof_${TAG} -f python bench.py --no-cpu-baseline --no-e2e --sustained 0 --reps 1 --steps 40 --warmup 4 ${NCU} > gpurun_out/${TAG}_ncu.log 2>&1
tail -1 gpurun_out/${TAG}_ncu.log
fi
