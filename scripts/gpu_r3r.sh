set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_fulllength.py > gpurun_out/r3r_pytest.log 2>&1
tail -4 gpurun_out/r3r_pytest.log
B="python bench.py --no-cpu-baseline --no-e2e --sustained 0"
: > gpurun_out/r3r_bench.log
for a in "--config C2 --order 2 --steps 2000" "--config C2 --order 4 --steps 2000" "--config C2 --order 6 --steps 2000" "--config C2 --order 8 --steps 2000" "--config C2 --order 2 --steps 2000 --kplane" "--config C3 --order 2 --steps 200"; do
  echo "# $a" >> gpurun_out/r3r_bench.log
  timeout 300 $B $a >> gpurun_out/r3r_bench.log 2>&1
done
python scripts/bench_lines.py gpurun_out/r3r_bench.log
