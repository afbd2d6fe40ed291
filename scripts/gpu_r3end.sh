set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_fulllength.py > gpurun_out/r3e_pytest_all.log 2>&1
tail -2 gpurun_out/r3e_pytest_all.log
FD_PARITY_LOG=gpurun_out/parity_fulllength_r3d.jsonl timeout 1200 python -m pytest -q tests/test_gpu_fulllength.py -k "C2" > gpurun_out/r3e_fulllength.log 2>&1
tail -1 gpurun_out/r3e_fulllength.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3e_smoke.log 2>&1; echo "smoke rc=$?"
B="python bench.py --no-cpu-baseline --no-e2e --sustained 0"
: > gpurun_out/r3e_bench.log
for a in "--config C2 --order 2 --steps 2000" "--config C2 --order 4 --steps 2000" "--config C2 --order 6 --steps 2000" "--config C2 --order 2 --steps 2000 --kplane"; do
  echo "# $a" >> gpurun_out/r3e_bench.log
  timeout 300 $B $a >> gpurun_out/r3e_bench.log 2>&1
done
python scripts/bench_lines.py gpurun_out/r3e_bench.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r3e_bench_default.log 2>&1; tail -1 gpurun_out/r3e_bench_default.log | cut -c1-120
