set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_fulllength.py > gpurun_out/r3f_pytest_all.log 2>&1
tail -3 gpurun_out/r3f_pytest_all.log
FD_PARITY_LOG=gpurun_out/parity_fulllength_r3c.jsonl timeout 2400 python -m pytest -q tests/test_gpu_fulllength.py > gpurun_out/r3f_fulllength.log 2>&1
tail -2 gpurun_out/r3f_fulllength.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3f_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/r3f_bench_default.log 2>&1; tail -1 gpurun_out/r3f_bench_default.log | cut -c1-200
