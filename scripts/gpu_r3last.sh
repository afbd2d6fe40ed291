set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_fulllength.py > gpurun_out/r3l_pytest_all.log 2>&1
tail -2 gpurun_out/r3l_pytest_all.log
KREGEX=rs2d KSKIP=2 SPECS="C2:2:4" TAG=r3b bash scripts/gpu_profile.sh > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3l_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/r3l_bench_default.log 2>&1; tail -1 gpurun_out/r3l_bench_default.log | cut -c1-160
