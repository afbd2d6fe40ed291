mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests9.log 2>&1; echo EXIT $? >> gpurun_out/gpu_tests9.log
B="python bench.py --no-cpu-baseline --no-e2e"
for a in "--config C3" "--config C3 --order 8" "--config C3 --order 4" "--config C2 --steps 2000" "--config C2 --order 4 --steps 2000" "--config C2 --order 8 --steps 2000" "--config C3 --kplane" "--config C3 --order 8 --kplane" "--config C2 --steps 2000 --kplane" "--config C2 --order 8 --steps 2000 --kplane"; do
  timeout 300 $B $a >> gpurun_out/bench9.log 2>&1
done
