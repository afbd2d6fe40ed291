#!/bin/bash
# A/B of the r >= 3 queue-shift period kQShift (fd_kernels.cuh) on C3 orders 6 / 8
mkdir -p gpurun_out
for u in 1 2 3 4; do
  FD_NVCC_EXTRA=-DFD_QSHIFT=$u python -c "import __graft_entry__ as g; g.build_lib(force=True)" > /dev/null 2>&1
  for a in "--order 8" "--order 6" "--order 8"; do
    echo "u=$u $a" >> gpurun_out/ab_qshift.log
    timeout 300 python bench.py --config C3 $a --no-cpu-baseline --no-e2e --sustained 0 >> gpurun_out/ab_qshift.log 2>&1
  done
done
python -c "import __graft_entry__ as g; g.build_lib(force=True)" > /dev/null 2>&1
