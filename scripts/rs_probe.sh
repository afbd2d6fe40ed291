#!/bin/bash
# Compile a few rs2d_step_kernel configurations (variant 0) with ptxas -v and
# summarise registers / spills:  scripts/rs_probe.sh 'make_rs2d<1,2,1,4,3,6,4>()' ...
set -e
CS=$(cd "$(dirname "$0")/../paper_2311_05038_b200/csrc" && pwd)
T=$(mktemp -d)
{
  echo '#define FD_TABLE_TU'
  echo '#include "fd_rs2d.cuh"'
  echo '#include "fd_tables.cuh"'
  echo 'FD_LAUNCHER(launch_rs2d, rs2d_step_kernel)'
  echo 'template <int R, int S, int HQ, int W, int Q, int MINB = 1, bool TMA = false>'
  echo 'static TileCfg make_rs2d() { using C = CfgRS2<R, S, HQ, W, Q, MINB, TMA>;'
  echo '  TileCfg t{2, R, C::TX, 1, W, Q, C::U, 64, 64, 8, 8, C::NTHREADS, C::SMEM_BYTES, {}, {}};'
  echo "  FD_VARIANT(t, C, rs2d_step_kernel, launch_rs2d, ${VARIANT:-0}); return t; }"
  echo "std::vector<TileCfg> probe() { return { $(IFS=,; echo "$*") }; }"
} > $T/p.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I$CS -I$CS/../../include -Xptxas -v \
  ${NVCC_EXTRA:-} -c -o $T/p.o $T/p.cu 2>&1 | tee $T/log | python "$(dirname "$0")/ptxas_summary.py" rs2d
[ -n "${SASS:-}" ] && cuobjdump -sass $T/p.o > "$SASS"
grep -m5 error $T/log || true
rm -rf $T
