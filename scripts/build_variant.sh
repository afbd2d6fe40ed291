#!/bin/bash
# Build an A/B variant of libfd.so next to the default one (here, on the CPU):
#   bash scripts/build_variant.sh NAME "-DFLAG=0 ..."  -> paper_2311_05038_b200/libfd_NAME.so
# (run scripts/ab.sh on the GPU box with FD_LIB pointing at each variant)
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
FD_NVCC_EXTRA="$*" python -c "
import __graft_entry__ as g; g.build_lib(force=True)"
cp paper_2311_05038_b200/libfd.so paper_2311_05038_b200/libfd_${NAME}.so
echo built paper_2311_05038_b200/libfd_${NAME}.so with "$*"
