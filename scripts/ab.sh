#!/bin/bash
# A/B of library variants on the GPU box (gpurun): bench.py value pass only,
# short runs (below the ~0.3 s after which the 1 kW power cap engages),
# variants interleaved ROUNDS times.  VARIANTS = names of libfd_NAME.so ("" =
# the default libfd.so); CASES = bench argument sets separated by ';'.
#   VARIANTS="O A B" CASES="--config C3 --steps 200;--config C2 --steps 1000" bash scripts/ab.sh
set -u
mkdir -p gpurun_out
TAG=${TAG:-ab}
ROUNDS=${ROUNDS:-3}
out=gpurun_out/${TAG}.log
: > $out
IFS=';' read -ra CS <<< "${CASES}"
for r in $(seq 1 $ROUNDS); do
  for c in "${CS[@]}"; do
    for v in ${VARIANTS}; do
      # a variant is a library name (libfd_NAME.so; "default" = libfd.so) or
      # env:VAR=VALUE (the default library with that environment variable)
      lib=paper_2311_05038_b200/libfd_${v}.so
      envs=""
      [ "$v" = "default" ] && lib=paper_2311_05038_b200/libfd.so
      case "$v" in env:*) lib=paper_2311_05038_b200/libfd.so; envs="${v#env:}";; esac
      echo "# $v | $c" >> $out
      env $envs FD_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --sustained 0 --reps 5 $c >> $out 2>&1
    done
  done
done
python scripts/ab_summary.py $out
