#!/bin/bash
# One GPU call after a kernel change (run under gpurun): the -m gpu suite minus
# the slow full-length parity file, then short bench lines of the headline
# configurations.  TAG names the outputs under gpurun_out/.
#   TAG=r2c bash scripts/quick_check.sh
set -u
TAG=${TAG:-quick}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_fulllength.py ${PYTEST_EXTRA:-} \
    > gpurun_out/${TAG}_pytest.log 2>&1
tail -5 gpurun_out/${TAG}_pytest.log
B="python bench.py --no-cpu-baseline --no-e2e --sustained 0"
: > gpurun_out/${TAG}_bench.log
for a in ${BENCH_CASES:-"--config C3 --order 2" "--config C2 --order 2 --steps 2000" "--config C2 --order 4 --steps 2000"}; do
  echo "# $a" >> gpurun_out/${TAG}_bench.log
  timeout 300 $B $a >> gpurun_out/${TAG}_bench.log 2>&1
done
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
case = None
for ln in open(f"gpurun_out/{tag}_bench.log"):
    if ln.startswith("# "):
        case = ln[2:].strip()
    elif ln.startswith("{"):
        d = json.loads(ln)
        r = d["repetitions"]
        print(f"{case:45s} value {d['value']:7.1f} (min {r['value_min']:.1f} max {r['value_max']:.1f}) "
              f"frac {d['roofline']['frac']:.3f} {d['roofline']['kernel']} clocks {d['clocks'].get('sm_mhz')}")
PY
