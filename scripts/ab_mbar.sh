run() {
  for spec in "C3 2 0" "C3 2 1" "C3 8 1" "C2 2 0" "C2 8 1"; do
    set -- $spec
    python bench.py --config $1 --order $2 --tsteps $3 --steps 600 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 o$2 t$3', round(d['value'],1), d['clocks']['sm_mhz'])"
  done
}
echo "== hint"; run
FD_NVCC_EXTRA=-DFD_MBAR_SUSPEND_NS=0 python -c "from __graft_entry__ import build_lib; build_lib(force=True)"
echo "== nohint"; run
