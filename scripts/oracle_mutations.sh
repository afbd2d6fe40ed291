#!/bin/bash
# Mutation check of the oracle pins: each plausible mistake must fail a pin.
# Restores oracle/fd_oracle.c at the end.  Run: bash scripts/oracle_mutations.sh
set -u
cp /root/repo/oracle/fd_oracle.c /tmp/fd_oracle_orig.c
cd /root/repo
run_mut() {
  python - "$1" "$2" <<'PY'
import sys
s=open('/tmp/fd_oracle_orig.c').read()
a,b=sys.argv[1],sys.argv[2]
assert a in s, a
open('oracle/fd_oracle.c','w').write(s.replace(a,b,1))
PY
  out=$(timeout 600 python -m pytest tests/test_oracle_pins.py -q -x 2>&1 | tail -1)
  echo "MUT [$1 -> $2]: $out"
}
run_mut "dt2 * V[i] * V[i] * lap" "dt2 * V[i] * lap"
run_mut "2.0 * P[i] - Pold[i]" "2.0 * P[i] + Pold[i]"
run_mut "acc += c[m] * (P[i - m * s] + P[i + m * s]);" "acc += c[m] * (P[i - m * s] + P[i + (m-1) * s]);"
run_mut "if (i_a < r || i_a >= n_a - r)" "if (i_a < r || i_a > n_a - r)"
run_mut "T[(int64_t)j * nt + k] = cur[rl[j]];" "T[(int64_t)j * nt + k] = old[rl[j]];"
run_mut "src_amp[s] * oracle_ricker((double)k * dt," "src_amp[s] * oracle_ricker((double)(k+1) * dt,"
run_mut "*out = (iz * g->n[1] + iy) * g->n[0] + ix;" "*out = (ix * g->n[1] + iy) * g->n[0] + iz;"
run_mut "c[0] = -205.0 / 72.0;" "c[0] = -205.0 / 71.0;"
run_mut "return (1.0 - 2.0 * a) * exp(-a);" "return (1.0 - a) * exp(-a);"
run_mut "out[i] = acc / h2;" "out[i] = acc / h;"
run_mut "double *t = old; old = cur; cur = nxt; nxt = t;" "double *t = old; old = nxt; nxt = t;"
# sponge frame (R#18)
run_mut "const int64_t d = j < n - 1 - j ? j : n - 1 - j;" "const int64_t d = j < n - j ? j : n - j;"
run_mut "nxt[i] = G[i] * (2.0 * cur[i] - G[i] * old[i]" "nxt[i] = G[i] * (2.0 * cur[i] - old[i]"
run_mut "nxt[i] = G[i] * (2.0 * cur[i]" "nxt[i] = (2.0 * cur[i]"
run_mut "g[j] = exp(-(a * a));" "g[j] = exp(-a);"
run_mut "= gz[iz] * gy[iy] * gx[ix];" "= gz[iz] * gx[ix];"
cp /tmp/fd_oracle_orig.c oracle/fd_oracle.c
python -c "import oracle; oracle.build(force=True)"
