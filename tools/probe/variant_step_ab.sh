#!/bin/bash
# In-step A/B of library variants at config 5: alternating bench runs (one process each),
# value and per-stage times.  usage: variant_step_ab.sh ROUNDS VAR1 VAR2 ...  ("-" = product build)
R=${1:-3}; shift
for i in $(seq $R); do for v in "$@"; do
  vv=$v; [ "$v" = "-" ] && vv=""; ee="ENKF_UNUSED=1"; case "$v" in *=*) ee="$v"; vv="";; esac
  env "$ee" ENKF_LIB_VARIANT=$vv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('variant=$v', round(d['value'],2), {k:round(x,2) for k,x in d['kernels_ms'].items()}, d.get('energy_j_per_step'), d['clocks']['sm_mhz'])"
done; done
