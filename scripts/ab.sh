#!/bin/bash
# A/B: run C4 bench for each value of an env var: ./scripts/ab.sh VAR v1 v2 ...
var=$1; shift
for v in "$@"; do
  env $var=$v python bench.py --config ${CFG:-C4} --steps ${STEPS:-40} --warmup 3 --impl fused --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$var=$v', '%.3e'%d['value'], {k:round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
done
