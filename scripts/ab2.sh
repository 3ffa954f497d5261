#!/bin/bash
# A/B over env assignments: ./scripts/ab2.sh "A=1 B=2" "A=0 B=1" ...
for e in "$@"; do
  env $e python bench.py --config ${CFG:-C4} --steps 40 --warmup 3 --impl fused --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$e', '%.3e'%d['value'], {k:round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
done
