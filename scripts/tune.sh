#!/bin/bash
# sweep SALE_TUNE="nw_force,nw_energy,zchunk" on C3 and C4
for t in "$@"; do
  for cfg in C3 C4; do
    SALE_TUNE=$t python bench.py --config $cfg --steps 30 --warmup 3 --impl fused --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$t', '$cfg', '%.3e'%d['value'], 'lag %.3f'%d['kernels_ms_per_step']['lagrange'])"
  done
done
