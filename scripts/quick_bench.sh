#!/bin/bash
# quick perf check of both workloads (no cpu baseline, 1 e2e step)
python bench.py --steps ${STEPS:-60} --warmup 3 --impl ${IMPL:-fused} --no-cpu-baseline --e2e-steps 1 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('C4', '%.3e'%d['value'], 'ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
python bench.py --config C3 --steps ${STEPS:-40} --warmup 3 --impl ${IMPL:-fused} --no-cpu-baseline --e2e-steps 1 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('C3', '%.3e'%d['value'], 'ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
