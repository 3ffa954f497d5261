python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_materials.py tests/test_gpu_fuzz.py tests/test_gpu_problems.py -x -q 2>&1 | tail -2
for r in 1 2; do
  SALE_LIB_PATH=abtmp/libsale_head.so python bench.py --config C4 --steps 100 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('head', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernels_ms_per_step'].items() if k in ('lagrange','remap')})"
  python bench.py --config C4 --steps 100 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new ', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernels_ms_per_step'].items() if k in ('lagrange','remap')})"
done
