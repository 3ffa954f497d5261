#!/bin/bash
# One gpurun call: bench lines (C4 default, C3), reference arm, launch list, and the
# ncu --set full captures the traffic files come from.  Output: gpurun_out/$TAG/
TAG=${TAG:-m}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --config C3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference.json 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/ncu_launch.log 2>&1
python scripts/prof_run.py C4 fused 3 > $O/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"kf_|kr_|kn_" -s 6 -c 6 -o $O/full_c4 \
    python scripts/prof_run.py C4 fused 3 > $O/ncu_full_c4.log 2>&1
python scripts/prof_run.py C3 fused 3 > $O/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"kf_" -s 2 -c 2 -o $O/full_c3 \
    python scripts/prof_run.py C3 fused 3 > $O/ncu_full_c3.log 2>&1
tail -c 300 $O/bench_c4.json; echo; tail -c 300 $O/bench_c3.json; echo; tail -c 200 $O/bench_reference.json
