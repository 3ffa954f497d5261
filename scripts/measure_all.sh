#!/bin/bash
# One gpurun call: the default bench line (C4 + its C3 / P0 / golden legs), the
# reference arm, the launch lists, the ncu --set full captures the traffic files come
# from, material and Steinberg throughput.  Output: gpurun_out/$TAG/
TAG=${TAG:-m}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --config C3 --no-cpu-baseline --no-extras > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference.json 2>&1
python scripts/materials_bench.py $O/materials.json > $O/materials.log 2>&1
python scripts/steinberg_bench.py $O/steinberg.json > $O/steinberg.log 2>&1
for C in C4 C3; do
  python scripts/prof_run.py $C 4 > $O/plain_$C.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$C.csv \
      python scripts/prof_run.py $C 4 > $O/ncu_launch_$C.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"kc_|ke_|kl_|kr_|kn_" -s 6 -c 6 -o $O/full_c4 \
    python scripts/prof_run.py C4 4 > $O/ncu_full_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"kc_|kl_" -s 3 -c 3 -o $O/full_c3 \
    python scripts/prof_run.py C3 4 > $O/ncu_full_c3.log 2>&1
tail -c 300 $O/bench_c4.json; echo; tail -c 300 $O/bench_c3.json; echo; tail -c 200 $O/bench_reference.json
