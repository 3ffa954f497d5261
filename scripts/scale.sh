#!/bin/bash
# Weak-scaling bench lines (C4: 256^3 cells per GPU) at N = 1, 2, 4, 8 GPUs of one node,
# one JSON line per N, with NCCL's INFO log kept per N so the communicator's rank count,
# transport (P2P / NVLS) and ring / tree setup are visible.
#   usage: [HALO=copy|peer] scripts/scale.sh [steps] [warmup] [config C4|C3]   -> gpurun_out/scale_<cfg>.jsonl
#   (HALO=peer: the producing kernels store the ghost planes into the neighbours over NVLink)
cd "$(dirname "$0")/.."
STEPS=${1:-50}; WARM=${2:-5}; CFG=${3:-C4}; HALO=${HALO:-copy}
NG=$(python -c "import torch; print(torch.cuda.device_count())")
OUT=gpurun_out/scale_${CFG}_${HALO}.jsonl; mkdir -p gpurun_out; : > $OUT
for N in 1 2 4 8; do
  [ "$N" -le "$NG" ] || break
  if [ "$N" = 1 ]; then
    python bench.py --config $CFG --steps $STEPS --warmup $WARM --no-cpu-baseline --e2e-steps 0 | tail -1 >> $OUT
  else
    NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,GRAPH python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --config $CFG --steps $STEPS \
      --warmup $WARM --no-cpu-baseline --e2e-steps 0 --halo $HALO 2> gpurun_out/scale_${CFG}_${HALO}_n${N}.nccl.log | tail -1 >> $OUT
  fi
done
cat $OUT
