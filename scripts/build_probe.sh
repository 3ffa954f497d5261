#!/bin/bash
# build lib/libsale_probe.so with one source recompiled under extra -D flags (timing probes only)
# usage: scripts/build_probe.sh kernels_fused.cu -DSALE_PROBE_NOLOAD
set -e
R=/root/repo; SRC=$1; shift
NCCL=$(python -c 'import nvidia,os;print(os.path.join(nvidia.__path__[0],"nccl"))')
OBJ=$R/paper_2209_01983_b200/lib/obj
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -I $R/include -I $R/paper_2209_01983_b200/csrc -I $NCCL/include "$@" -c $R/paper_2209_01983_b200/csrc/$SRC -o /tmp/probe_${SRC%.cu}.o
objs=""; for o in $OBJ/*.o; do b=$(basename $o); [ "$b" = "${SRC%.cu}.o" ] || objs="$objs $o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/paper_2209_01983_b200/lib/libsale_probe.so $objs /tmp/probe_${SRC%.cu}.o -L $NCCL/lib -l:libnccl.so.2 -Xlinker -rpath,$NCCL/lib
echo built probe
