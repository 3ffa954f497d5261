#!/bin/bash
# Build abtmp/libsale_<tag>.so with one source recompiled under extra -D flags, for
# A/B timing runs only (SALE_LIB_PATH=abtmp/libsale_<tag>.so python bench.py ...).
# usage: scripts/build_probe.sh <tag> kernels_lag.cu -DSALE_NW_FORCE=16 ...
#        (SRCPATH=/path/to/a/variant.cu replaces that source with another file)
set -e
R=/root/repo; TAG=$1; SRC=$2; shift 2
NCCL=$(cd $R/paper_2209_01983_b200 && python -c "import build,os; print(os.path.dirname(build.nccl_dirs()[0]))")
OBJ=$R/paper_2209_01983_b200/lib/obj
mkdir -p $R/abtmp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC \
    -I $R/include -I $R/paper_2209_01983_b200/csrc -I $NCCL/include "$@" \
    -c ${SRCPATH:-$R/paper_2209_01983_b200/csrc/$SRC} -o /tmp/probe_${TAG}.o
objs=""; for c in $R/paper_2209_01983_b200/csrc/*.cu; do b=$(basename ${c%.cu}).o; [ "$b" = "${SRC%.cu}.o" ] || objs="$objs $OBJ/$b"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/abtmp/libsale_${TAG}.so $objs /tmp/probe_${TAG}.o \
    -L $NCCL/lib -l:libnccl.so.2 -Xlinker -rpath,$NCCL/lib
echo built abtmp/libsale_${TAG}.so
