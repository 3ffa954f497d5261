#!/bin/bash
# Build abtmp/libsale_<tag>.so from ALL current sources under extra -D flags (A/B runs
# of header-level switches; build_probe.sh recompiles one source only).
# usage: scripts/build_variant.sh <tag> -DSALE_ZPLAN=0 ...
set -e
R=/root/repo; TAG=$1; shift
NCCL=$(cd $R/paper_2209_01983_b200 && python -c "import build,os; print(os.path.dirname(build.nccl_dirs()[0]))")
O=/tmp/variant_$TAG; mkdir -p $O $R/abtmp
for f in $R/paper_2209_01983_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC \
    -I $R/include -I $R/paper_2209_01983_b200/csrc -I $NCCL/include "$@" -c $f -o $O/$(basename ${f%.cu}).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/abtmp/libsale_${TAG}.so $O/*.o \
    -L $NCCL/lib -l:libnccl.so.2 -Xlinker -rpath,$NCCL/lib
echo built abtmp/libsale_${TAG}.so
