#!/usr/bin/env bash
# Build an experimental variant of libffst.so: bash scripts/variant.sh <tag> <-DMACRO ...>
# (recompiles only the float32 kernel unit; selected at run time with FFST_LIB=paper_1202_1773_b200/_variants/libffst_<tag>.so)
set -e
cd "$(dirname "$0")/.."
tag=$1; shift
P=paper_1202_1773_b200; V=$P/_variants; mkdir -p $V
NCCL=$(python -c "from paper_1202_1773_b200.build import NCCL; print(NCCL)")
nvcc -std=c++17 -O3 --expt-relaxed-constexpr -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
  -Xptxas -warn-spills -Iinclude -I$P/csrc -I$NCCL/include "$@" -c $P/csrc/ffst_kern_f32.cu -o $V/kern_f32_$tag.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a $P/_build/ffst_api.o $V/kern_f32_$tag.o $P/_build/ffst_kern_f64.o \
  $P/_build/ffst_gen_f32.o $P/_build/ffst_gen_f64.o -o $V/libffst_$tag.so -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib
echo built $V/libffst_$tag.so
