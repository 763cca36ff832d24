#!/bin/bash
# A/B build of libellwarp_b200.so with extra nvcc flags for ew_spmv.cu only:
#   tools/ab_build.sh NAME "-DMACRO=VALUE ..."  ->  scratch/ab/NAME.so
# (the other objects from paper_1501_00324_b200/_build; run make first).
# Use with EW_B200_LIB=scratch/ab/NAME.so.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
P=$ROOT/paper_1501_00324_b200
mkdir -p $ROOT/scratch/ab
NCCL_INC=$(python -c "import os,nvidia.nccl as m;print(os.path.join(list(m.__path__)[0],'include'))" 2>/dev/null || echo /usr/include)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC \
  -I$ROOT/include -I$NCCL_INC --expt-relaxed-constexpr $2 -c $P/csrc/ew_spmv.cu -o $ROOT/scratch/ab/$1_spmv.o
OBJS=$(ls $P/_build/ew_*.o | grep -v ew_spmv.o)
g++ -shared -o $ROOT/scratch/ab/$1.so $OBJS $ROOT/scratch/ab/$1_spmv.o -L/usr/local/cuda/lib64 -lcudart_static -lrt -ldl \
  -lpthread -nostdlib++ /usr/lib/x86_64-linux-gnu/libstdc++.so.6
echo built $ROOT/scratch/ab/$1.so
