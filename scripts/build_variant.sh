#!/bin/bash
# Builds an experiment variant of libpmf_gpu.so with one translation unit recompiled under extra flags:
#   scripts/build_variant.sh NAME SRC.cu "-DMACRO=1 ..."  ->  scripts/_variants/libpmf_gpu_NAME.so
# (timing experiments only; on the GPU box copy it over paper_1511_02433_b200/libpmf_gpu.so)
set -e
HERE=$(cd "$(dirname "$0")/.." && pwd)
PKG=$HERE/paper_1511_02433_b200
NAME=$1; SRC=$2; FLAGS=$3
NCCL=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl
mkdir -p $HERE/scripts/_variants /tmp/pmfvar
BASE=$(basename $SRC .cu)
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-pthread,-O3 \
    -I$NCCL/include --expt-relaxed-constexpr $FLAGS -c $PKG/csrc/$SRC -o /tmp/pmfvar/$BASE.o
OBJS=$(ls $PKG/build/*.o | grep -v "/$BASE.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $HERE/scripts/_variants/libpmf_gpu_$NAME.so $OBJS /tmp/pmfvar/$BASE.o \
    -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath,$NCCL/lib -lpthread
echo built scripts/_variants/libpmf_gpu_$NAME.so
