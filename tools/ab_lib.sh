#!/bin/bash
# Build an A/B variant of libgear.so with one kernel source recompiled under
# extra nvcc flags:  tools/ab_lib.sh <name> <kernel.cu> [nvcc flags...]
# -> paper_2310_05205_b200/ab/libgear_<name>.so (use with GEAR_LIB=...)
set -e
name=$1; src=$2; shift 2
ROOT=$(cd $(dirname $0)/.. && pwd)
NCCL=$(cd $ROOT && python -c "import paper_2310_05205_b200.build as b; print(b._nccl_dir())")
mkdir -p $ROOT/paper_2310_05205_b200/ab /tmp/ab_$name
base=$(basename $src)
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -Xcompiler -fPIC -lineinfo -gencode arch=compute_100a,code=sm_100a \
  -I $ROOT/include -I $NCCL/include -I $ROOT/paper_2310_05205_b200/csrc/kernels "$@" -c $src -o /tmp/ab_$name/$base.o
cd $ROOT/paper_2310_05205_b200/build
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../ab/libgear_$name.so \
  $(ls *.o | grep -v "^$base.o$") /tmp/ab_$name/$base.o -L $NCCL/lib -l:libnccl.so.2 -Xlinker -rpath,$NCCL/lib
echo paper_2310_05205_b200/ab/libgear_$name.so
