#!/bin/bash
# Build a variant of libpic.so with extra nvcc defines into exp/libpic_<name>.so
#   bash tools/build_variant.sh name "-DPIC_STAGE=1 -DPIC_BBOX=1"
set -e
name=$1; shift
defs="$*"
cd "$(dirname "$0")/.."
make -s build/diag.o build/fields.o build/push_naive.o build/runtime.o build/slab.o build/sort.o >/dev/null
mkdir -p exp build/var_$name
NCCL_INC=$(python3 -c "import os,nvidia.nccl as m; print(os.path.join(list(m.__path__)[0],'include'))")
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
  -Xptxas -v -cudart static --expt-relaxed-constexpr -I$NCCL_INC $defs \
  -c paper_1608_01009_b200/csrc/push_tile.cu -o build/var_$name/push_tile.o 2> build/var_$name/ptxas.log \
  || { grep -m5 error build/var_$name/ptxas.log; echo "BUILD FAILED: $name"; rm -f exp/libpic_$name.so; exit 1; }
grep -A1 'k_push_tileILi4' build/var_$name/ptxas.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | tr '\n' ' '; echo " <- $name"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o exp/libpic_$name.so \
  build/diag.o build/fields.o build/push_naive.o build/var_$name/push_tile.o build/runtime.o build/slab.o build/sort.o -ldl
