#!/bin/bash
# Build the whole libpic with extra nvcc defines into exp/libpic_<name>.so
#   bash tools/build_full_variant.sh name "-DPIC_GHOST=3"
set -e
name=$1; shift
defs="$*"
cd "$(dirname "$0")/.."
mkdir -p exp build/full_$name
NCCL_INC=$(python3 -c "import os,nvidia.nccl as m; print(os.path.join(list(m.__path__)[0],'include'))")
objs=""
for f in paper_1608_01009_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
    -Xptxas -v -cudart static --expt-relaxed-constexpr -I$NCCL_INC $defs -c $f -o build/full_$name/$b.o 2> build/full_$name/$b.ptxas.log &
  objs="$objs build/full_$name/$b.o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o exp/libpic_$name.so $objs -ldl
echo "built exp/libpic_$name.so"
