#!/bin/bash
# ncu --set full of the fused kernel of a variant library (exp/libpic_<v>.so):
#   bash tools/ncu_variant.sh <variant> <workload> [launch-skip]
v=$1; wl=${2:-C3}; skip=${3:-3}
mkdir -p gpurun_out
cp paper_1608_01009_b200/libpic.so /tmp/cur.so
cp exp/libpic_$v.so paper_1608_01009_b200/libpic.so
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_push_tile -s $skip -c 1 \
  -o gpurun_out/prof_${v}_$wl python tools/run_steps.py $wl 8 > gpurun_out/ncu_${v}_$wl.log 2>&1
echo "ncu $v $wl rc=$?"
cp /tmp/cur.so paper_1608_01009_b200/libpic.so
