#!/bin/bash
# A/B the variants exp/libpic_<v>.so (tools/build_variant.sh) on the GPU box:
#   bash tools/ab.sh "C2 C3" v1 v2 ...   -> gpurun_out/ab.txt
wls=$1; shift
mkdir -p gpurun_out
cp paper_1608_01009_b200/libpic.so /tmp/cur.so
for v in "$@"; do
  if [ ! -f exp/libpic_$v.so ]; then echo "$v missing" | tee -a gpurun_out/ab.txt; continue; fi
  cp exp/libpic_$v.so paper_1608_01009_b200/libpic.so
  timeout -k 5 120 python -c "import __graft_entry__ as g; g.smoke()" > /tmp/smoke_$v.log 2>&1 && sm=ok || sm=FAIL
  for w in $wls; do
    r=$(timeout -k 5 600 python tools/ab_run.py $w 40 2>/tmp/ab_err_$v_$w.log | tail -1)
    echo "$v $w smoke=$sm $r" | tee -a gpurun_out/ab.txt
  done
done
cp /tmp/cur.so paper_1608_01009_b200/libpic.so
