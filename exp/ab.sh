cp paper_1608_01009_b200/libpic.so /tmp/cur.so
for v in base b1; do
  cp exp/libpic_$v.so paper_1608_01009_b200/libpic.so
  for w in C2 C3; do
    timeout 600 python bench.py --workload $w --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$w.json 2>gpurun_out/ab_${v}_$w.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$w.json'));print('$v $w', round(d['roofline']['avg_launch_ms'],4), round(d['value']/1e9,2))"
  done
done
cp /tmp/cur.so paper_1608_01009_b200/libpic.so
