#!/bin/bash
# GPU iteration script (run under gpurun): parity tests, bench, optional ncu.
#   bash tools/gpu_check.sh [tag] [ncu-kernel-regex] [workload]
tag=${1:-run}
kern=${2:-}
wl=${3:-C2}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$tag.log
timeout 900 python bench.py --steps 100 --warmup 5 --workload $wl --no-cpu-baseline > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench rc=$?"; cat gpurun_out/bench_$tag.json | python -c "
import json,sys
d=json.loads(sys.stdin.read())
r=d['roofline']
print('value %.3e upd/s  ms/step %.4f  particle ms %.4f  frac %.3f  stage %s e2e %.3e' % (d['value'], d['ms_per_step'], r['avg_launch_ms'], r['frac'], r['stage_ms_per_step'], d['e2e']['value']))
" ; tail -2 gpurun_out/bench_$tag.err
if [ -n "$kern" ]; then
  python tools/run_steps.py $wl 25 > gpurun_out/plain_$tag.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$kern -s 3 -c 1 -o gpurun_out/prof_$tag python tools/run_steps.py $wl 25 > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu rc=$?"; tail -2 gpurun_out/ncu_$tag.log
fi
