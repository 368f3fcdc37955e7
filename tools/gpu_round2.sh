#!/bin/bash
# Round-2 measurement pass on one B200 (run under gpurun):
#   bash tools/gpu_round2.sh TAG
# GPU test suite, smoke, the default bench (C3) three times, the other
# workloads, the reference arm, the ncu launch list of the default bench
# command, and the per-launch ncu counts (DRAM, fp64, data pipe) per workload.
tag=${1:-final}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt
nproc >> $out/gpu.txt; grep -m1 "model name" /proc/cpuinfo >> $out/gpu.txt
timeout -k 10 2400 python -m pytest tests -m gpu -q --timeout 900 -rA -s > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $out/smoke.log
for r in 1 2 3; do
  timeout -k 10 900 python bench.py > $out/bench_C3_$r.json 2> $out/bench_C3_$r.err; echo "bench C3 $r rc=$?"
done
for w in C2 FROZEN C5_1g; do
  timeout -k 10 900 python bench.py --workload $w --no-cpu-baseline > $out/bench_$w.json 2> $out/bench_$w.err; echo "bench $w rc=$?"
done
timeout -k 10 1200 python bench.py --workload C4 --steps 40 --no-cpu-baseline --no-e2e > $out/bench_C4.json 2> $out/bench_C4.err; echo "bench C4 rc=$?"
timeout -k 10 900 python bench.py --impl reference --steps 20 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?"
timeout -k 10 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $out/plain_launch.log 2>&1 && \
timeout -k 10 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1; echo "launches rc=$?"
M=dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,l1tex__data_pipe_lsu_wavefronts.sum
for w in C3 C2 FROZEN C5_1g; do
  timeout -k 10 600 ncu --metrics $M --clock-control none -k regex:k_push_tile -s 3 -c 1 --csv python tools/run_steps.py $w 6 > $out/ncu_counts_$w.csv 2>&1; echo "ncu $w rc=$?"
done
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:k_push_tile -s 3 -c 1 -o $out/prof_C3 python tools/run_steps.py C3 6 > $out/ncu_full_C3.log 2>&1; echo "ncu full rc=$?"
