mkdir -p gpurun_out/r02m
M=dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,l1tex__data_pipe_lsu_wavefronts.sum
for w in C3 C2 FROZEN C5_1g; do
  timeout -k 10 600 ncu --metrics $M --clock-control none -k regex:k_push_tile -s 3 -c 1 --csv python tools/run_steps.py $w 6 > gpurun_out/r02m/ncu_counts_$w.csv 2>&1; echo "ncu $w rc=$?"
done
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:k_push_tile -s 3 -c 1 -o gpurun_out/r02m/prof_C3 python tools/run_steps.py C3 6 > gpurun_out/r02m/ncu_full_C3.log 2>&1; echo "ncu full rc=$?"
timeout -k 10 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02m/plain_launch.log 2>&1 && \
timeout -k 10 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02m/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02m/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout -k 10 1200 python tools/sweep.py C3 40 > gpurun_out/r02m/sweep_C3.md 2> gpurun_out/r02m/sweep_C3.err; echo "sweep C3 rc=$?"
timeout -k 10 900 python tools/sweep.py C2 40 > gpurun_out/r02m/sweep_C2.md 2> gpurun_out/r02m/sweep_C2.err; echo "sweep C2 rc=$?"
for w in C2 FROZEN C5_1g; do
  timeout -k 10 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r02m/bench_$w.json 2> gpurun_out/r02m/bench_$w.err; echo "bench $w rc=$?"
done
timeout -k 10 1200 python bench.py --workload C4 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/r02m/bench_C4.json 2> gpurun_out/r02m/bench_C4.err; echo "bench C4 rc=$?"
