mkdir -p gpurun_out/r02l
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02l/gpu.txt
timeout -k 10 2400 python -m pytest tests -m gpu -q --timeout 900 -rA > gpurun_out/r02l/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02l/pytest_gpu.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02l/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02l/smoke.log
timeout -k 10 900 python bench.py > gpurun_out/r02l/bench_C3.json 2> gpurun_out/r02l/bench_C3.err; echo "bench rc=$?"
M=dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
for w in C3 C2 FROZEN C5_1g; do
  timeout -k 10 600 ncu --metrics $M --clock-control none -k regex:k_push_tile -s 3 -c 1 --csv python tools/run_steps.py $w 6 > gpurun_out/r02l/ncu_counts_$w.csv 2>&1; echo "ncu $w rc=$?"
done
