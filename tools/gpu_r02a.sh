mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_r02a.txt
nproc >> gpurun_out/gpu_r02a.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/gpu_r02a.txt; free -g >> gpurun_out/gpu_r02a.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_open.py -m gpu -x -q -s > gpurun_out/pytest_new_r02a.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_new_r02a.log
timeout 900 python bench.py > gpurun_out/bench_default_r02a.json 2> gpurun_out/bench_default_r02a.err; echo "bench rc=$?"
