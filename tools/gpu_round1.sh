set -x
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/host.txt; nproc >> gpurun_out/host.txt; lscpu | grep -i "model name" >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
timeout 120 ./build/microbench > gpurun_out/micro.json 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/micro.json gpurun_out/smoke.log gpurun_out/bench.json; tail -5 gpurun_out/bench.err
