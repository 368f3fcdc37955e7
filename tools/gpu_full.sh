#!/bin/bash
# Round-end style run: tests, smoke, default bench (with cpu baseline), reference arm,
# C3 bench, and the ncu launch list of the bench command.
tag=${1:-full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$tag.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$tag.log
timeout 900 python bench.py > gpurun_out/bench_default_$tag.json 2> gpurun_out/bench_default_$tag.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err; echo "ref rc=$?"
timeout 900 python bench.py --workload C3 --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C3_$tag.json 2> gpurun_out/bench_C3_$tag.err; echo "C3 rc=$?"
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_launch_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$tag.log 2>&1; echo "ncu launches rc=$?"
timeout 900 python bench.py --workload C5_1g --steps 100 --warmup 5 > gpurun_out/bench_C5_1g_$tag.json 2> gpurun_out/bench_C5_1g_$tag.err; echo "C5_1g rc=$?"
timeout 900 python bench.py --workload FROZEN --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_frozen_$tag.json 2> gpurun_out/bench_frozen_$tag.err; echo "FROZEN rc=$?"
python tools/run_steps.py C3 8 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_push_tile -s 3 -c 1 -o gpurun_out/prof_C3_$tag python tools/run_steps.py C3 8 > gpurun_out/ncu_C3_$tag.log 2>&1; echo "ncu C3 rc=$?"
python tools/run_steps.py C2 25 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_push_tile -s 3 -c 1 -o gpurun_out/prof_C2_$tag python tools/run_steps.py C2 25 > gpurun_out/ncu_C2_$tag.log 2>&1; echo "ncu C2 rc=$?"
timeout 1200 python bench.py --workload C4 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_$tag.json 2> gpurun_out/bench_C4_$tag.err; echo "C4 rc=$?"
