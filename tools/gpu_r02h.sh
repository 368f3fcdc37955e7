mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/dbg_h2.py 2>&1 | tail -5
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all_r02h.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_all_r02h.log
bash tools/gpu_ab.sh "C3 C3:k40 C2 FROZEN" cur
