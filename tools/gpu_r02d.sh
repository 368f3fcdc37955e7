bash tools/gpu_ab.sh "C2 C3 FROZEN" base noacc acc
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_parity_r02d.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/pytest_parity_r02d.log
