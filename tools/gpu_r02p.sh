mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 2>&1 | tail -2
bash tools/gpu_ab.sh "C3 C2" wu sortsc
