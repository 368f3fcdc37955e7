mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
timeout -k 10 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_diag.py tests/test_gpu_fullsize.py -m gpu -x -q --timeout 600 -s 2>&1 | grep -E "passed|failed|Error|^C[0-9]|FAIL" | tail -12
bash tools/gpu_ab.sh "C3 C3:split C2 C2:split FROZEN FROZEN:split" cur
