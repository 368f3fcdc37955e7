mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
./tools/bin/tmem_probe
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
bash tools/gpu_ab.sh "C3 C2 FROZEN" base notmem tmem
