mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
timeout -k 10 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "fused_yee or fdtd or plane_wave or c1 or frozen" 2>&1 | tail -2
bash tools/gpu_ab.sh "C3 C2 C3:split" cur y8z4 y4z4 y8z8 y4z8
