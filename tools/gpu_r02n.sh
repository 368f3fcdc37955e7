mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
bash tools/gpu_ab.sh "C3 C2 FROZEN" cur wu cur wu
