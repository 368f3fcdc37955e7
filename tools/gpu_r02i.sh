mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
cp paper_1608_01009_b200/libpic.so /tmp/keep.so
for v in g2 g3; do
  cp exp/libpic_$v.so paper_1608_01009_b200/libpic.so
  echo "== $v"; CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/dbg_h2.py 2>&1 | tail -4
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_diag.py -m gpu -x -q -k "slab or halo or diag or c1 or supercell" 2>&1 | tail -2
done
cp /tmp/keep.so paper_1608_01009_b200/libpic.so
bash tools/gpu_ab.sh "C3 C2 FROZEN" g2 g3
