mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
cp paper_1608_01009_b200/libpic.so /tmp/keep.so
cp exp/libpic_pers.so paper_1608_01009_b200/libpic.so
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 2>&1 | tail -2
cp /tmp/keep.so paper_1608_01009_b200/libpic.so
bash tools/gpu_ab.sh "C3 C2 FROZEN" wu pers nopers
