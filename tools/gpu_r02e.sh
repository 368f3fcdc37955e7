bash tools/gpu_ab.sh "C2 C3 FROZEN" base acc384 noacc384 acc320
