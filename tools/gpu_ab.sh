#!/bin/bash
# usage: bash tools/gpu_ab.sh "C2 C3 FROZEN" v1 v2 ...  (variants exp/libpic_<v>.so), then parity
wls=$1; shift
mkdir -p gpurun_out
rm -f gpurun_out/ab.txt
bash tools/ab.sh "$wls" "$@"
