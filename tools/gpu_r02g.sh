mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "halo or c1 or two_species or supercell" > gpurun_out/pytest_halo.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_halo.log
bash tools/gpu_ab.sh "C3 C3:h2 C3:h2:k40 C2:h2 C2:h2:k40" cur
python tools/run_steps.py C3 6 > gpurun_out/ncu_plain.log 2>&1 && ncu --metrics ,l1tex__data_pipe_lsu_wavefronts_cmd_read.sum,l1tex__data_pipe_lsu_wavefronts_cmd_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_cmd_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_misc.sum --clock-control none -k regex:k_push_tile -s 3 -c 1 --csv python tools/run_steps.py C3 6 > gpurun_out/ncu_lsu_C3.csv 2>&1; echo "rc=$?"
