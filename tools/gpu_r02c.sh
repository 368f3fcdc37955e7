mkdir -p gpurun_out
./tools/bin/mb_smem > gpurun_out/mb_smem.json 2>&1; echo "mb rc=$?"; cat gpurun_out/mb_smem.json
ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_atom.sum,smsp__inst_executed.sum --csv ./tools/bin/mb_smem > gpurun_out/mb_smem_ncu.csv 2>&1; echo "ncu rc=$?"
