mkdir -p gpurun_out
./tools/bin/mb_tex > gpurun_out/mb_tex.json 2>&1
ncu --metrics l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_tex_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__f_wavefronts.sum,gpu__time_duration.sum --csv ./tools/bin/mb_tex > gpurun_out/mb_tex_ncu.csv 2>&1
