# ncu --set full of the SP row-stream kernel at c2 (new grid barrier) and of the tiled transposed GEMV at c3
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sp_persistent_kernel" -s 1 -c 1 -o gpurun_out/r2i_prof_c2sp python tools/sp_one_solve.py > gpurun_out/r2i_ncu_c2sp.log 2>&1; echo ncu_c2sp=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cols_tile_kernel" -s 14 -c 1 -o gpurun_out/r2i_prof_c3cols python tools/probe_perf.py --config c3 --methods sp --reps 1 > gpurun_out/r2i_ncu_c3cols.log 2>&1; echo ncu_c3cols=$?
