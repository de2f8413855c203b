# cols_tile_kernel: CTAs-per-SM sweep at c3 and the launch list of the new solve
set -x
for c in 4 8 16 32; do ILS_COLS_CPS=$c timeout 600 python tools/probe_perf.py --config c3 --methods sp --reps 3 > gpurun_out/cols_cps$c.log 2>&1; echo cps$c=$?; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches_c3sp2.csv python tools/probe_perf.py --config c3 --methods sp --reps 1 > gpurun_out/r2i_c3sp2.log 2>&1; echo rc=$?
