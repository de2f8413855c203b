# launch list of one c3 SP solve (setup + 6 outer steps): which kernels carry the 10.6 ms solve
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches_c3sp.csv python tools/probe_perf.py --config c3 --methods sp --reps 1 > gpurun_out/r2i_c3sp.log 2>&1; echo rc=$?
