set -x
ILS_RK_PROF=1 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 > gpurun_out/fillprof.log 2>&1; echo p=$?
ILS_RK_PROF=1 ILS_RK_NAP=0 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 > gpurun_out/fillprof_nap0.log 2>&1; echo p=$?
