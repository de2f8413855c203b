set -x
timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 3 > gpurun_out/u2_base.log 2>&1; echo base=$?
ILS_RK_U=2 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 3 > gpurun_out/u2_u2.log 2>&1; echo u2=$?
ILS_RK_U=2 ILS_RK_NAP=150 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 3 > gpurun_out/u2_u2nap150.log 2>&1; echo u2n=$?
ILS_RK_U=2 ILS_RK_PROF=1 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 > gpurun_out/u2_u2prof.log 2>&1; echo u2p=$?
ILS_RK_PROF=1 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 > gpurun_out/u2_baseprof.log 2>&1; echo bp=$?
