# fill-warp look-ahead of the look-ahead RK-RGS kernel (Gram ring 32 blocks, lead 16 vs 24) at c1,
# phase profile of the c2 gmode blocked kernel
set -x
ILS_RK_LEAD=16 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 3 > gpurun_out/lead16.log 2>&1; echo l16=$?
ILS_RK_LEAD=24 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 3 > gpurun_out/lead24.log 2>&1; echo l24=$?
ILS_RK_LEAD=24 ILS_RK_NAP=100 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 3 > gpurun_out/lead24n100.log 2>&1; echo l24n=$?
ILS_RK_LEAD=24 ILS_RK_PROF=1 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 > gpurun_out/lead24prof.log 2>&1; echo l24p=$?
ILS_RK_PROF=1 timeout 600 python tools/probe_perf.py --config c2 --methods rk --reps 1 --max-iter 1 --max-inner 20000 > gpurun_out/c2prof.log 2>&1; echo c2p=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rk" > gpurun_out/lead_t1.log 2>&1; echo t1=$?
