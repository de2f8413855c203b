# Round-2 sixth session: time-to-tolerance of the randomized methods at c3 and the capped c2 probes at HEAD
# (after the 16-CTA cluster SP-RK-RGS kernel at c3 and the tree SP setup).
set -x
timeout 900 python tools/probe_perf.py --config c3 --methods sp,rk,rgs,rcd --reps 1 --max-inner 2000000 > gpurun_out/r2h_c3_converge.log 2>&1; echo c3=$?
timeout 600 python tools/probe_perf.py --config c2 --methods rk,rgs,rcd --reps 1 --max-iter 2 --max-inner 20000 > gpurun_out/r2h_c2_capped.log 2>&1; echo c2cap=$?
ILS_RK_PROF=1 timeout 600 python tools/probe_perf.py --config c2 --methods rk --reps 1 --max-iter 1 --max-inner 20000 > gpurun_out/r2h_c2_prof.log 2>&1; echo c2prof=$?
