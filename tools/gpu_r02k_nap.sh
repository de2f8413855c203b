# look-ahead RK-RGS: helper-warp poll sleep (ILS_RK_NAP ns) re-swept at HEAD
set -x
for v in 300 150 600 1000 300; do ILS_RK_NAP=$v timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 3 > gpurun_out/nap_$v.log 2>&1; echo nap$v=$? $(grep -o '"solve_ms": [0-9.]*' gpurun_out/nap_$v.log | tr '\n' ' '); done
