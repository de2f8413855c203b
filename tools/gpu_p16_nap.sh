# look-ahead SP-RK-RGS: helper-warp polling with __nanosleep (ILS_RK_NAP ns) vs busy polling, c1 full solve
for nap in 0 32 100 300 0 100; do
  ILS_RK_NAP=$nap timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 2 2>&1 | grep -o '"solve_ms": [0-9.]*' | tail -1 | sed "s/^/nap=$nap /"
done
ILS_RK_NAP=100 ILS_RK_PROF=1 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 --max-iter 2 2>&1 | grep "ILS_RK_PROF" | head -2
