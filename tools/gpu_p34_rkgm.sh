# blocked SP-RK-RGS in gmode (c2 geometry: B = 2 or 4 steps per cluster reduction, tables in global
# memory): parity (c2 Mode F, forced-large, paper families, all RK tests) + c2 per-step timing
set -x
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_large.py tests/test_gpu_parity.py -m gpu -x -q -k "rk or large or paper or c2" > gpurun_out/p34_tests.log 2>&1; echo tests=$?
timeout 600 python tools/probe_perf.py --config c2 --methods rk --reps 1 --max-iter 1 --max-inner 20000 2>&1 | grep -o '"solve_ms": [0-9.]*\|"hot_ms": \[[0-9., ]*' | head -2
ILS_RK_SINGLE_STEP=1 timeout 600 python tools/probe_perf.py --config c2 --methods rk --reps 1 --max-iter 1 --max-inner 20000 2>&1 | grep -o '"solve_ms": [0-9.]*\|"hot_ms": \[[0-9., ]*' | head -2
ILS_RK_BLOCK=2 timeout 600 python tools/probe_perf.py --config c2 --methods rk --reps 1 --max-iter 1 --max-inner 20000 2>&1 | grep -o '"solve_ms": [0-9.]*\|"hot_ms": \[[0-9., ]*' | head -2
