# batched SP-SCD templated on (weighted, n == 32): parity at n = 32 and generic n, A/B timing
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "batched or c4" > gpurun_out/p14_tests.log 2>&1; echo tests=$?
for i in 1 2; do
timeout 300 python tools/probe_perf.py --config c4 --methods rgs --reps 2 2>&1 | grep -o '"solve_ms": [0-9.]*' | sed "s/^/new /"
ILS_LIB_PATH=paper_2203_15340_b200/lib_base/libils.so timeout 300 python tools/probe_perf.py --config c4 --methods rgs --reps 2 2>&1 | grep -o '"solve_ms": [0-9.]*' | sed "s/^/base /"
done
