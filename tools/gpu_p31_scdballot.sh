# c1 SP-SCD chunk kernel: winner's r_j by vote + shuffle (A/B against HEAD) + parity
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "scd or rgs or subset or c1_full" > gpurun_out/p31_tests.log 2>&1; echo tests=$?
for i in 1 2 3; do
timeout 300 python tools/probe_perf.py --config c1 --methods rgs --reps 2 2>&1 | grep -o '"solve_ms": [0-9.]*' | tail -1 | sed "s/^/new /"
ILS_LIB_PATH=paper_2203_15340_b200/lib_base/libils.so timeout 300 python tools/probe_perf.py --config c1 --methods rgs --reps 2 2>&1 | grep -o '"solve_ms": [0-9.]*' | tail -1 | sed "s/^/base /"
done
