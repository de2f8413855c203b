# column pass (X^T y, warp-interleaved rows): eight rows in flight per warp; c3 SP and large-n paths
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_sparse.py -m gpu -x -q -k "sp or large or sparse or paper" > gpurun_out/p39_tests.log 2>&1; echo tests=$?
for i in 1 2; do
timeout 300 python tools/probe_perf.py --config c3 --methods sp --reps 2 2>&1 | grep -o '"solve_ms": [0-9.]*' | tail -1 | sed "s/^/new /"
ILS_LIB_PATH=paper_2203_15340_b200/lib_base/libils.so timeout 300 python tools/probe_perf.py --config c3 --methods sp --reps 2 2>&1 | grep -o '"solve_ms": [0-9.]*' | tail -1 | sed "s/^/base /"
done
