# 16-CTA cluster SP-SCD: every warp reduces the 16 CTA winners (no second CTA barrier), step length by
# reciprocal multiply: parity (cluster paths, c3 Mode F) + A/B against HEAD on c3
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_sparse.py tests/test_gpu_fullsize.py -m gpu -x -q -k "scd or rgs or large or sparse or c3" > gpurun_out/p33_tests.log 2>&1; echo tests=$?
for i in 1 2; do
timeout 300 python tools/c3_inner_probe.py rgs 20000 2>&1 | tail -1 | sed "s/^/new /"
ILS_LIB_PATH=paper_2203_15340_b200/lib_base/libils.so timeout 300 python tools/c3_inner_probe.py rgs 20000 2>&1 | tail -1 | sed "s/^/base /"
done
timeout 300 python tools/probe_perf.py --config c3 --methods rgs --reps 2 2>&1 | grep -o '"solve_ms": [0-9.]*\|"inner_iters_total": [0-9]*\|"err": [0-9.e-]*' | tail -3
