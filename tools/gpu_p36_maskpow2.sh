# forward masks kernel: shift/mask word and bit when NT is a power of two (A/B against HEAD) + parity
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "scd or rgs or subset" > gpurun_out/p36_tests.log 2>&1; echo tests=$?
for i in 1 2; do
timeout 300 python tools/c3_inner_probe.py rgs 20000 2>&1 | tail -1 | sed "s/^/new /"
ILS_LIB_PATH=paper_2203_15340_b200/lib_base/libils.so timeout 300 python tools/c3_inner_probe.py rgs 20000 2>&1 | tail -1 | sed "s/^/base /"
done
