# forward masks kernel: parity (SCD tests) and c3 / c1 SP-SCD per-step cost
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "scd or subset" > gpurun_out/p3_tests.log 2>&1; echo tests=$?
timeout 300 python tools/c3_inner_probe.py rgs 20000 > gpurun_out/p3_c3_20000.log 2>&1
ILS_MASKS_FWD=0 timeout 300 python tools/c3_inner_probe.py rgs 20000 > gpurun_out/p3_c3_20000_old.log 2>&1
timeout 300 python tools/probe_perf.py --config c1 --methods rgs --reps 2 > gpurun_out/p3_c1.log 2>&1
timeout 300 python tools/probe_perf.py --config c3 --methods rgs --reps 1 > gpurun_out/p3_c3_full.log 2>&1
