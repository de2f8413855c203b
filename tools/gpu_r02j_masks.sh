# SP-SCD: masks of chunk i + 1 on an auxiliary stream while chunk i runs (ILS_SCD_MASK_OVERLAP=0: in turn)
set -x
ILS_SCD_MASK_OVERLAP=0 timeout 300 python tools/probe_perf.py --config c1 --methods rgs --reps 3 > gpurun_out/masks0.log 2>&1; echo a=$?
timeout 300 python tools/probe_perf.py --config c1 --methods rgs --reps 3 > gpurun_out/masks1.log 2>&1; echo b=$?
ILS_SCD_MASK_OVERLAP=0 timeout 300 python tools/probe_perf.py --config c0 --methods rgs --reps 3 > gpurun_out/masks0_c0.log 2>&1; echo a0=$?
timeout 300 python tools/probe_perf.py --config c0 --methods rgs --reps 3 > gpurun_out/masks1_c0.log 2>&1; echo b0=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "scd or rgs or SCD or rcd" > gpurun_out/masks_t1.log 2>&1; echo t1=$?
