# static / dynamic shared base addresses of the look-ahead RK-RGS kernel held in registers (no S2UR SR_CgaCtaId per iteration)
set -x
timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 3 > gpurun_out/launder_c1.log 2>&1; echo a=$?
ILS_RK_PROF=1 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 > gpurun_out/launder_prof.log 2>&1; echo c=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rk" > gpurun_out/launder_t1.log 2>&1; echo t1=$?
