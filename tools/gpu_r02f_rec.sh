set -x
timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 3 > gpurun_out/rec_c1.log 2>&1; echo c1=$?
ILS_RK_PROF=1 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 > gpurun_out/rec_c1prof.log 2>&1; echo c1p=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rk" > gpurun_out/rec_t1.log 2>&1; echo t1=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c1" > gpurun_out/rec_t2.log 2>&1; echo t2=$?
