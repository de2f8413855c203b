set -x
timeout 300 python tools/c3_inner_probe.py rk 20000 > gpurun_out/g4_c3rk.log 2>&1; echo p1=$?
ILS_SRK_PROF=1 timeout 300 python tools/c3_inner_probe.py rk 20000 > gpurun_out/g4_c3rk_prof.log 2>&1; echo p2=$?
timeout 600 python -m pytest tests/test_gpu_sparse.py -q -x -k "rk or methods" > gpurun_out/g4_sparse.log 2>&1; echo t1=$?
