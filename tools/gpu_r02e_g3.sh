# cluster sparse SP-RK-RGS: parity tests, c3 per-step probe (new vs ILS_SRK_CL=0)
set -x
timeout 600 python -m pytest tests/test_gpu_sparse.py -q -x > gpurun_out/g3_sparse.log 2>&1; echo t1=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3 or csr_long" > gpurun_out/g3_full.log 2>&1; echo t2=$?
timeout 300 python tools/c3_inner_probe.py rk 20000 > gpurun_out/g3_c3rk.log 2>&1; echo p1=$?
ILS_SRK_CL=0 timeout 300 python tools/c3_inner_probe.py rk 20000 > gpurun_out/g3_c3rk_old.log 2>&1; echo p2=$?
