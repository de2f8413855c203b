set -x
timeout 900 python -m pytest tests/test_gpu_sparse.py -q -x > gpurun_out/g1_sparse.log 2>&1; echo t=$?
timeout 300 python tools/sp_setup_probe.py c3 2 > gpurun_out/g1_c3_setup.log 2>&1; echo c3s=$?
ILS_SPGRAM_OLD=1 timeout 300 python tools/sp_setup_probe.py c3 2 > gpurun_out/g1_c3_setup_old.log 2>&1; echo c3o=$?
