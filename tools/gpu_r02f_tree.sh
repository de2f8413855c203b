set -x
timeout 900 python -m pytest tests/test_gpu_sparse.py -q -x -k "tree_inverse or sp_fixed or direct" > gpurun_out/tree_t1.log 2>&1; echo t1=$?
timeout 900 python -m pytest tests/test_gpu_large.py -q -x > gpurun_out/tree_t2.log 2>&1; echo t2=$?
for th in 8 16 32 64; do
ILS_ZT_TH=$th timeout 300 python tools/sp_setup_probe.py c3 2 > gpurun_out/tree_c3_th$th.log 2>&1; echo c3_$th=$?
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3" > gpurun_out/tree_t3.log 2>&1; echo t3=$?
