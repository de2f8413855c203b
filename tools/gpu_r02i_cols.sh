# tiled transposed GEMV (cols_tile_kernel): c3 SP solve A/B and the tests that reach it
set -x
ILS_COLS_TILED=0 timeout 600 python tools/probe_perf.py --config c3 --methods sp --reps 3 > gpurun_out/cols0.log 2>&1; echo a=$?
timeout 600 python tools/probe_perf.py --config c3 --methods sp --reps 3 > gpurun_out/cols1.log 2>&1; echo b=$?
timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_large.py -q -x > gpurun_out/cols_t1.log 2>&1; echo t1=$?
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3" > gpurun_out/cols_t2.log 2>&1; echo t2=$?
