set -x
timeout 600 python tools/probe_perf.py --config c3 --methods sp --reps 3 > gpurun_out/cols3.log 2>&1; echo b=$?
timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_large.py -q -x > gpurun_out/cols3_t1.log 2>&1; echo t1=$?
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3" > gpurun_out/cols3_t2.log 2>&1; echo t2=$?
