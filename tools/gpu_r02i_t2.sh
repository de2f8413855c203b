# paper Table 2 first size (43000 x 13000): SP with the 32-column transposed GEMV vs the tiled one (+ 16-byte row pass)
set -x
ILS_COLS_TILED=0 timeout 900 python tools/paper_tables.py --tables t2 --sizes 0 --trials 3 --methods sp,scd --out gpurun_out/t2_cols0.json > gpurun_out/t2_cols0.log 2>&1; echo a=$?
timeout 900 python tools/paper_tables.py --tables t2 --sizes 0 --trials 3 --methods sp,scd --out gpurun_out/t2_cols1.json > gpurun_out/t2_cols1.log 2>&1; echo b=$?
timeout 900 python -m pytest tests/test_gpu_large.py -q -x > gpurun_out/t2_t1.log 2>&1; echo t1=$?
