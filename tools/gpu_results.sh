# full GPU validation + per-config bench lines (round results)
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu_full.log
timeout 900 python bench.py > gpurun_out/res_bench_c1.json 2> gpurun_out/res_bench_c1.err; echo c1=$?
timeout 600 python bench.py --config c0 --no-cpu-baseline > gpurun_out/res_bench_c0.json 2> gpurun_out/res_bench_c0.err; echo c0=$?
timeout 900 python bench.py --config c2 --steps 3 > gpurun_out/res_bench_c2.json 2> gpurun_out/res_bench_c2.err; echo c2=$?
timeout 900 python bench.py --config c3 --steps 3 > gpurun_out/res_bench_c3.json 2> gpurun_out/res_bench_c3.err; echo c3=$?
timeout 600 python bench.py --config c4 --steps 3 > gpurun_out/res_bench_c4.json 2> gpurun_out/res_bench_c4.err; echo c4=$?
timeout 600 python tools/probe_perf.py --config c2 --methods rk,rgs,rcd --reps 1 --max-iter 2 --max-inner 20000 > gpurun_out/res_probe_c2_capped.log 2>&1; echo c2cap=$?
timeout 600 python tools/probe_perf.py --config c3 --methods rk,rgs --reps 1 --max-iter 2 --max-inner 100000 > gpurun_out/res_probe_c3_capped.log 2>&1; echo c3cap=$?
