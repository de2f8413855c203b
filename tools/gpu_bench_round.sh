# round bench + evidence: plain bench (c1 default), c4 and c0 per-method lines, launch list, ncu captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench=$?
timeout 600 python bench.py --config c0 --no-cpu-baseline > gpurun_out/bench_c0.json 2> gpurun_out/bench_c0.err; echo bench_c0=$?
timeout 600 python bench.py --config c4 --steps 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench_c4=$?
timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 --max-iter 1 > gpurun_out/pr_rk.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rk_rgs_block_kernel" -c 1 -o gpurun_out/prof_c1_rkb python tools/probe_perf.py --config c1 --methods rk --reps 1 --max-iter 1 > gpurun_out/ncu_rkb.log 2>&1; echo ncu_rk=$?
timeout 300 python tools/probe_perf.py --config c1 --methods rgs --reps 1 --max-iter 1 > gpurun_out/pr_rgs.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_chunk_kernel|scd_masks_kernel|scd_check_kernel" -c 3 -o gpurun_out/prof_c1_scd python tools/probe_perf.py --config c1 --methods rgs --reps 1 --max-iter 1 > gpurun_out/ncu_scd.log 2>&1; echo ncu_scd=$?
timeout 300 python tools/probe_perf.py --config c1 --methods sp --reps 2 > gpurun_out/pr_sp.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sp_persistent|gemm_dmma" -c 4 -o gpurun_out/prof_c1_sp python tools/probe_perf.py --config c1 --methods sp --reps 2 > gpurun_out/ncu_sp.log 2>&1; echo ncu_sp=$?
