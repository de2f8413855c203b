# Round evidence refresh: bench lines for c0..c4, capped probes for c2/c3, the c1 launch list, and
# full ncu captures of the two single-instance inner kernels. Outputs under gpurun_out/.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/res_bench_c1.json 2> gpurun_out/res_bench_c1.err; echo c1=$?
timeout 600 python bench.py --config c0 --no-cpu-baseline > gpurun_out/res_bench_c0.json 2> gpurun_out/res_bench_c0.err; echo c0=$?
timeout 900 python bench.py --config c2 --steps 3 > gpurun_out/res_bench_c2.json 2> gpurun_out/res_bench_c2.err; echo c2=$?
timeout 900 python bench.py --config c3 --steps 3 > gpurun_out/res_bench_c3.json 2> gpurun_out/res_bench_c3.err; echo c3=$?
timeout 600 python bench.py --config c4 --steps 3 > gpurun_out/res_bench_c4.json 2> gpurun_out/res_bench_c4.err; echo c4=$?
timeout 600 python tools/probe_perf.py --config c2 --methods rk,rgs,rcd --reps 1 --max-iter 2 --max-inner 20000 > gpurun_out/res_probe_c2_capped.log 2>&1; echo c2cap=$?
timeout 600 python tools/probe_perf.py --config c3 --methods rk,rgs --reps 1 --max-iter 2 --max-inner 100000 > gpurun_out/res_probe_c3_capped.log 2>&1; echo c3cap=$?
timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/res_bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/res_launches_c1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/res_ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 --max-iter 1 > gpurun_out/res_pr_rk.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rk_rgs_block_kernel" -s 2 -c 1 -o gpurun_out/res_prof_c1_rkb python tools/probe_perf.py --config c1 --methods rk --reps 1 --max-iter 1 > gpurun_out/res_ncu_rkb.log 2>&1; echo ncu_rk=$?
timeout 300 python tools/probe_perf.py --config c1 --methods rgs --reps 1 --max-iter 1 > gpurun_out/res_pr_rgs.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_chunk_kernel|scd_masks_kernel|scd_check_kernel" -s 3 -c 3 -o gpurun_out/res_prof_c1_scd python tools/probe_perf.py --config c1 --methods rgs --reps 1 --max-iter 1 > gpurun_out/res_ncu_scd.log 2>&1; echo ncu_scd=$?
timeout 1500 python tools/paper_tables.py --trials 10 --out gpurun_out/res_paper_tables > gpurun_out/res_paper_tables.log 2>&1; echo tables=$?
timeout 600 python tools/alpha_study.py --config c1 --seeds 3 --out gpurun_out/res_alpha_c1 > gpurun_out/res_alpha.log 2>&1; echo alpha=$?
