# Round-2 final evidence: full GPU suite, default bench line, smoke, c1 launch list, ncu captures of the
# kernels changed late in the round (cluster SP-SCD, gmode blocked RK-RGS at c2, one-CTA RK-RGS at c0,
# batched SP-SCD alone, forward masks) plus the dominant c1 kernels. Outputs under gpurun_out/r2d_*.
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2d_gputest.log 2>&1; echo gputest=$?
timeout 900 python bench.py > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo bench=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1; echo smoke=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launches_c1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --extra-configs '' > gpurun_out/r2d_ncu_launch.log 2>&1; echo launch=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rk_rgs_la_kernel" -s 1 -c 1 -o gpurun_out/r2d_prof_c1_rkla python tools/probe_perf.py --config c1 --methods rk --reps 1 --max-iter 2 > gpurun_out/r2d_ncu_rk.log 2>&1; echo ncu_rk=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_chunk_kernel" -s 3 -c 1 -o gpurun_out/r2d_prof_c1_scd python tools/probe_perf.py --config c1 --methods rgs --reps 1 --max-iter 1 > gpurun_out/r2d_ncu_scd.log 2>&1; echo ncu_scd=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"batched_scd_kernel" -c 1 -o gpurun_out/r2d_prof_c4scd python tools/probe_perf.py --config c4 --methods rgs --reps 1 > gpurun_out/r2d_ncu_c4scd.log 2>&1; echo ncu_c4scd=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scd_cluster_kernel" -s 1 -c 1 -o gpurun_out/r2d_prof_c3scd python tools/c3_inner_probe.py rgs 4000 > gpurun_out/r2d_ncu_c3.log 2>&1; echo ncu_c3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rk_rgs_block_kernel" -s 1 -c 1 -o gpurun_out/r2d_prof_c2rk python tools/probe_perf.py --config c2 --methods rk --reps 1 --max-iter 1 --max-inner 8000 > gpurun_out/r2d_ncu_c2rk.log 2>&1; echo ncu_c2rk=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rk_rgs_small_kernel" -s 1 -c 1 -o gpurun_out/r2d_prof_c0rk python tools/probe_perf.py --config c0 --methods rk --reps 1 --max-iter 2 > gpurun_out/r2d_ncu_c0rk.log 2>&1; echo ncu_c0rk=$?
