# Round-2 (second session) evidence: full GPU suite, default bench line, c1 launch list, ncu --set full
# captures of the kernels changed this session and the dominant ones. Outputs under gpurun_out/r2b_*.
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2b_gputest.log 2>&1; echo gputest=$?
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo bench=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo smoke=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_c1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --extra-configs '' > gpurun_out/r2b_ncu_launch.log 2>&1; echo launch=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rk_rgs_la_kernel" -s 1 -c 1 -o gpurun_out/r2b_prof_c1_rkla python tools/probe_perf.py --config c1 --methods rk --reps 1 --max-iter 2 > gpurun_out/r2b_ncu_rk.log 2>&1; echo ncu_rk=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_chunk_kernel" -s 3 -c 1 -o gpurun_out/r2b_prof_c1_scd python tools/probe_perf.py --config c1 --methods rgs --reps 1 --max-iter 1 > gpurun_out/r2b_ncu_scd.log 2>&1; echo ncu_scd=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sp_persistent" -s 1 -c 1 -o gpurun_out/r2b_prof_c2_sp python tools/sp_one_solve.py > gpurun_out/r2b_ncu_sp.log 2>&1; echo ncu_sp=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"batched_rkb_kernel|batched_scd_kernel" -c 2 -o gpurun_out/r2b_prof_c4 python tools/probe_perf.py --config c4 --methods rk,rgs --reps 1 > gpurun_out/r2b_ncu_c4.log 2>&1; echo ncu_c4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scd_cluster_kernel|scd_masks_fwd_kernel" -s 2 -c 2 -o gpurun_out/r2b_prof_c3 python tools/c3_inner_probe.py rgs 4000 > gpurun_out/r2b_ncu_c3.log 2>&1; echo ncu_c3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"potrf_trtri64" -s 5 -c 1 -o gpurun_out/r2b_prof_leaf python tools/mb/leaf_probe.py > gpurun_out/r2b_ncu_leaf.log 2>&1; echo ncu_leaf=$?
