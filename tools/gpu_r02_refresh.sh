# Round-2 evidence: c1 launch list of the bench step, full ncu captures of the dominant kernels
# (c1 look-ahead SP-RK-RGS = one inner solve per launch; c1 SP-SCD chunk; c2 SP row stream; c4
# batched RK-RGS / SP-SCD; c3 CSR look-ahead RK-RGS and cluster SP-SCD). Outputs under gpurun_out/.
set -x
timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --extra-configs '' > gpurun_out/r02_bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --extra-configs '' > gpurun_out/r02_ncu_launch.log 2>&1; echo launch=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rk_rgs_la_kernel" -s 1 -c 1 -o gpurun_out/r02_prof_c1_rkla python tools/probe_perf.py --config c1 --methods rk --reps 1 --max-iter 2 > gpurun_out/r02_ncu_rk.log 2>&1; echo ncu_rk=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_chunk_kernel" -s 3 -c 1 -o gpurun_out/r02_prof_c1_scd python tools/probe_perf.py --config c1 --methods rgs --reps 1 --max-iter 1 > gpurun_out/r02_ncu_scd.log 2>&1; echo ncu_scd=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sp_persistent" -s 1 -c 1 -o gpurun_out/r02_prof_c2_sp python tools/sp_one_solve.py > gpurun_out/r02_ncu_sp.log 2>&1; echo ncu_sp=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"batched_rkb_kernel|batched_scd_kernel" -c 2 -o gpurun_out/r02_prof_c4 python tools/probe_perf.py --config c4 --methods rk,rgs --reps 1 > gpurun_out/r02_ncu_c4.log 2>&1; echo ncu_c4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sparse_rk_la_kernel|scd_cluster_kernel" -s 2 -c 2 -o gpurun_out/r02_prof_c3 python tools/c3_inner_probe.py rk,rgs 4000 > gpurun_out/r02_ncu_c3.log 2>&1; echo ncu_c3=$?
