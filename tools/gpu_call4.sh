for c in c0 c1; do
for ce in 0 1000000000; do
timeout 300 python tools/probe_perf.py --config $c --methods rk,rgs --reps 1 --fixed 20000 --check-every $ce > gpurun_out/probe4_${c}_$ce.log 2>&1; echo probe $c $ce=$?
done; done
timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 --fixed 20000 --check-every 1000000000 > gpurun_out/p4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rk_rgs_kernel" -c 1 -o gpurun_out/prof4_c1_rk python tools/probe_perf.py --config c1 --methods rk --reps 1 --fixed 20000 --check-every 1000000000 > gpurun_out/ncu4_rk.log 2>&1; echo ncu_rk=$?
timeout 300 python tools/probe_perf.py --config c1 --methods rgs --reps 1 --fixed 20000 --check-every 1000000000 > gpurun_out/p4b.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_kernel" -c 1 -o gpurun_out/prof4_c1_scd python tools/probe_perf.py --config c1 --methods rgs --reps 1 --fixed 20000 --check-every 1000000000 > gpurun_out/ncu4_scd.log 2>&1; echo ncu_scd=$?
