for c in c0 c1; do
timeout 300 python tools/probe_perf.py --config $c --methods rk --reps 1 --fixed 20000 --check-every 1000000000 > gpurun_out/p7_$c.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rk_rgs_kernel" -c 1 -o gpurun_out/prof7_${c}_rk python tools/probe_perf.py --config $c --methods rk --reps 1 --fixed 20000 --check-every 1000000000 > gpurun_out/ncu7_$c.log 2>&1; echo ncu_$c=$?
done
