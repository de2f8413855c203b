set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench=$?
timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
for m in rk rgs sp; do
timeout 300 python tools/probe_perf.py --config c1 --methods $m --reps 1 > gpurun_out/probe1_$m.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rk_rgs_kernel|scd_kernel|sp_persistent" -s 1 -c 1 -o gpurun_out/prof_c1_$m python tools/probe_perf.py --config c1 --methods $m --reps 1 > gpurun_out/ncu_full_$m.log 2>&1; echo ncu_$m=$?
done
