# Round-2 sixth session: evidence at HEAD: full GPU suite, default bench line, smoke, c1 launch list,
# ncu captures of the two dominant c1 kernels.
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2h_gputest.log 2>&1; echo gputest=$?
timeout 900 python bench.py > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo bench=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo smoke=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_launches_c1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --extra-configs '' > gpurun_out/r2h_ncu_launch.log 2>&1; echo launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rk_rgs_la_kernel" -s 2 -c 1 -o gpurun_out/r2h_prof_c1rk python tools/probe_perf.py --config c1 --methods rk --reps 1 > gpurun_out/r2h_ncu_c1rk.log 2>&1; echo ncu_c1rk=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scd_chunk_kernel" -s 20 -c 1 -o gpurun_out/r2h_prof_c1scd python tools/probe_perf.py --config c1 --methods rgs --reps 1 > gpurun_out/r2h_ncu_c1scd.log 2>&1; echo ncu_c1scd=$?
