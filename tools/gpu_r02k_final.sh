# Round-2 closing run at HEAD: full GPU suite, default bench line, smoke, c1 launch list.
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2k_gputest.log 2>&1; echo gputest=$?
timeout 900 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err; echo bench=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo smoke=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k_launches_c1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --extra-configs '' > gpurun_out/r2k_ncu_launch.log 2>&1; echo launch=$?
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r2k_bench_ref.json 2> gpurun_out/r2k_bench_ref.err; echo ref=$?
