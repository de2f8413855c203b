# closing check at HEAD (masks overlap opt-in): full GPU suite, smoke, default bench line, c1 launch list
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2m_gputest.log 2>&1; echo gputest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2m_launches_c1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --extra-configs '' > gpurun_out/r2m_ncu_launch.log 2>&1; echo launch=$?
