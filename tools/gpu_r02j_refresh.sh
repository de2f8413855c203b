# Round-2 final refresh at HEAD (after the SP grid barrier, the tiled transposed GEMV and the 16-byte row pass):
# full GPU suite, default bench line, smoke, c1 launch list, c3 SP solve probe.
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2j_gputest.log 2>&1; echo gputest=$?
timeout 900 python bench.py > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err; echo bench=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; echo smoke=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2j_launches_c1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --extra-configs '' > gpurun_out/r2j_ncu_launch.log 2>&1; echo launch=$?
timeout 600 python tools/probe_perf.py --config c3 --methods sp --reps 3 > gpurun_out/r2j_c3sp.log 2>&1; echo c3sp=$?
