timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_gpu.log
for c in c0 c1; do
for ce in 0 1000000000; do
timeout 300 python tools/probe_perf.py --config $c --methods rk --reps 1 --fixed 20000 --check-every $ce > gpurun_out/probe5_${c}_$ce.log 2>&1; echo probe $c $ce=$?
done
timeout 300 python tools/probe_perf.py --config $c --methods rk --reps 2 > gpurun_out/probe5_${c}_full.log 2>&1; echo probe $c full=$?
done
