timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_gpu.log
for c in c0 c1; do
timeout 300 python tools/probe_perf.py --config $c --methods rgs,rcd --reps 1 --fixed 20000 --check-every 1000000000 > gpurun_out/probe8_${c}_nochk.log 2>&1; echo probe $c nochk=$?
timeout 300 python tools/probe_perf.py --config $c --methods rgs,rcd --reps 2 > gpurun_out/probe8_${c}_full.log 2>&1; echo probe $c full=$?
done
