# blocked 64x64 leaf v5 (stride 68, DMMA panel/trailing, uniform row/column lanes): parity + setup timing
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "sp or direct or spd or large or fullsize or literal or auto or batched" > gpurun_out/p10_tests.log 2>&1; echo tests=$?
timeout 300 python tools/mb/leaf_probe.py > gpurun_out/p10_leaf.log 2>&1
timeout 300 python tools/sp_setup_probe.py c2 3 > gpurun_out/p10_c2.log 2>&1
timeout 300 python tools/sp_setup_probe.py c3 3 > gpurun_out/p10_c3.log 2>&1
timeout 300 python tools/probe_perf.py --config c1 --methods sp --reps 3 > gpurun_out/p10_c1sp.log 2>&1
