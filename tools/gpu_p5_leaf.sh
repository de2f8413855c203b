# blocked 64x64 leaf (potrf_trtri64_kernel): parity of every SP / direct / NOT_SPD path, then setup A/B
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "sp or direct or spd or large or fullsize or literal or auto or batched" > gpurun_out/p5_tests.log 2>&1; echo tests=$?
timeout 300 python tools/mb/leaf_probe.py > gpurun_out/p5_leaf_new.log 2>&1
ILS_LEAF_OLD=1 timeout 300 python tools/mb/leaf_probe.py > gpurun_out/p5_leaf_old.log 2>&1
timeout 300 python tools/sp_setup_probe.py c2 3 > gpurun_out/p5_c2_new.log 2>&1
ILS_LEAF_OLD=1 timeout 300 python tools/sp_setup_probe.py c2 3 > gpurun_out/p5_c2_old.log 2>&1
timeout 300 python tools/sp_setup_probe.py c3 2 > gpurun_out/p5_c3_new.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p5_launch_c2.csv python tools/sp_setup_probe.py c2 1 > /dev/null 2>&1; echo ncu=$?
