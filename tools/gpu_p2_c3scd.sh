# c3 SP-SCD per-step cost by horizon and the launch list of a 40000-step run (masks / chunk / check split)
set -x
timeout 300 python tools/c3_inner_probe.py rgs 4000 > gpurun_out/p2_c3_4000.log 2>&1
timeout 300 python tools/c3_inner_probe.py rgs 20000 > gpurun_out/p2_c3_20000.log 2>&1
timeout 300 python tools/c3_inner_probe.py rgs 60000 > gpurun_out/p2_c3_60000.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/p2_launch_c3scd.csv -k regex:"scd|check" python tools/c3_inner_probe.py rgs 40000 > gpurun_out/p2_ncu.log 2>&1; echo ncu=$?
