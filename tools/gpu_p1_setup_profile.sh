set -x
timeout 300 python tools/sp_setup_probe.py c2 2 > gpurun_out/p1_c2_setup.log 2>&1
timeout 300 python tools/sp_setup_probe.py c3 2 > gpurun_out/p1_c3_setup.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p1_launch_c2.csv python tools/sp_setup_probe.py c2 1 > gpurun_out/p1_ncu_c2.log 2>&1; echo c2=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p1_launch_c3.csv python tools/sp_setup_probe.py c3 1 > gpurun_out/p1_ncu_c3.log 2>&1; echo c3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"batched_scd_kernel" -c 1 -o gpurun_out/p1_prof_c4scd python tools/probe_perf.py --config c4 --methods rgs --reps 1 > gpurun_out/p1_ncu_c4.log 2>&1; echo c4=$?
