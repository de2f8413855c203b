# Round-2 fourth session: evidence at HEAD after the late c3 commits (cluster SP-RK-RGS, staged sparse
# Gram, MLP of the GEMV passes): full GPU suite, default bench line, smoke, c1 launch list, ncu captures
# of the c3 cluster RK-RGS kernel and the sparse Gram, SP setup launch lists at c2 / c3.
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2f_gputest.log 2>&1; echo gputest=$?
timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo bench=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo smoke=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launches_c1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --extra-configs '' > gpurun_out/r2f_ncu_launch.log 2>&1; echo launch=$?
timeout 300 python tools/c3_inner_probe.py rk 20000 > gpurun_out/r2f_c3rk.log 2>&1; echo c3rk=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sparse_rk_cl_kernel" -s 1 -c 1 -o gpurun_out/r2f_prof_c3rk python tools/c3_inner_probe.py rk 20000 > gpurun_out/r2f_ncu_c3rk.log 2>&1; echo ncu_c3rk=$?
timeout 300 python tools/sp_setup_probe.py c2 2 > gpurun_out/r2f_c2_setup.log 2>&1; echo c2s=$?
timeout 300 python tools/sp_setup_probe.py c3 2 > gpurun_out/r2f_c3_setup.log 2>&1; echo c3s=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launch_c2setup.csv python tools/sp_setup_probe.py c2 1 > gpurun_out/r2f_ncu_c2.log 2>&1; echo c2=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launch_c3setup.csv python tools/sp_setup_probe.py c3 1 > gpurun_out/r2f_ncu_c3.log 2>&1; echo c3=$?
