# Round-2 third session: baseline at HEAD in a fresh container (full GPU suite, default bench line,
# smoke, SP setup launch lists at c2 and c3 for the factorization work).
set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2e_gputest.log 2>&1; echo gputest=$?
timeout 900 python bench.py > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo bench=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1; echo smoke=$?
timeout 300 python tools/sp_setup_probe.py c2 2 > gpurun_out/r2e_c2_setup.log 2>&1; echo c2s=$?
timeout 300 python tools/sp_setup_probe.py c3 2 > gpurun_out/r2e_c3_setup.log 2>&1; echo c3s=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_launch_c2setup.csv python tools/sp_setup_probe.py c2 1 > gpurun_out/r2e_ncu_c2.log 2>&1; echo c2=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_launch_c3setup.csv python tools/sp_setup_probe.py c3 1 > gpurun_out/r2e_ncu_c3.log 2>&1; echo c3=$?
