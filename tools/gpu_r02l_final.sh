# closing check at HEAD: full GPU suite, smoke, default bench line
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2l_gputest.log 2>&1; echo gputest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err; echo bench=$?
