# checkpoint: full GPU suite, default bench line, smoke
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2c_gputest.log 2>&1; echo gputest=$?
timeout 900 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo bench=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo smoke=$?
