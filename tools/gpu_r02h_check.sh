# full GPU suite + default bench after the SP grid-barrier change
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2i_gputest.log 2>&1; echo gputest=$?
timeout 900 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo bench=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1; echo smoke=$?
