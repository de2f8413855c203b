# faster grid barrier of the SP row-stream kernel: c2 stream rate + phase timers, then SP parity tests
set -x
timeout 600 python tools/sp_stream_probe.py c2 default > gpurun_out/spbar_base.log 2>&1; echo base=$?
ILS_SP_PROF=1 timeout 600 python tools/sp_stream_probe.py c2 default > gpurun_out/spbar_prof.log 2>&1; echo prof=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "sp or rhs or check or rr or xref" > gpurun_out/spbar_t1.log 2>&1; echo t1=$?
