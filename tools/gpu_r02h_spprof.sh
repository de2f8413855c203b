# phase timers of the c2 SP K1 + P stream (ILS_SP_PROF) and the stream rate with / without them
set -x
timeout 600 python tools/sp_stream_probe.py c2 default > gpurun_out/spprof_base.log 2>&1; echo base=$?
ILS_SP_PROF=1 timeout 600 python tools/sp_stream_probe.py c2 default > gpurun_out/spprof.log 2>&1; echo prof=$?
