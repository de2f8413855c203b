# done_s by a relaxed store after the barrier (MEMBAR.ALL.CTA off the compute chain); U = 2 (8 compute warps)
set -x
timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 3 > gpurun_out/relax_c1.log 2>&1; echo a=$?
ILS_RK_U=2 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 3 > gpurun_out/relax_c1_u2.log 2>&1; echo b=$?
ILS_RK_PROF=1 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 > gpurun_out/relax_prof.log 2>&1; echo c=$?
ILS_RK_U=2 ILS_RK_PROF=1 timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 > gpurun_out/relax_prof_u2.log 2>&1; echo d=$?
timeout 300 python tools/c3_inner_probe.py rk 20000 > gpurun_out/relax_c3rk.log 2>&1; echo e=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rk" > gpurun_out/relax_t1.log 2>&1; echo t1=$?
timeout 900 python -m pytest tests/test_gpu_sparse.py -q -x > gpurun_out/relax_t2.log 2>&1; echo t2=$?
