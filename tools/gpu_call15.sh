timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rk" 2>&1 | tail -1
for B in 1 2 4; do for C in 8 16; do
ILS_RK_BLOCK=$B ILS_RK_CLUSTER=$C timeout 300 python tools/probe_perf.py --config c1 --methods rk --reps 1 > gpurun_out/p15_c1_B${B}_C$C.log 2>&1; echo "B=$B C=$C"; python tools/show_probe.py gpurun_out/p15_c1_B${B}_C$C.log | grep rk
done; done
for B in 1 2 4; do
ILS_RK_BLOCK=$B timeout 300 python tools/probe_perf.py --config c0 --methods rk --reps 1 > gpurun_out/p15_c0_B${B}.log 2>&1; echo "c0 B=$B"; python tools/show_probe.py gpurun_out/p15_c0_B${B}.log | grep rk
done
