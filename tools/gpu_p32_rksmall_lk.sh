# one-CTA SP-RK-RGS with Gram lookups (c0): parity + A/B (ILS_RK_SMALL_LOOKUP=0), CTA sizes
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rk or smoke" > gpurun_out/p32_tests.log 2>&1; echo tests=$?
for nt in 256 128; do for lk in 1 0; do
  ILS_RK_SMALL_LOOKUP=$lk ILS_RK_SMALL_NT=$nt timeout 300 python tools/probe_perf.py --config c0 --methods rk --reps 3 2>&1 | grep -o '"solve_ms": [0-9.]*\|"inner_iters_total": [0-9]*' | tail -2 | tr '\n' ' ' | sed "s/^/nt=$nt lk=$lk /"; echo
done; done
