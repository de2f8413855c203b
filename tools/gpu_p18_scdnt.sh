# c1 SP-SCD chunk kernel CTA size (ILS_SCD_NT): 256 (default) vs 128 vs 512
for nt in 256 128 512 256 128; do
  ILS_SCD_NT=$nt timeout 300 python tools/probe_perf.py --config c1 --methods rgs --reps 2 2>&1 | grep -o '"solve_ms": [0-9.]*' | tail -1 | sed "s/^/nt=$nt /"
done
