# A/B of a c1 method between the current library and lib_old (tools/build_ab.py <rev> old); extra env in $2
for i in 1 2; do
  for L in paper_2203_15340_b200/lib/libils.so paper_2203_15340_b200/lib_old/libils.so; do
    env ${2:-X=1} ILS_LIB_PATH=$L timeout 300 python tools/probe_perf.py --config c1 --methods ${1:-rgs} --reps 2 2>&1 | grep -o "\"solve_ms\": [0-9.]*\|\"inner_iters_total\": [0-9]*" | tr '\n' ' '; echo " $L ${2:-}"
  done
done
