# SP-SCD masks overlap, A/B inside the full default bench step (sp, rk, rgs per step), two rounds each
set -x
for r in 1 2; do
ILS_SCD_MASK_OVERLAP=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra-configs '' > gpurun_out/mabf0_$r.json 2> gpurun_out/mabf0_$r.err; echo a$r=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra-configs '' > gpurun_out/mabf1_$r.json 2> gpurun_out/mabf1_$r.err; echo b$r=$?
done
