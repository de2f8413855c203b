# SP-SCD masks overlap with the shared auxiliary stream, A/B inside the full default bench step + SCD tests
set -x
for r in 1 2; do
ILS_SCD_MASK_OVERLAP=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra-configs '' > gpurun_out/mabg0_$r.json 2> gpurun_out/mabg0_$r.err; echo a$r=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra-configs '' > gpurun_out/mabg1_$r.json 2> gpurun_out/mabg1_$r.err; echo b$r=$?
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "scd or rgs or SCD or rcd" > gpurun_out/mabg_t1.log 2>&1; echo t1=$?
