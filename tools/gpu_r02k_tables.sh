# paper Tables 2-5 protocol at HEAD (all 12 sizes x 3 methods x 10 trials)
set -x
timeout 2400 python tools/paper_tables.py --trials 10 --out gpurun_out/r2k_paper_tables > gpurun_out/r2k_paper_tables.log 2>&1; echo tables=$?
