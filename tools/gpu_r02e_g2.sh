set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sparse_gram --csv --log-file gpurun_out/g2_gram_new.csv python tools/sp_setup_probe.py c3 1 > gpurun_out/g2_ncu1.log 2>&1; echo a=$?
ILS_SPGRAM_OLD=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sparse_gram --csv --log-file gpurun_out/g2_gram_old.csv python tools/sp_setup_probe.py c3 1 > gpurun_out/g2_ncu2.log 2>&1; echo b=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_gram_staged -c 1 -o gpurun_out/g2_gram_staged python tools/sp_setup_probe.py c3 1 > gpurun_out/g2_ncu3.log 2>&1; echo c=$?
