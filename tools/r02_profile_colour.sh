python tools/sweep2_probe.py > gpurun_out/sweep2.txt 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_lmo_sweep -s 1 -c 1 -o /tmp/r02_col python tools/sweep2_probe.py > gpurun_out/r02_ncu_col.log 2>&1
ncu -i /tmp/r02_col.ncu-rep --page raw --csv > gpurun_out/r02_ncu_col.raw.csv 2>&1
ncu -i /tmp/r02_col.ncu-rep --page source --csv > gpurun_out/r02_ncu_col.source.csv 2>&1
