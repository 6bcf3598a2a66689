# ncu --set full of one FW-ELS iteration's dense sweep at config [1] (k_lmo_sweep_bulk, 64 MB)
ncu --set full --clock-control none --cache-control none -k regex:k_lmo_sweep_bulk -s 20 -c 1 -o /tmp/r02_fwsw python tools/solo_fw_batched.py fw1 > gpurun_out/r02_ncu_fwsw.log 2>&1
ncu -i /tmp/r02_fwsw.ncu-rep --page raw --csv > gpurun_out/r02_ncu_fwsw.raw.csv 2>&1
ncu -i /tmp/r02_fwsw.ncu-rep --page details --csv > gpurun_out/r02_ncu_fwsw.details.csv 2>&1
