# ncu --set full of one block-step sweep (k_lmo_sweep<SrcColour<float>, 1>) in the batched config-[2] solve
REPS=1 ncu --set full --clock-control none --cache-control none --import-source on -k k_lmo_sweep -s 40 -c 1 -o /tmp/r02_bsw python tools/batched_probe.py 2:256 > gpurun_out/r02_ncu_bsw.log 2>&1
cp /tmp/r02_bsw.ncu-rep gpurun_out/
ncu -i /tmp/r02_bsw.ncu-rep --page raw --csv > gpurun_out/r02_ncu_bsw.raw.csv 2>&1
ncu -i /tmp/r02_bsw.ncu-rep --page details --csv > gpurun_out/r02_ncu_bsw.details.csv 2>&1
ncu -i /tmp/r02_bsw.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_ncu_bsw.sass.csv 2>&1
