# ncu --set full of the packed-fp32 fused colour sweep (config [2]); raw + source pages to gpurun_out/
python tools/sweep2_probe.py > gpurun_out/sweep2.txt 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_lmo_sweep -s 1 -c 1 -o /tmp/r02_col2 python tools/sweep2_probe.py > gpurun_out/r02_ncu_col2.log 2>&1
cp /tmp/r02_col2.ncu-rep gpurun_out/
ncu -i /tmp/r02_col2.ncu-rep --page raw --csv > gpurun_out/r02_ncu_col2.raw.csv 2>&1
ncu -i /tmp/r02_col2.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_ncu_col2.sass.csv 2>&1
ncu -i /tmp/r02_col2.ncu-rep --page details --csv > gpurun_out/r02_ncu_col2.details.csv 2>&1
