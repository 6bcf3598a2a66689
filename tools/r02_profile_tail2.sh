# ncu --set full of one k_block_tail_sm (batched config [2], B = 256) with per-source-line stall samples
REPS=1 ncu --set full --clock-control none --cache-control none --import-source on -k k_block_tail_sm -s 40 -c 1 -o /tmp/r02_tail2 python tools/batched_probe.py 2:256 > gpurun_out/r02_ncu_tail2.log 2>&1
ncu -i /tmp/r02_tail2.ncu-rep --page raw --csv > gpurun_out/r02_ncu_tail2.raw.csv 2>&1
ncu -i /tmp/r02_tail2.ncu-rep --page source --csv --print-source cuda > gpurun_out/r02_ncu_tail2.src.csv 2>&1
ncu -i /tmp/r02_tail2.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_ncu_tail2.sass.csv 2>&1
