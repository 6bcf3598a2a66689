# ncu --set full of one block-step LMO sweep (config [2], B = 256): summary back only
set -x
python tools/step_kernels.py 2:256 > gpurun_out/r02_sweepb.txt 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_lmo_sweep -s 40 -c 1 -o /tmp/r02_sweepb python tools/step_kernels.py 2:256 > gpurun_out/r02_ncu_sweepb.log 2>&1
ncu -i /tmp/r02_sweepb.ncu-rep --page raw --csv > gpurun_out/r02_ncu_sweepb.raw.csv 2>&1
ncu -i /tmp/r02_sweepb.ncu-rep --page source --csv > gpurun_out/r02_ncu_sweepb.source.csv 2>&1
echo done
