# ncu --set full captures of the block tail at configs [4] and [2] (summaries only come back) and a bench line.
set -x
python tools/step_kernels.py 4:1024 2:256 > gpurun_out/r02_step_kernels.txt 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_block_tail_sm -s 40 -c 1 -o /tmp/r02_tail4 python tools/step_kernels.py 4:1024 > gpurun_out/r02_ncu_tail4.log 2>&1
ncu -i /tmp/r02_tail4.ncu-rep --page raw --csv > gpurun_out/r02_ncu_tail4.raw.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_block_tail_sm -s 40 -c 1 -o /tmp/r02_tail2 python tools/step_kernels.py 2:256 > gpurun_out/r02_ncu_tail2.log 2>&1
ncu -i /tmp/r02_tail2.ncu-rep --page raw --csv > gpurun_out/r02_ncu_tail2.raw.csv 2>&1
ncu -i /tmp/r02_tail2.ncu-rep --page source --csv > gpurun_out/r02_ncu_tail2.source.csv 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err
echo done
