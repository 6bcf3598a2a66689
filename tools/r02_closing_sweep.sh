# ncu --set full of the HBM-bound dense gap sweep (k_lmo_sweep_bulk, config [3]) on the closing round-2
# build: the source of bench.py's sweep_roofline.traffic.
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lmo_sweep_bulk -s 1 -c 1 -o /tmp/r02_sweep3 python tools/sweep3_probe.py > gpurun_out/r02_ncu_sweep3.log 2>&1
ncu -i /tmp/r02_sweep3.ncu-rep --page raw --csv > gpurun_out/r02_ncu_sweep3.raw.csv 2>&1
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_traffic.json 2> gpurun_out/r02_bench_traffic.err
echo done
