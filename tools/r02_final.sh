# Round-2 closing measurement (one B200): the bench line, the reference arm, the bench launch list
set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err || exit 1
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02f_bench_reference.json 2> gpurun_out/r02f_bench_reference.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep-check > gpurun_out/r02f_ncu_bench.log 2>&1
python tools/batched_probe.py > gpurun_out/r02f_batched.txt 2>&1
python tools/solo_fw_batched.py fw1 fw3 >> gpurun_out/r02f_batched.txt 2>&1
python tools/colour_sweep_probe.py >> gpurun_out/r02f_batched.txt 2>&1
echo done
