# Round-2 measurement run (one B200): bench lines, ncu captures summarised on the box (the .ncu-rep
# files themselves are too large to bring back), launch list of one bench step.
set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err || exit 1
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
for spec in "k_bcfw_ga_pipe:ga:tools/bcfw_probe.py GA 1:1" "k_bcfw_pipe:pipe:tools/bcfw_probe.py P 1:1" "k_block_tail_sm:tail4:tools/step_kernels.py 4:1024:30" "k_block_tail_sm:tail2:tools/step_kernels.py 2:256:30"; do
  IFS=: read -r kern tag cmd skip <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$kern -s $skip -c 1 -o /tmp/r02_$tag python $cmd > gpurun_out/r02_ncu_$tag.log 2>&1
  ncu -i /tmp/r02_$tag.ncu-rep --page details --csv > gpurun_out/r02_ncu_$tag.details.csv 2>&1
  ncu -i /tmp/r02_$tag.ncu-rep --page raw --csv > gpurun_out/r02_ncu_$tag.raw.csv 2>&1
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep-check > gpurun_out/r02_ncu_bench.log 2>&1
ls -la gpurun_out
echo done
