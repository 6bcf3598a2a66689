# Closing measurement of round 2 (one B200): ncu --set full of the GA pipe with the speculative
# pre-scan (the bench's dominant kernel; refreshes profiles/r02_ncu_traffic.json), then the randomized
# parity sweep on the same build.
set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bcfw_ga_pipe -s 1 -c 1 -o /tmp/r02_ga_spec python tools/bcfw_probe.py GA 1 > gpurun_out/r02_ncu_ga_spec.log 2>&1
ncu -i /tmp/r02_ga_spec.ncu-rep --page raw --csv > gpurun_out/r02_ncu_ga_spec.raw.csv 2>&1
ncu -i /tmp/r02_ga_spec.ncu-rep --page details --csv > gpurun_out/r02_ncu_ga_spec.details.csv 2>&1
SRO_FUZZ_N=${SRO_FUZZ_N:-4000} SRO_FUZZ_SHARDED_N=${SRO_FUZZ_SHARDED_N:-1500} timeout 900 python -m pytest tests/test_gpu_random_configs.py -q -x > gpurun_out/r02_fuzz_spec.txt 2>&1
tail -2 gpurun_out/r02_fuzz_spec.txt
echo done
