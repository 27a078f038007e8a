set -u
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_filter.py tests/test_gpu_fullsize.py tests/test_gpu_query.py tests/test_gpu_capt_files.py -q -x > gpurun_out/pre1_tests.log 2>&1; echo rc=$? >> gpurun_out/pre1_tests.log
python bench.py --config 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pre1_cfg2.json 2>&1
python bench.py --config 3 --no-parity --no-cpu-baseline --e2e-steps 0 > gpurun_out/pre1_cfg3.json 2>&1
python bench.py --config 1 --no-parity --no-cpu-baseline --e2e-steps 0 > gpurun_out/pre1_cfg1.json 2>&1
cmd="python bench.py --config 2 --no-parity --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3"
$cmd > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pre1_cfg2_launches.csv $cmd > /dev/null 2>&1
