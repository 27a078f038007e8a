# small-batch path: query/field tests, then the config-4 sweep (up to 4^12) per library
set -u
tag=${1:-sm}
timeout 900 python -m pytest tests/test_gpu_field.py tests/test_gpu_query.py tests/test_gpu_binned.py tests/test_gpu_filter.py tests/test_trace.py -q -x > gpurun_out/${tag}_tests.log 2>&1; echo rc=$? >> gpurun_out/${tag}_tests.log
for v in "" ${VARIANTS:-}; do
  CAPT_LIB_VARIANT=$v timeout 600 python bench.py --sweep --sweep-max-exp 12 > gpurun_out/${tag}_${v:-base}_sweep.json 2> gpurun_out/${tag}_${v:-base}_sweep.err
  CAPT_LIB_VARIANT=$v python bench.py --config 0 --no-parity --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_${v:-base}_cfg0.json 2>&1
done
