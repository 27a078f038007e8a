# list-stage variants: field tests, then config 3/2/1/0 timings for the main library and $VARIANTS
set -u
tag=${1:-li}
timeout 900 python -m pytest tests/test_gpu_field.py tests/test_gpu_fullsize.py -q -x > gpurun_out/${tag}_tests.log 2>&1; echo rc=$? >> gpurun_out/${tag}_tests.log
for v in "" ${VARIANTS:-}; do for c in 3 2 1 0; do
  CAPT_LIB_VARIANT=$v python bench.py --config $c --no-parity --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_${v:-base}_cfg$c.json 2>&1
done; done
