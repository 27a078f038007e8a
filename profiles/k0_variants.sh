# K0 variants side by side (experiment runner; gpurun from the repo root)
set -u
out=gpurun_out
tag=${1:-k0}
timeout 900 python -m pytest tests/test_gpu_field.py tests/test_gpu_fullsize.py tests/test_gpu_query.py -q -x > $out/${tag}_tests.log 2>&1; echo rc=$? >> $out/${tag}_tests.log
for v in "" ${VARIANTS:-}; do
  for c in 3 1 2; do
    CAPT_LIB_VARIANT=$v python bench.py --config $c --no-parity --no-cpu-baseline --e2e-steps 0 > $out/${tag}_${v:-base}_cfg$c.json 2>&1
  done
done
