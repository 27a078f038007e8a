# K0 diagnostics: record-load and block-table counts (stats builds), then
# same-box timing of the listed variants
set -u
out=gpurun_out; tag=${1:-k2}
for v in libcapt_stats.so libcapt_stats40k.so; do
  for c in 3 1 2; do
    CAPT_LIB_VARIANT=$v python bench.py --config $c --no-parity --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3 2>&1 | grep "capt field" | tail -1 > $out/${tag}_${v}_cfg$c.txt
  done
done
for v in "" ${VARIANTS:-}; do
  for c in 3 1 2; do
    CAPT_LIB_VARIANT=$v python bench.py --config $c --no-parity --no-cpu-baseline --e2e-steps 0 > $out/${tag}_${v:-base}_cfg$c.json 2>&1
  done
done
