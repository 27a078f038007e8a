# K0 iteration loop: field tests, bench timings (main library + $VARIANTS),
# then a small ncu metric set on K0 (instructions, issue, L1->L2 requests)
set -u
out=gpurun_out; tag=${1:-it}
timeout 900 python -m pytest tests/test_gpu_field.py tests/test_gpu_fullsize.py -q -x > $out/${tag}_tests.log 2>&1; echo rc=$? >> $out/${tag}_tests.log
for v in "" ${VARIANTS:-}; do
  for c in 3 1; do
    CAPT_LIB_VARIANT=$v python bench.py --config $c --no-parity --no-cpu-baseline --e2e-steps 0 > $out/${tag}_${v:-base}_cfg$c.json 2>&1
  done
done
M=smsp__inst_executed.sum,gpu__time_duration.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed
for v in "" ${VARIANTS:-}; do
  for c in 3 1; do
    cmd="python bench.py --config $c --no-parity --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3"
    CAPT_LIB_VARIANT=$v $cmd > /dev/null 2>&1 && \
    CAPT_LIB_VARIANT=$v ncu --metrics $M --clock-control none -k regex:k_resolve -s 3 -c 1 --csv $cmd 2>/dev/null | grep -E '"(smsp|gpu|l1tex|lts|launch|sm)__' > $out/${tag}_${v:-base}_ncu_cfg$c.csv
  done
done
