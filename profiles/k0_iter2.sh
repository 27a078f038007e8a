# K0 variant loop (round 2, session 5): parity tests of $TESTV variants, then
# bench timings of the main library and $VARIANTS on $CFGS, then K0's ncu
# instruction / issue metrics for each
set -u
out=gpurun_out; tag=${1:-it}
mkdir -p $out
if [ -n "${TESTMAIN:-}" ]; then
  timeout 1500 python -m pytest tests/test_gpu_field.py tests/test_gpu_fullsize.py tests/test_gpu_query.py -q -x > $out/${tag}_main_tests.log 2>&1; echo rc=$? >> $out/${tag}_main_tests.log
fi
for v in ${TESTV:-}; do
  CAPT_LIB_VARIANT=${v:+libcapt_b200_$v.so} timeout 900 python -m pytest tests/test_gpu_field.py tests/test_gpu_fullsize.py -q -x > $out/${tag}_${v}_tests.log 2>&1; echo rc=$? >> $out/${tag}_${v}_tests.log
done
for v in "" ${VARIANTS:-}; do
  for c in ${CFGS:-3}; do
    CAPT_LIB_VARIANT=${v:+libcapt_b200_$v.so} python bench.py --config $c --no-parity --no-cpu-baseline --e2e-steps 0 > $out/${tag}_${v:-base}_cfg$c.json 2>&1
  done
done
M=smsp__inst_executed.sum,gpu__time_duration.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum
if [ -z "${NONCU:-}" ]; then
for v in "" ${VARIANTS:-}; do
  for c in ${CFGS:-3}; do
    cmd="python bench.py --config $c --no-parity --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3"
    CAPT_LIB_VARIANT=${v:+libcapt_b200_$v.so} ncu --metrics $M --clock-control none -k regex:k_resolve -s 3 -c 1 --csv $cmd 2>/dev/null | grep -E '"(smsp|gpu|l1tex|lts|launch|sm|dram)__' > $out/${tag}_${v:-base}_ncu_cfg$c.csv
  done
done
fi
python - <<PY
import json,glob,os
for f in sorted(glob.glob("$out/${tag}_*_cfg*.json")):
    try:
        d=json.loads([l for l in open(f) if l.startswith("{")][-1])
        st=d["roofline"]["stages"]
        print(os.path.basename(f), "step %.4f"%d["ms_per_step"], "K0 %.4f frac %.3f"%(st[0]["ms"],st[0]["frac"]), "list %.4f"%st[1]["ms"], d["clocks"].get("sm_mhz"))
    except Exception as e:
        print(os.path.basename(f), "ERR", e)
PY
