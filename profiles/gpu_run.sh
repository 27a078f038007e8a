#!/bin/bash
# The GPU-box commands behind the committed evidence (run under gpurun from
# the repo root): GPU tests, the bench lines, the ncu launch list and one
# ncu --set full capture of the field pipeline's kernels.
#   bash profiles/gpu_run.sh <tag> [tests] [bench] [ncu] [cfgs...]
set -u
tag=${1:-r02}; shift || true
what=${*:-tests bench ncu}
out=gpurun_out
mkdir -p $out
(free -g; nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > $out/${tag}_host.txt 2>&1
if [[ " $what " == *" tests "* ]]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $out/${tag}_gputest.log 2>&1
  echo "rc=$?" >> $out/${tag}_gputest.log
fi
if [[ " $what " == *" bench "* ]]; then
  for c in 3 1 2 0; do
    timeout 900 python bench.py --config $c > $out/${tag}_bench_cfg$c.json 2> $out/${tag}_bench_cfg$c.err
    echo "cfg$c rc=$?" >> $out/${tag}_bench_rc.txt
  done
  timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $out/${tag}_bench_reference.json 2>&1
fi
if [[ " $what " == *" ncu "* ]]; then
  for c in 3 1; do
    cmd="python bench.py --config $c --no-parity --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3"
    $cmd > $out/${tag}_plain_cfg$c.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $out/${tag}_cfg${c}_launches.csv $cmd > $out/${tag}_ncu_launch_cfg$c.log 2>&1
    $cmd > $out/${tag}_plain2_cfg$c.log 2>&1 && \
    ncu --set full --clock-control none --import-source on \
        -k regex:"k_resolve|k_list_knn|k_tree_list" -s 6 -c 3 \
        -o $out/${tag}_cfg${c}_full $cmd > $out/${tag}_ncu_full_cfg$c.log 2>&1
  done
fi
