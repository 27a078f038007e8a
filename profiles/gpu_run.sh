#!/bin/bash
# The GPU-box commands behind the committed evidence (run under gpurun from
# the repo root): GPU tests, the bench lines (configs 3, 1, 2, 0, the
# reference arm, the config-4 sweep), the ncu launch lists and ncu --set full
# captures of the query kernels (configs 3, 1) and of the preprocessing
# kernels (config 2).
#   bash profiles/gpu_run.sh <tag> [tests] [bench] [ncu]
set -u
tag=${1:-r02}; shift || true
what=${*:-tests bench ncu}
out=gpurun_out
mkdir -p $out
(free -g; nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > $out/${tag}_host.txt 2>&1
if [[ " $what " == *" tests "* ]]; then
  timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > $out/${tag}_gputest.log 2>&1
  echo "rc=$?" >> $out/${tag}_gputest.log
  python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1
fi
if [[ " $what " == *" bench "* ]]; then
  for c in 3 1 2 0; do
    timeout 900 python bench.py --config $c > $out/${tag}_bench_cfg$c.json 2> $out/${tag}_bench_cfg$c.err
    echo "cfg$c rc=$?" >> $out/${tag}_bench_rc.txt
  done
  timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $out/${tag}_bench_reference.json 2>&1
  timeout 900 python bench.py --sweep > $out/${tag}_sweep.json 2> $out/${tag}_sweep.err
fi
if [[ " $what " == *" ncu "* ]]; then
  for c in 3 1; do
    cmd="python bench.py --config $c --no-parity --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3"
    $cmd > $out/${tag}_plain_cfg$c.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $out/${tag}_cfg${c}_launches.csv $cmd > $out/${tag}_ncu_launch_cfg$c.log 2>&1
    $cmd > $out/${tag}_plain2_cfg$c.log 2>&1 && \
    ncu --set full --clock-control none --import-source on \
        -k regex:"k_resolve|k_list_knn|k_bucket_list|k_tree_list" -s 8 -c 4 \
        -o $out/${tag}_cfg${c}_full $cmd > $out/${tag}_ncu_full_cfg$c.log 2>&1
  done
  cmd="python bench.py --config 2 --no-parity --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3"
  $cmd > $out/${tag}_plain_cfg2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $out/${tag}_cfg2_launches.csv $cmd > $out/${tag}_ncu_launch_cfg2.log 2>&1
  for kern in k_orphans k_count_b k_fill_b k_field_cand; do
    ncu --set full --clock-control none --import-source on -k regex:"^${kern}$" -c 1 \
        -o $out/${tag}_cfg2_${kern} $cmd > $out/${tag}_ncu_${kern}.log 2>&1
  done
fi
