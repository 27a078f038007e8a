# One ncu --set full capture (with source) of K0 on config $1
set -u
c=${1:-3}; tag=${2:-src}
cmd="python bench.py --config $c --no-parity --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3"
$cmd > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_resolve|k_list_knn|k_bucket_list|k_tree_list" -s 3 -c 3 -o gpurun_out/${tag}_cfg$c $cmd > gpurun_out/${tag}_ncu.log 2>&1
