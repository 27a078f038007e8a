#!/bin/bash
# Turn the outputs of `bash profiles/gpu_run.sh <tag> tests bench ncu` (merged
# back into gpurun_out/) into the committed r02_* evidence files.
#   bash profiles/refresh.sh <tag>
set -eu
T=${1:?tag}; G=gpurun_out
for c in 3 1 2; do python profiles/summarize.py launches $G/${T}_cfg${c}_launches.csv profiles/r02_cfg${c}_launches.md; done
python profiles/summarize.py full $G/${T}_cfg3_full.ncu-rep profiles/r02_cfg3_ncu_full.json
python profiles/summarize.py full $G/${T}_cfg1_full.ncu-rep profiles/r02_cfg1_ncu_full.json
python - "$T" <<'PY'
import json, sys
sys.path.insert(0, "profiles")
import summarize
res = []
for k in ("k_orphans", "k_count_b", "k_fill_b", "k_field_cand"):
    summarize.full(f"gpurun_out/{sys.argv[1]}_cfg2_{k}.ncu-rep", "/tmp/_x.json")
    res += json.load(open("/tmp/_x.json"))
json.dump(res, open("profiles/r02_cfg2_preprocess_ncu_full.json", "w"), indent=1)
PY
for c in 3 1 2 0; do cp $G/${T}_bench_cfg$c.json profiles/r02_bench_cfg$c.json; done
cp $G/${T}_bench_reference.json profiles/r02_bench_reference.json
cp $G/${T}_sweep.json profiles/r02_sweep.json
cp $G/${T}_gputest.log profiles/r02_gpu_tests.log
cp $G/${T}_smoke.log profiles/r02_smoke.log
cp $G/${T}_host.txt profiles/r02_host.txt
python profiles/k0_source_table.py $G/${T}_cfg3_full.ncu-rep k_resolve1 profiles/r02_k0_cfg3_source.md \
  "K0 (k_resolve1<1>) on config 3: per-source-line executed instructions and stall samples (ncu --set full --import-source on; profiles/gpu_run.sh)"
python profiles/k0_source_table.py $G/${T}_cfg1_full.ncu-rep k_resolve1 profiles/r02_k0_cfg1_source.md \
  "K0 (k_resolve1<8>, groups of 8) on config 1: per-source-line executed instructions and stall samples"
[ -f $G/${T}_k0_paths.json ] && cp $G/${T}_k0_paths.json profiles/r02_k0_paths.json || true
