# build-time variants: build tests, then the warm build time of configs 3, 1, 2 per library
set -u
tag=${1:-bi}
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_filter.py -q -x > gpurun_out/${tag}_tests.log 2>&1; echo rc=$? >> gpurun_out/${tag}_tests.log
for v in "" ${VARIANTS:-}; do
  CAPT_LIB_VARIANT=$v python - >> gpurun_out/${tag}_build.jsonl 2>> gpurun_out/${tag}_build.err <<'PY'
import json, os, time, torch, sys
sys.path.insert(0, '.')
import paper_2406_02807_b200 as P
from paper_2406_02807_b200 import workloads as W
out = {"variant": os.environ.get("CAPT_LIB_VARIANT", "")}
for name, cloud, band in (("cfg3", W.cfg3_cloud(), (0.01, 0.1)), ("cfg1", W.cfg1_cloud(), (0.02, 0.08))):
    P.construct(P.PointCloud(cloud), P.BuildParams(*band)); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); tr = P.construct(P.PointCloud(cloud), P.BuildParams(*band)); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3); del tr
    out[name] = min(ts)
print(json.dumps(out))
PY
done
