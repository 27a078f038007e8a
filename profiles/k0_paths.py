"""K0 device-resident timings of the less common paths on the config-3 cloud:
float64 inputs, lane masks, lane widths 2 and 32 (profiles/, experiment
runner: python profiles/k0_paths.py)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2406_02807_b200 as P  # noqa: E402
from paper_2406_02807_b200 import workloads as W  # noqa: E402
from paper_2406_02807_b200.query import query_bits  # noqa: E402

pts = W.cfg3_cloud()
tree = P.construct(P.PointCloud(pts), P.BuildParams(0.01, 0.1), device=0)
n = 1 << 24
c, r = W.cfg3_queries(n)
dc, dr = torch.from_numpy(c).cuda(), torch.from_numpy(r).cuda()
mask = (torch.rand(n, device="cuda") > 0.1).to(torch.uint8)
res = {}


def timeit(name, **kw):
    for _ in range(3):
        query_bits(tree, kw.get("c", dc), kw.get("r", dr), lane_width=kw.get("L", 1),
                   lane_mask=kw.get("m"))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        query_bits(tree, kw.get("c", dc), kw.get("r", dr), lane_width=kw.get("L", 1),
                   lane_mask=kw.get("m"))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res[name] = {"ms": ms, "G_spheres_per_s": n / ms / 1e6}


timeit("fp32 L=1")
timeit("fp32 L=1 masked", m=mask)
timeit("fp32 L=2", L=2)
timeit("fp32 L=8", L=8)
timeit("fp32 L=8 masked", L=8, m=mask)
timeit("fp32 L=32", L=32)
timeit("fp64 L=1", c=dc.double(), r=dr.double())
print(json.dumps({"n": n, "paths": res}, indent=1))
