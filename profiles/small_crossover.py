import sys, json, torch, numpy as np
sys.path.insert(0, ".")
import paper_2406_02807_b200 as P
from paper_2406_02807_b200 import workloads as W, _lib
from paper_2406_02807_b200.query import query_bits
for name, pts, rr, qf in (("cfg1", W.cfg1_cloud(), (0.02, 0.08), None), ("cfg3", W.cfg3_cloud(), (0.01, 0.1), None)):
    tree = P.construct(P.PointCloud(pts), P.BuildParams(*rr), device=0)
    for n in (1 << 18, 3 << 17, 1 << 19, 5 << 17, 3 << 18, 7 << 17, (1 << 20) - 128):
        if name == "cfg1":
            c, r = W.cfg1_queries(pts, n_groups=n, lane_width=1, seed=3)
        else:
            c, r = W.cfg3_queries(n)
        dc, dr = torch.from_numpy(c).cuda(), torch.from_numpy(r).cuda()
        out = {}
        for label, mode in (("small", 0), ("pipeline", _lib.MODE_FIELD)):
            for _ in range(5): query_bits(tree, dc, dr, mode=mode)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(50): query_bits(tree, dc, dr, mode=mode)
            e1.record(); torch.cuda.synchronize()
            out[label] = round(e0.elapsed_time(e1) / 50 * 1e3, 2)
        print(name, n, out)
