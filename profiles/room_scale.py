"""Room-scale stress case (8 x 8 x 3 m room, 200 k points, r 0.01-0.08):
query step time and list sizes for the field-size variants named on the
command line (CAPT_LIB_VARIANT builds), plus a parity check of 1 M spheres
against the oracle.  Prints one JSON line per variant."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02807_b200 as P
from paper_2406_02807_b200 import _lib, workloads as W
import ctypes

cloud = W.room_cloud()
c, r = W.room_queries(cloud)
tree = P.construct(P.PointCloud(cloud), P.BuildParams(0.01, 0.08))
f = tree.clearance_field()
cd, rd = torch.from_numpy(c).cuda(), torch.from_numpy(r).cuda()
s = torch.cuda.current_stream()
for _ in range(3):
    w = P.query_bits(tree, cd, rd, 1, stream=s.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(50):
    P.query_bits(tree, cd, rd, 1, out=w, stream=s.cuda_stream)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 50
lc = (ctypes.c_uint32 * 3)()
_lib.lib().capt_field_list_counts(ctypes.c_void_p(s.cuda_stream), lc)
from oracle import oracle as O
ref = O.construct(cloud, 0.01, 0.08)
m = 1 << 20
got = np.unpackbits(w.cpu().numpy().view(np.uint8), bitorder="little")[:m].astype(bool)
mism = int((got != O.collides_many(ref, c[:m], r[:m])).sum())
print(json.dumps({"variant": os.environ.get("CAPT_LIB_VARIANT", ""), "cells": f["n_cells"],
                  "h": float(f["h"]), "ms": ms, "q_per_s": len(r) / ms * 1e3,
                  "list": list(lc), "mismatches_1M": mism}))
