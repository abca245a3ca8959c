#!/usr/bin/env python3
"""C1 eval_batch through bench.run_c1 alone (back-to-back launches and the
same launches as one CUDA graph), one JSON line per variant."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1901_04162_b200 as gk  # noqa: E402

res = bench.run_c1(gk, gk.Context.get(0))
for key, v in res.items():
    if isinstance(v, dict):
        print(f"{key:22s} {v['us_per_batch']:7.2f} us ({v['hbm_frac']:.3f})  graph "
              f"{v['graph_us_per_batch']:7.2f} us ({v['graph_hbm_frac']:.3f})")
print(json.dumps({k: v for k, v in res.items() if not isinstance(v, dict)}))
