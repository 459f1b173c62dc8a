"""C1 graph latency (bench.c1_graph_latency) printed for the current TTC_SMALL_THREADS setting."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2109_00626_b200 as ttc  # noqa: E402

r = bench.c1_graph_latency(ttc, torch.device("cuda:0"), 20210901)
print(json.dumps({k: round(v, 3) for k, v in r.items() if k.startswith("us_per_call")}))
