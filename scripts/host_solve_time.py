import os, sys, time, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import bench
import paper_1710_08679_b200 as ts
for rep in range(2):
    g = bench.gpu_solve(ts, torch, (140, 210, 70), bench.THREE_LAYER, 16, 31)
    print(json.dumps({k: g[k] for k in ("setup_s", "solve_s", "device_solve_s", "s_per_case", "device_s_per_case")}), flush=True)
