"""Time the bench's time-step regime (bench.timestep_regime: 512^3, 7,417
spheres, s_f = 2, V(3,3)) and print its JSON: python scripts/timestep_time.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1410_6609_b200 import mg  # noqa: E402
from paper_1410_6609_b200 import workloads as W  # noqa: E402

st = torch.cuda.Stream()
r = bench.timestep_regime(mg, W, st, 0)
print(json.dumps({k: r[k] for k in ("value", "ms_per_step", "breakdown_ms")}), flush=True)
