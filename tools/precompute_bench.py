"""Time the GPU offline precompute on a BASELINE-shaped volume.

python tools/precompute_bench.py --config c3 [--dims 64,64,64] [--m 150] [--degree 24]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1607_04174_b200 as swb  # noqa: E402
from paper_1607_04174_b200 import workloads as W  # noqa: E402
from paper_1607_04174_b200.precompute import precompute  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--dims", default=None)
ap.add_argument("--m", type=int, default=None)
ap.add_argument("--degree", type=int, default=24)
ap.add_argument("--tol", type=float, default=1e-6)
a = ap.parse_args()
dims = tuple(int(x) for x in a.dims.split(",")) if a.dims else None
w = W.make_image(a.config, dims)
p = w.params
m = a.m or p["m"]
img = swb.Image(w.dims, w.intensities)
torch.cuda.synchronize()
t0 = time.perf_counter()
pack = precompute(img, p["beta0"], m, eig_tol=a.tol, connectivity=p["connectivity"], weight_mode=p["weight_mode"],
                  degree=a.degree)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
info = dict(pack.solver_info)
hist = info.pop("history", [])
print(json.dumps({"config": a.config, "dims": w.dims, "m": m, "seconds": dt, "lam_head": pack.values[:4].tolist(),
                  "lam_m": float(pack.values[-1]), **info, "last": hist[-3:]}))
