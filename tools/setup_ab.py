#!/usr/bin/env python
"""Device-setup time A/B between library builds (GPU box):
    python tools/setup_ab.py --m 256 --libs default path/to/variant.so
Each lib in a fresh subprocess: setup time of build_hierarchy (median of 3)
and a digest of every level (must agree across builds)."""
import argparse, json, os, subprocess, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, time, hashlib, statistics
sys.path.insert(0, sys.argv[1])
import torch, numpy as np, paper_2407_09848_b200 as P
m = int(sys.argv[2])
ts = []
for _ in range(3):
    D0 = P.poisson3d_device(m)
    torch.cuda.synchronize(); t = time.perf_counter()
    h = P.build_hierarchy(D0, smoother=P.PolySmootherConfig(family="opt_cheb1", degree=4))
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
hs = hashlib.sha256()
for lv in h.levels:
    H = lv.A.to_csr(); hs.update(H.values.tobytes()); hs.update(H.col_idx.tobytes())
print(json.dumps({"setup_s": statistics.median(ts), "all": ts, "digest": hs.hexdigest()[:16]}))
'''
ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=256)
ap.add_argument("--libs", nargs="+", required=True)
a = ap.parse_args()
for l in a.libs:
    env = dict(os.environ)
    if l != "default":
        env["AMGP_LIB"] = l
    out = subprocess.run([sys.executable, "-c", CHILD, REPO, str(a.m)], capture_output=True, text=True, env=env)
    line = [x for x in out.stdout.splitlines() if x.startswith("{")]
    print(os.path.basename(l), line[-1] if line else out.stderr[-500:], flush=True)
