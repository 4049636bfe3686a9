#!/usr/bin/env python
"""A/B of solve time between library builds in ONE process series on one box:
    python tools/ab_solve.py --m 128 --libs a.so b.so --rounds 4
    python tools/ab_solve.py --m 128 --libs AMGP_PDL=0 AMGP_PDL=1   (env settings instead of builds)
Each round runs every lib in a fresh subprocess (median of 7 solves)."""
import argparse, json, os, subprocess, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, statistics
sys.path.insert(0, sys.argv[1])
import torch, paper_2407_09848_b200 as P
m = int(sys.argv[2]); fam = sys.argv[3]
D0 = P.poisson3d_device(m)
h = P.build_hierarchy(D0, smoother=P.PolySmootherConfig(family=fam, degree=4))
b = torch.ones(D0.nrows, dtype=torch.float64, device="cuda")
pre = P.as_vcycle_preconditioner(h)
c = D0.ctx
P.solve(D0, b, precond=pre, cfg=P.KrylovConfig(tol=1e-6))
ts = []
for _ in range(7):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(c.stream); _, rep = P.solve(D0, b, precond=pre, cfg=P.KrylovConfig(tol=1e-6)); e1.record(c.stream)
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(json.dumps({"ms": statistics.median(ts), "it": rep.iterations}))
'''
ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=128)
ap.add_argument("--family", default="opt_cheb1")
ap.add_argument("--libs", nargs="+", required=True)
ap.add_argument("--rounds", type=int, default=3)
a = ap.parse_args()
res = {l: [] for l in a.libs}
for r in range(a.rounds):
    for l in a.libs:
        env = dict(os.environ)
        if "=" in l:
            k, v = l.split("=", 1)
            env[k] = v
        elif l != "default":
            env["AMGP_LIB"] = l
        out = subprocess.run([sys.executable, "-c", CHILD, REPO, str(a.m), a.family], capture_output=True, text=True, env=env)
        line = [x for x in out.stdout.splitlines() if x.startswith("{")]
        res[l].append(json.loads(line[-1])["ms"] if line else None)
for l, v in res.items():
    print(os.path.basename(l), [round(x, 3) if x else None for x in v])
