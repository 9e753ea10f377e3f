"""Projected 1->8-GPU parallel efficiency of the sharded solve (a PROJECTION
from one-GPU measurements, not a scaling curve: only one GPU is available).

Runs W windows of a BASELINE config on one B200 and records every
subdomain's work per window (RHS evaluations x box nodes = node-updates, the
controller's own tally, Plan.sub_evals).  A window of the sharded solve
costs max over ranks of that rank's node-updates (no communication inside a
window); efficiency = total / (N x max).  Partitions compared:
  * static : distributed.partition (box-node balanced lattice blocks)
  * lpt_w0 : LPT on window-0/1 tallies, then fixed
  * lpt_dyn: LPT re-balanced every window on the previous window's tallies
             (an upper bound: ignores the cost of migrating subdomains).

    python tools/project_scaling.py C3 8 [--dtau X] [--profile stable]
"""
import argparse
import json
import sys

sys.path.insert(0, ".")
import numpy as np

import bench
import paper_2006_14602_b200 as P
from paper_2006_14602_b200.distributed import makespan, partition, partition_lpt
from paper_2006_14602_b200.plan import Plan

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("windows", type=int)
ap.add_argument("--dtau", type=float, default=None)
ap.add_argument("--profile", default="default")
a = ap.parse_args()

g, d, m = bench.case(a.config, P)
kw = dict(tol=1e-300, max_windows=a.windows, transmission="parallel")
if a.dtau:
    kw["dtau"] = a.dtau
if a.profile == "stable":
    kw.update(rtol=1e-6, atol=1e-9)
plan = Plan.for_grid(g, d.subdomains, m, P.SolverConfig(**kw))
plan.set_state(None)
nodes = np.array([np.prod(s.shape()) for s in d.subdomains], dtype=np.float64)
prev = plan.sub_evals()
per_win = []
for w in range(a.windows):
    plan.run(1, 1e-300)
    cur = plan.sub_evals()
    per_win.append((cur - prev) * nodes)
    prev = cur
per_win = np.array(per_win)
out = {"config": a.config, "windows": a.windows, "dtau": kw.get("dtau", 1e-3),
       "profile": a.profile, "note": "projection from 1-GPU per-subdomain node-update tallies",
       "per_rank_count": {}}
for world in (1, 2, 4, 8):
    st = partition(d, world)
    lpt0 = partition_lpt(d, world, per_win[:min(2, a.windows)].sum(axis=0))
    tot = per_win.sum()
    ms_static = sum(makespan(w, st, world)[0] for w in per_win)
    ms_lpt0 = sum(makespan(w, lpt0, world)[0] for w in per_win)
    ms_dyn = per_win[0].max() if world > 1 else per_win[0].sum()
    ms_dyn = makespan(per_win[0], partition_lpt(d, world, per_win[0]), world)[0]
    for i in range(1, len(per_win)):
        ms_dyn += makespan(per_win[i], partition_lpt(d, world, per_win[i - 1]), world)[0]
    out["per_rank_count"][world] = {
        "eff_static": tot / (world * ms_static), "eff_lpt_first_windows": tot / (world * ms_lpt0),
        "eff_lpt_dynamic": tot / (world * ms_dyn),
        "largest_subdomain_share": float((per_win.max(axis=1) / per_win.sum(axis=1)).mean())}
print(json.dumps(out, indent=1))
