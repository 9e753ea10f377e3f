import os, subprocess, sys, collections
code = """
import paper_2006_14602_b200 as P
from paper_2006_14602_b200.plan import Plan
g = P.build_grid(2, ((0.0,1.0),)*2, (4097,4097)); d = P.build_decomposition(g,(8,8),16)
m = P.density_monitor(P.seeded_mixture(32,2), g.extents)
cfg = P.SolverConfig(tol=1e-300, max_windows=%d, transmission='parallel'%s)
plan = Plan.for_grid(g, d.subdomains, m, cfg); plan.set_state(None)
import sys
for w in range(%d):
    plan.run(1, 1e-300); print('WINDOW', w, file=sys.stderr, flush=True)
"""
W = int(sys.argv[1]); extra = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run([sys.executable, "-c", code % (W, extra, W)], env=dict(os.environ, DDPMA_TRACE="1"),
                     capture_output=True, text=True)
w = 0
stats = collections.defaultdict(lambda: [0, 0, 0, 0])   # steps, stages, rejects, flagged
for line in out.stderr.splitlines():
    if line.startswith("WINDOW"):
        tot = sorted(((v[1], k, v) for k, v in stats.items()), reverse=True)
        print(f"window {w}: stages per sub: max {tot[0][0]} (sub {tot[0][1]}), median {tot[len(tot)//2][0]}, min {tot[-1][0]}, sum {sum(t[0] for t in tot)}")
        print("   top5:", [(k, v) for _, k, v in tot[:5]])
        stats.clear(); w += 1
    elif line.startswith("TRACE") and " step " in line:
        f = line.split(); sid = int(f[1]); s = int(f[4]); acc = int(f[7]); fl = int(f[6])
        st = stats[sid]; st[0] += 1; st[1] += s + 1; st[2] += 1 - acc; st[3] += fl
print(out.stderr[-500:] if out.returncode else "")
