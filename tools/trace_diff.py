"""Debug helper: compare the device controller's decision trace
(DDPMA_TRACE=1 on stderr) with the oracle's for the first windows of C1."""
import os, subprocess, sys, re
import numpy as np
sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import ddpma_oracle as O

W = int(sys.argv[1]) if len(sys.argv) > 1 else 3
tr = sys.argv[2] if len(sys.argv) > 2 else "parallel"
g, lay, ov, mon, dom, _ = O.baseline_case("C1")
d = O.make_decomposition(g, lay, ov)
traces = {}
O.solve(g, d, mon, dom, O.Config(tol=1e-300, max_windows=W, transmission=tr), traces=traces)
code = f"""
import paper_2006_14602_b200 as P
g = P.build_grid(2, ((0.0,1.0),(0.0,1.0)), (65,65)); d = P.build_decomposition(g,(2,2),4)
m = P.density_monitor(P.RingDensity(), g.extents)
P.solve(g, d, m, P.SolverConfig(tol=1e-300, max_windows={W}, transmission='{tr}'))
"""
env = dict(os.environ, DDPMA_TRACE="1")
out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
gpu = {}
for line in out.stderr.splitlines():
    if not line.startswith("TRACE"): continue
    f = line.split()
    sid = int(f[1])
    if f[2] == "sigma": gpu.setdefault(sid, []).append(("sigma", float(f[3])))
    else: gpu.setdefault(sid, []).append((float(f[3]), int(f[4]), float(f[5]), bool(int(f[6])), bool(int(f[7]))))
for sid in sorted(traces)[:1]:
    a, b = traces[sid], gpu.get(sid, [])
    print("sub", sid, "oracle", len(a), "gpu", len(b))
    for i, (x, y) in enumerate(zip(a, b)):
        same = (x[0] == y[0]) if x[0] == "sigma" else (x[1] == y[1] and x[4] == y[4] and x[3] == y[3])
        if x[0] == "sigma" and y[0] == "sigma":
            rel = abs(x[1]-y[1])/abs(x[1])
            same = rel < 1e-9
        if not same or i < 3:
            print("  ", i, "oracle", x, "\n      gpu   ", y)
        if not same:
            for j in range(i, min(i + 25, len(a), len(b))):
                print("     ", j, a[j], "|", b[j])
            break
print(out.stderr[-2000:] if out.returncode else "")
