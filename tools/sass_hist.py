"""Histogram of an ncu source-page SASS dump (ncu --page source --csv --print-source sass):
instructions executed and stall samples per opcode, plus the hottest instructions."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS, iN, iI = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
ops = collections.Counter(); smp = collections.Counter(); stalls = collections.Counter()
tot_i = tot_s = 0
body = []
for r in rows[2:]:
    if len(r) <= iI or not r[iI].strip().isdigit():
        continue
    src = r[iS].strip()
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    op = op.split(".")[0]
    n = int(r[iI]); s = int(r[iN] or 0)
    ops[op] += n; smp[op] += s; tot_i += n; tot_s += s
    for c in stall_cols:
        try: stalls[hdr[c]] += int(r[c] or 0)
        except ValueError: pass
    body.append((s, n, r[0], src))
print(f"total warp-instructions {tot_i:.4g}, stall samples {tot_s}")
print("opcode            instr%   samples%")
for op, n in ops.most_common(40):
    print(f"{op:16s} {100*n/tot_i:7.2f} {100*smp[op]/max(tot_s,1):9.2f}")
print("\nstall reasons (samples):")
for k, v in stalls.most_common(15):
    print(f"  {k:40s} {100*v/max(tot_s,1):6.2f}%")
print("\nhottest instructions by samples:")
for s, n, a, src in sorted(body, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{s:8d} {n:12d} {a} {src}")
