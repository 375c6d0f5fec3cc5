"""Per-opcode histogram of executed warp instructions from an ncu source page
(ncu -i X.ncu-rep --page source --csv --print-source sass).
Usage: python scripts/sass_hist.py src.csv [trial_steps] [--listing]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ie = hdr.index("Instructions Executed"); src = hdr.index("Source"); samp = hdr.index("Warp Stall Sampling (All Samples)")
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
ops = collections.Counter(); tot = 0; stall = collections.Counter()
seq = []
for r in rows[2:]:
    try: n = int(r[ie])
    except ValueError: continue
    s = r[src].strip()
    op = s.split()[0]
    if op.startswith("@"): op = s.split()[1]
    op = op.split(".")[0].rstrip(";")
    ops[op] += n; tot += n; stall[op] += int(r[samp] or 0)
    seq.append((r[0], s, n, int(r[samp] or 0)))
fp64 = sum(v for k, v in ops.items() if k in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"))
print(f"total warp instr {tot:.4g}  per trial step (x32 lanes) {tot*32/steps:.1f}; fp64 share {fp64/tot:.3f}")
for k, v in ops.most_common(30):
    print(f"{k:10s} {v/tot*100:6.2f}%  per-step {v*32/steps:8.1f}  stall-samples {stall[k]}")
if "--listing" in sys.argv:
    for a, s, n, st in seq:
        print(f"{a[-5:]} {n:>11d} {st:>6d}  {s}")
