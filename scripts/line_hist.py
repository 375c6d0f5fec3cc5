"""Executed warp instructions per CUDA source line: joins an ncu SASS source
page (per-address execution counts) with the line table of the same cubin
(nvdisasm -g). Usage:
  python scripts/line_hist.py src.csv kernel.cubin mangled_kernel_name [top]"""
import collections, csv, re, subprocess, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
counts = []
for r in rows[2:]:
    try:
        counts.append((int(r[0], 16), int(r[ie]), r[src].strip()))
    except ValueError:
        pass
base = counts[0][0]
exe = {a - base: (n, s) for a, n, s in counts}
full = subprocess.run(["nvdisasm", "-g", sys.argv[2]], capture_output=True, text=True).stdout
start = full.index(f"\n.text.{sys.argv[3]}:")
end = full.find("//---------------------", start)
dis = full[start:end if end > 0 else len(full)]
cur = "?"
per_line = collections.Counter()
fp = collections.Counter()
for ln in dis.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/\s+(.*)', ln)
    if m:
        off = int(m.group(1), 16)
        if off in exe:
            n, s = exe[off]
            per_line[cur] += n
            if re.search(r'\b(DFMA|DMUL|DADD|DSETP)\b', s):
                fp[cur] += n
tot = sum(per_line.values())
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
for k, v in per_line.most_common(top):
    print(f"{100 * v / tot:6.2f}%  fp64 {100 * fp[k] / max(v, 1):5.1f}%  {k}")
