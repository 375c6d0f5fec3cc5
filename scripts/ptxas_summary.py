"""Summarise ptxas -v output: registers / stack / spills per solve kernel."""
import re, subprocess, sys
txt = open(sys.argv[1] if len(sys.argv) > 1 else 'build/ptxas_libodegpu.txt').read()
pat = re.compile(r"Compiling entry function '(\S+)' for 'sm_100a'\s*\n(?:ptxas info\s*: .*\n)*?ptxas info\s*: Function properties for \S+\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\nptxas info\s*: Used (\d+) registers")
for m in pat.finditer(txt):
    name = m.group(1)
    if 'solve_kernel' not in name:
        continue
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    mm = re.search(r'guarded_solve_kernel<([\w:<>]+?), \(odegpu::Algorithm\)(\d)', dem)
    label = (f"{mm.group(1).replace('odegpu::models::', '').replace('odegpu::fakes::', 'fakes::')} "
             f"{'RK4' if mm.group(2) == '0' else 'RKCK45'}") if mm else dem[:60]
    print(f"{label:40s} regs {m.group(5):>4s}  stack {m.group(2):>3s}  spill st/ld {m.group(3)}/{m.group(4)}")
