"""Summarise ptxas -v output: registers / stack / spills per solve kernel."""
import re, sys
txt = open(sys.argv[1] if len(sys.argv) > 1 else 'build/ptxas_libodegpu.txt').read()
pat = re.compile(r"Compiling entry function '(\S+)' for 'sm_100a'\s*\n(?:ptxas info\s*: .*\n)*?ptxas info\s*: Function properties for \S+\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\nptxas info\s*: Used (\d+) registers")
for m in pat.finditer(txt):
    name = m.group(1)
    if 'solve_kernel' not in name:
        continue
    mm = re.search(r'(\d+)(\w+?Hooks)ELN\w+?AlgorithmE(\d)', name)
    label = f"{mm.group(2)} {'RK4' if mm.group(3) == '0' else 'RKCK45'}" if mm else name[:60]
    print(f"{label:36s} regs {m.group(5):>4s}  stack {m.group(2):>3s}  spill st/ld {m.group(3)}/{m.group(4)}")
