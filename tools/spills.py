"""Registers / spills of every decode_kernel instantiation from the last build's ptxas output."""
import re
import sys

s = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2406_06220_b200/ptxas_info.txt").read()
for b in re.split(r"ptxas info    : Compiling entry function", s)[1:]:
    name = b.split("'")[1]
    if "decode_kernel" not in name:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", b)
    r = re.search(r"Used (\d+) registers", b)
    args = re.search(r"decode_kernelI(.*?)EEv", name)
    print(f"{args.group(1) if args else name[:60]:60s} regs {r.group(1) if r else '?':>4} spill st/ld {m.groups() if m else None}")
