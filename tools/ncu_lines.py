"""Aggregate an ncu source export (--page source --csv --print-source cuda,sass)
by CUDA source line: warp-stall samples, top stall reasons, shared wavefronts.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [top]"""
import csv, sys, collections

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = collections.defaultdict(lambda: collections.Counter())
src = {}
fname, hdr = "?", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].strip().isdigit():
        continue
    key = (fname, int(r[0]))
    if r[1].strip():
        src[key] = r[1].strip()
    c = agg[key]
    for i, h in enumerate(hdr[4:], start=4):
        try:
            c[h] += float(r[i] or 0)
        except ValueError:
            pass
S = "Warp Stall Sampling (All Samples)"
tot = sum(c[S] for c in agg.values()) or 1
print(f"total samples {tot:.0f}")
for key, c in sorted(agg.items(), key=lambda kv: -kv[1][S])[:top]:
    reasons = sorted(((h, v) for h, v in c.items() if h.startswith("stall_") and "Not Issued" not in h), key=lambda x: -x[1])[:3]
    rs = " ".join(f"{h[6:]}:{v / max(c[S], 1) * 100:.0f}%" for h, v in reasons if v > 0)
    wf = c.get("L1 Wavefronts Shared", 0)
    print(f"{c[S] / tot * 100:5.1f}% {key[0]}:{key[1]:<5} wf={wf:>9.0f} {rs:40s} {src.get(key, '')[:90]}")
