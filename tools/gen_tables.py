"""Regenerate the measurement table of DESIGN.md §7 and the headline table of
profiles/README.md from the committed bench lines (profiles/<tag>_bench_*.json).

    python tools/gen_tables.py [tag]      # rewrites the two tables in place
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
ROWS = [
    ("fc-rnnt", "fc-rnnt (config 2, headline)"),
    ("fc-tdt", "fc-tdt (config 3)"),
    ("stateless-b512", "stateless-b512 (config 4)"),
    ("sweep-rnnt", "sweep-rnnt (config 5, 8192 utt)"),
    ("sweep-tdt", "sweep-tdt (config 5, 8192 utt)"),
    ("sweep-rnnt_b32x4", "sweep-rnnt as B=32 launches on 4 streams"),
    ("fc-rnnt-4x", "fc-rnnt-4x (4× subsampling, 40 ms frames, T ≈ 500)"),
    ("fc-rnnt_alg3-batched", "fc-rnnt, Alg. 3 batched outer loop (--schedule batched)"),
    ("fc-tdt_alg3-batched", "fc-tdt, Alg. 3 batched outer loop"),
    ("fc-rnnt_frame-looping", "fc-rnnt, **frame-looping baseline** (Alg. 2)"),
    ("stateless-b512_frame-looping", "stateless-b512, frame-looping baseline"),
    ("fc-rnnt-4x_frame-looping", "fc-rnnt-4x, frame-looping baseline"),
]


def load(name):
    p = os.path.join(ROOT, "profiles", f"{TAG}_bench_{name}.json")
    if not os.path.exists(p):
        return None
    lines = [l for l in open(p) if l.strip().startswith("{")]
    return json.loads(lines[-1]) if lines else None


def main():
    out = ["| config | audio-s/s | ms / step | utt/s | e2e audio-s/s | oracle (16 host cores) |",
           "|---|---|---|---|---|---|"]
    d = {}
    for key, label in ROWS:
        j = load(key)
        if j is None:
            continue
        d[key] = j
        cpu = j.get("cpu_baseline") or {}
        cpu_s = f"{cpu['value']:,.0f}" if cpu.get("value") else "—"
        out.append(f"| {label} | {j['value']:,.0f} | {j['ms_per_step']:.3f} | {j['utterances_per_s']:,.0f} | "
                   f"{j['e2e']['value']:,.0f} | {cpu_s} |")
    table = "\n".join(out)
    p = os.path.join(ROOT, "DESIGN.md")
    s = open(p).read()
    s = re.sub(r"\| config \| audio-s/s \| ms / step.*?\n\n", table + "\n\n", s, count=1, flags=re.S)
    open(p, "w").write(s)

    h = d["fc-rnnt"]
    fl, b3 = d.get("fc-rnnt_frame-looping"), d.get("fc-rnnt_alg3-batched")
    rf = h["roofline"]
    share = rf.get("kernel_share_of_step")
    rows = [
        ("decoded audio-s/s (device, inputs resident)",
         f"{h['value']:,.0f} ({h['ms_per_step']:.3f} ms per {h['config'].get('audio_s_per_step', 0):.1f} audio-s batch)"),
        ("utterances/s", f"{h['utterances_per_s']:,.0f}"),
        ("e2e through the public API (H2D of enc + D2H of hypotheses timed)", f"{h['e2e']['value']:,.0f} audio-s/s"),
        ("float64 oracle on the box's 16 host cores (same batch)", f"{h['cpu_baseline']['value']:,.0f} audio-s/s"),
    ]
    if b3:
        rows.append(("the paper's batched outer loop (Alg. 3 as listed, --schedule batched)", f"{b3['value']:,.0f} audio-s/s"))
    if fl:
        rows.append(("frame-looping baseline (Alg. 2) on the same kernels",
                     f"{fl['value']:,.0f} audio-s/s (label-looping {h['value'] / fl['value']:.2f}x faster"
                     + (f"; {b3['value'] / fl['value']:.2f}x with the batched loop)" if b3 else ")")))
    if share:
        rows.append(("decode_kernel share of the step (CUDA events)", f"{100 * share:.0f}%"))
    rows.append((f"roofline ({rf['bound']}, of measured {rf['peak']} {rf['unit']} bf16)",
                 f"{100 * rf['frac']:.1f}% — latency-bound, see DESIGN.md §7"))
    t2 = "| | value |\n|---|---|\n" + "\n".join(f"| {a} | {b} |" for a, b in rows)
    p = os.path.join(ROOT, "profiles", "README.md")
    s = open(p).read()
    s = re.sub(r"\| \| value \|\n\|---\|---\|\n.*?\n\n", t2 + "\n\n", s, count=1, flags=re.S)
    open(p, "w").write(s)
    print(table)
    print()
    print(t2)


if __name__ == "__main__":
    main()
