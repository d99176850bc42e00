"""Per-warp clock64 timeline of block 0 (cluster 0, rank 0) of the decode
kernel: every warp stamps phase boundaries of the first TL_N joint rounds and
predictor steps (decode.cuh tl_* hooks, buffer passed as ll_options.timeline).

    python tools/timeline.py [config]          (GPU box)

Prints, per phase, the critical-path increment (latest warp at this boundary
minus latest warp at the previous one) and the warp skew at the boundary,
averaged over the recorded events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2406_06220_b200 import build as llbuild
from paper_2406_06220_b200 import ll
_exp = [a[2:] for a in sys.argv if a.startswith("--exp")]   # --exp1 -> variant timeline_exp1 (-DLL_EXP1)
ll.LIB_PATH = llbuild.build(variant="timeline" + "".join("_" + e for e in _exp))   # timeline hooks compiled in
TL_N, TL_PH, NW = 128, 16, 10
NBLK = 160   # one record per block (the decode grid has <= 148 blocks)
buf = torch.zeros(NBLK * 2 * TL_N * TL_PH * NW, dtype=torch.int64, device="cuda")
ll.ll_set_options(ll.options(timeline=buf.data_ptr()).opts)   # this thread, for every decode below
import bench
from paper_2406_06220_b200.decoder import LabelLoopingDecoder, Model

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "fc-rnnt"
spec, w, enc, lengths = bench.workload(cfg, 1000)
if "--sorted" in sys.argv:   # longest utterances first: cluster 0 (block 0) decodes the critical group
    order = np.argsort(-lengths, kind="stable")
    enc, lengths = np.ascontiguousarray(enc[order]), np.ascontiguousarray(lengths[order])
model = Model(w, spec.pred_kind, spec.context, spec.blank_id, spec.durations, "bf16")
dec = LabelLoopingDecoder(model, spec.max_symbols, enc.shape[0], enc.shape[1])
e = torch.from_numpy(enc).to("cuda", torch.bfloat16); l = torch.from_numpy(lengths).cuda()
import time
for _ in range(3):
    buf.zero_()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    dec.decode(e, l)
    ev1.record()
    torch.cuda.synchronize()
print("decode ms (timeline build):", round(ev0.elapsed_time(ev1), 4))
torch.cuda.synchronize()
print(cfg, dec.stats())
allb = buf.cpu().numpy().reshape(NBLK, 2, TL_N, TL_PH, NW).astype(np.float64)
_blk = [int(a.split("=")[1]) for a in sys.argv if a.startswith("--block=")]
tl = allb[_blk[0] if _blk else 0]
if "--ranks" in sys.argv:   # per rank of cluster 0: own phase durations (clock64 is per SM: no cross-SM deltas)
    print("\nper rank of cluster 0 (averages over rounds, cycles):  build_z  MMA  epilogue  send  wait(others)  decide")
    for r in range(16):
        x = allb[r][0]
        ev = [i for i in range(TL_N) if all((x[i, ph] > 0).any() for ph in (1, 11, 12, 13, 4, 5, 6, 9))]
        if not ev:
            continue
        def d(a, b):
            return np.mean([x[i, b][x[i, b] > 0].max() - x[i, a][x[i, a] > 0].max() for i in ev])
        print(f"  rank {r:2d}: {d(1, 11):7.0f} {d(3, 12):7.0f} {d(12, 4):8.0f} {d(4, 5):6.0f} {d(5, 6):9.0f} {d(8, 9):8.0f}   ({len(ev)} rounds)")

def report(area, name, order, labels):
    x = tl[area]
    ev = [i for i in range(TL_N) if (x[i, order[0]] > 0).any() and (x[i, order[-1]] > 0).any()]
    print(f"\n{name}: {len(ev)} events recorded")
    tot = np.zeros(len(order))
    skew = np.zeros(len(order))
    ev = [i for i in ev if all((x[i, ph] > 0).any() for ph in order)]   # events with every stamp
    for i in ev:
        mx = [x[i, ph][x[i, ph] > 0].max() for ph in order]
        mn = [x[i, ph][x[i, ph] > 0].min() for ph in order]
        for k in range(1, len(order)):
            tot[k] += mx[k] - mx[k - 1]
            skew[k] += mx[k] - mn[k]
    n = max(1, len(ev))
    for k in range(1, len(order)):
        print(f"  {labels[k]:28s} {tot[k]/n:8.0f} cyc   (warp skew at end {skew[k]/n:6.0f})")
    print(f"  {'TOTAL':28s} {tot.sum()/n:8.0f} cyc")
    # next-event gap: from the last stamp of event i to the first of event i+1
    gaps = [x[ev[j + 1], order[0]][x[ev[j + 1], order[0]] > 0].max() - x[ev[j], order[-1]].max()
            for j in range(len(ev) - 1) if ev[j + 1] == ev[j] + 1]
    if gaps:
        print(f"  {'(gap to next event)':28s} {np.median(gaps):8.0f} cyc median")
    return ev

if "--tj" in sys.argv:   # the tcgen05 joint: stamps 11 (build_z before its proxy fence), 12 (joint MMAs done)
    report(0, "joint rounds", [0, 1, 11, 2, 15, 3, 12, 13, 4, 5, 6, 7, 8, 9, 10],
           ["", "wait_f/plan (+sync)", "build_z", "proxy fence", "sync", "spec issue", "joint MMA (post..done)",
            "epilogue TMEM+bfly (w0-3)", "epilogue end (all)", "exchange send", "exchange wait", "resolve", "sync (bar)",
            "decide", "sync+reload (bar)"])
    
else:
    report(0, "joint rounds", list(range(11)),
           ["", "wait_f/plan (+sync)", "build_z", "sync (bar)", "spec issue + joint", "exchange send",
            "exchange wait", "resolve", "sync (bar)", "decide", "sync+reload (bar)"])
if "--tj" in sys.argv:
    report(1, "tick (predictor + the windows around it)", [11, 12, 8, 0, 1, 2, 3, 4, 9, 10, 5, 6, 7, 13],
           ["", "spec wait + window plan + sync", "reload issue", "outer-step entry", "gate read + E' wait", "cell update",
            "sync (bar)", "h' exchange", "W_pred partial MMA", "sync (bar)", "W_pred reduce + g bcast", "sync (bar)",
            "g exchange + sync", "lists + reload wait"])
if "--sub" in sys.argv:   # warp 0's finish_round_rnnt sub-phases (slot 14, columns 1..6)
    x = tl[0]
    ev = [i for i in range(TL_N) if x[i, 8, 0] > 0 and all(x[i, 14, k] > 0 for k in range(1, 7))]
    labs = ["load state + decisions", "append + state store", "lists + counters", "plan_next_tj", "reload list", "E' issue"]
    prev = [x[i, 8, 0] for i in ev]
    print(f"\nfinish_round_rnnt sub-phases ({len(ev)} rounds)")
    for k in range(1, 7):
        cur = [x[i, 14, k] for i in ev]
        print(f"  {labs[k - 1]:28s} {np.mean(np.array(cur) - np.array(prev)):8.0f} cyc")
        prev = cur
    print(f"  {'to stamp 9':28s} {np.mean([x[i, 9, 0] - x[i, 14, 6] for i in ev]):8.0f} cyc")
if "--gate" in sys.argv:   # background gate batch vs the joint post (slot 14: col 7 pending flag, 8 post time, 9 gate done)
    x = tl[0]
    ev = [i for i in range(TL_N) if x[i, 14, 7] > 0]
    pend = [i for i in ev if x[i, 14, 7] == 2]
    print(f"\ngate batch still running at the joint post: {len(pend)} of {len(ev)} rounds")
    lag = [x[i, 14, 9] - x[i, 14, 8] for i in pend if x[i, 14, 9] > 0]
    if lag:
        print(f"  gate done after the post by {np.mean(lag):.0f} cyc on average (max {np.max(lag):.0f})")
report(1, "predictor steps", [8, 0, 1, 2, 3, 4, 9, 10, 5, 6, 7],
       ["", "outer-step entry", "first gate tile", "rest tiles + E' wait", "sync (bar)", "h' exchange",
        "W_pred partial MMA", "sync (bar)", "W_pred reduce + g bcast", "sync (bar)", "g exchange + sync"])
