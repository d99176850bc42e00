"""Tick-count model of the per-row tick schedule (CPU, no GPU): for the planted
config-2 batch (the bench workload), every tick each active row evaluates a
window of W frames and stops at its first planted label (the next round
re-evaluates that frame after the predictor step) or advances W frames.  The
group needs max over its rows of their rounds; the kernel, the max over groups
(the critical cluster).  Used to size window policies before building them
(DESIGN.md §7): W=6 reproduces the measured 102 ticks / 16585 joint rows.

    python tools/tick_sim.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def sim(rows_in, lengths, planted, policy):
    rows = [dict(L=int(lengths[b]), t=0, pend=sorted(planted[b][1]), active=True) for b in rows_in]
    ticks = evals = 0
    while any(r["active"] for r in rows):
        ticks += 1
        act = [r for r in rows if r["active"]]
        W = policy(len(act))
        for r in act:
            lo, hi = r["t"], min(r["t"] + W, r["L"])
            evals += hi - lo
            f = next((x for x in r["pend"] if lo <= x < hi), None)
            if f is not None:
                r["pend"].remove(f)
                r["t"] = f
            else:
                r["t"] = hi
                r["active"] = r["t"] < r["L"]
    return ticks, evals


def main():
    c = synth.CONFIGS["fc-rnnt"]
    spec = c["spec"]
    _, _, lengths, planted = synth.make_planted_rnnt(spec, 1000, c["B"], c["T_max"], c["len_lo"], c["len_hi"],
                                                     rho=c.get("rho", 0.28))
    R, B = 5, c["B"]
    groups = [list(range(g * R, min(B, g * R + R))) for g in range((B + R - 1) // R)]
    for name, pol in [("W=6 (production, R=5)", lambda n: 6), ("W=8", lambda n: 8),
                      ("dynamic min(8, 32/active)", lambda n: min(8, 32 // max(n, 1))),
                      ("W=32", lambda n: 32)]:
        res = [sim(g, lengths, planted, pol) for g in groups]
        print(f"{name:28s} critical group {max(r[0] for r in res):4d} ticks; per group {[r[0] for r in res]}; "
              f"joint rows {sum(r[1] for r in res)}")


if __name__ == "__main__":
    main()
