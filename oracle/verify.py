"""Teacher-forced verifier (TEST INFRASTRUCTURE, see oracle/__init__.py).

The north_star tolerance: token / timestamp / length sequences must match the
float64 oracle bit-exactly except at decisions whose float64 top-2 logit gap is
below `tol` (1e-3); those are flagged and accepted after re-checking in float64.
A free-running comparison would cascade after one accepted near-tie, so the
decoder under test is replayed against the float64 model along ITS OWN
decisions (SURVEY.md §8(c) "Teacher-forced verifier"):

  RNN-T: the full decision sequence is reconstructible from (tokens,
         timestamps, L, m): at each frame the labels stamped t, then a blank
         iff fewer than m labels were stamped t (Alg. 1 rules + guard A6).
  TDT:   blank skips are not recoverable from the outputs, so the replay is a
         depth-first search over the blank durations that are acceptable
         (float64 argmax or within tol); it must reach the emitted events and
         end exactly at t >= L.

A decision (y, and d for TDT) is accepted iff max(l) - l[y] < tol or y is the
lowest-index argmax (`argmax_lowest`).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np

from .model import Transducer, argmax_lowest, log_prob


@dataclasses.dataclass
class VerifyResult:
    ok: bool
    decisions: int = 0
    near_ties: int = 0
    message: str = ""
    score: float = 0.0   # float64 greedy score along the verified decisions (N2)
    path_scores: Optional[List[float]] = None   # TDT, all_paths=True: score of every acceptable path


def _accept(logits: np.ndarray, y: int, tol: float):
    """(accepted, is_near_tie) for choosing y under float64 logits."""
    if y < 0 or y >= len(logits):
        return False, False
    if argmax_lowest(logits) == y:
        return True, False
    return (float(logits.max() - logits[y]) < tol), True


def verify_rnnt(model: Transducer, enc_row, L: int, m: int, tokens: List[int],
                timestamps: List[int], tol: float = 1e-3) -> VerifyResult:
    tokens = [int(x) for x in tokens]
    timestamps = [int(x) for x in timestamps]
    if len(tokens) != len(timestamps):
        return VerifyResult(False, message="tokens/timestamps length mismatch")
    if any(b < a for a, b in zip(timestamps, timestamps[1:])):
        return VerifyResult(False, message="timestamps decrease")
    if timestamps and (timestamps[0] < 0 or timestamps[-1] >= L):
        return VerifyResult(False, message="timestamp out of range")
    if any(y == model.blank for y in tokens):
        return VerifyResult(False, message="blank emitted as a label")
    f = model.enc_proj(enc_row[:L]) if L > 0 else None
    st = model.pred_init()
    dec, st = model.pred_step(st, model.blank)
    g = model.pred_proj(dec)
    r = VerifyResult(True)
    i = 0
    for t in range(L):
        n_here = 0
        while i < len(tokens) and timestamps[i] == t:
            if n_here == m:
                return VerifyResult(False, r.decisions, r.near_ties, f"more than m labels at t={t}")
            logits, _ = model.joint(f[t], g)
            acc, tie = _accept(logits, tokens[i], tol)
            r.decisions += 1
            r.near_ties += int(tie and acc)
            if acc:
                r.score += log_prob(logits, tokens[i])
            if not acc:
                return VerifyResult(False, r.decisions, r.near_ties,
                                    f"label {tokens[i]} at t={t} (#{i}) rejected: gap "
                                    f"{float(logits.max() - logits[tokens[i]]):.3g}")
            dec, st = model.pred_step(st, tokens[i])
            g = model.pred_proj(dec)
            i += 1
            n_here += 1
        if n_here < m:
            logits, _ = model.joint(f[t], g)
            acc, tie = _accept(logits, model.blank, tol)
            r.decisions += 1
            r.near_ties += int(tie and acc)
            if acc:
                r.score += log_prob(logits, model.blank)
            if not acc:
                return VerifyResult(False, r.decisions, r.near_ties,
                                    f"blank at t={t} rejected: gap "
                                    f"{float(logits.max() - logits[model.blank]):.3g}")
    if i != len(tokens):
        return VerifyResult(False, r.decisions, r.near_ties, "labels left after the last frame")
    return r


def verify_tdt(model: Transducer, enc_row, L: int, m: int, tokens: List[int],
               timestamps: List[int], durations: List[int], tol: float = 1e-3,
               max_nodes: int = 100000, all_paths: bool = False) -> VerifyResult:
    """all_paths: keep searching after the first acceptable decision path and
    return the scores of all of them (`path_scores`): near-tie blank durations
    are not visible in the outputs, so the path a decoder took (and hence its
    greedy score, N2) is one of these."""
    import sys
    sys.setrecursionlimit(max(sys.getrecursionlimit(), 4 * (L + len(tokens)) + 1000))
    tokens = [int(x) for x in tokens]
    timestamps = [int(x) for x in timestamps]
    durations = [int(x) for x in durations]
    if not (len(tokens) == len(timestamps) == len(durations)):
        return VerifyResult(False, message="output length mismatch")
    if any(y == model.blank for y in tokens):
        return VerifyResult(False, message="blank emitted as a label")
    D = model.durations
    f = model.enc_proj(enc_row[:L]) if L > 0 else None
    st0 = model.pred_init()
    dec, st0 = model.pred_step(st0, model.blank)
    g0 = model.pred_proj(dec)
    nodes = [0]
    best = {"msg": "no acceptable path"}

    def rec(i, t, k, st, g, dec_count, ties, score):
        nodes[0] += 1
        if nodes[0] > max_nodes:
            return None
        if t >= L:
            if i == len(tokens):
                if all_paths:
                    found.append((dec_count, ties, score))
                    return None
                return (dec_count, ties, score)
            best["msg"] = f"utterance ended with {len(tokens) - i} labels left"
            return None
        logits, dl = model.joint(f[t], g)
        if i < len(tokens) and timestamps[i] == t:
            y, d = tokens[i], durations[i]
            if d not in D:
                best["msg"] = f"duration {d} not in the duration set"
                return None
            acc_y, tie_y = _accept(logits, y, tol)
            acc_d, tie_d = _accept(dl, D.index(d), tol)
            if not (acc_y and acc_d):
                best["msg"] = (f"label {y}/d={d} at t={t} (#{i}) rejected: gaps "
                               f"{float(logits.max() - logits[y]):.3g}, "
                               f"{float(dl.max() - dl[D.index(d)]):.3g}")
                return None
            dec2, st2 = model.pred_step(st, y)
            g2 = model.pred_proj(dec2)
            if d > 0:
                nt, nk = t + d, 0
            else:
                nt, nk = (t + 1, 0) if k + 1 == m else (t, k + 1)
            return rec(i + 1, nt, nk, st2, g2, dec_count + 1, ties + int(tie_y) + int(tie_d),
                       score + log_prob(logits, y) + log_prob(dl, D.index(d)))
        if i < len(tokens) and timestamps[i] < t:
            best["msg"] = f"label #{i} stamped {timestamps[i]} was skipped over (t={t})"
            return None
        acc_b, tie_b = _accept(logits, model.blank, tol)
        if not acc_b:
            best["msg"] = (f"blank at t={t} rejected: gap "
                           f"{float(logits.max() - logits[model.blank]):.3g}")
            return None
        order = [argmax_lowest(dl)] + [j for j in range(len(D)) if j != argmax_lowest(dl)]
        for j in order:
            acc_d, tie_d = _accept(dl, j, tol)
            if not acc_d:
                continue
            out = rec(i, t + max(D[j], 1), 0, st, g, dec_count + 1, ties + int(tie_b) + int(tie_d),
                      score + log_prob(logits, model.blank) + log_prob(dl, j))
            if out is not None:
                return out
        return None

    found = []
    out = rec(0, 0, 0, st0, g0, 0, 0, 0.0)
    if all_paths and found:
        out = found[0]
        return VerifyResult(True, out[0], out[1], score=out[2], path_scores=[f[2] for f in found])
    if out is None:
        return VerifyResult(False, message=best["msg"] if nodes[0] <= max_nodes else "search budget exceeded")
    return VerifyResult(True, out[0], out[1], score=out[2])
