"""Greedy Transducer decoders in float64 (TEST INFRASTRUCTURE, see oracle/__init__.py).

decode_sequential     Alg. 1 per utterance = THE oracle definition.
                      Rules: t advances only after blank; only
                      non-blank labels are appended and update the predictor.
                      + max-symbols guard (A6): after the m-th label at one
                      frame, go to t+1 without a blank evaluation.
                      TDT (A13/A14): blank -> t += max(d,1);
                      label -> append, then d == 0 ? (k += 1; k == m -> t += 1)
                      : t += d.
decode_frame_looping  Alg. 2, batched over utterances, with
                      per-utterance lengths (:119), the guard, and Alg. 1's
                      predictor semantics (A20).  RNN-T only (the paper's TDT
                      frame-looping baseline is approximate, :299; out of scope).
decode_label_looping  Alg. 3 corrected per readings A1-A5,
                      A21: outer loop over labels, inner loop over
                      frames; RNN-T and TDT.  This is the CPU form of the method
                      the CUDA path implements.

Every decoder returns per-utterance (tokens, timestamps[, durations]) and
counters.  Timestamps (A15): RNN-T = frame of emission, TDT = frame where the
joint was evaluated; durations = raw predicted d.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np

from .model import Transducer, argmax_lowest, log_prob


@dataclasses.dataclass
class DecodeResult:
    tokens: List[int]
    timestamps: List[int]
    durations: Optional[List[int]] = None
    joint_evals: int = 0          # joint evaluations of this utterance
    predictor_calls: int = 0      # predictor calls of this utterance (incl. SOS)
    trace: Optional[list] = None  # every decision (t, y[, d]) in order
    score: float = 0.0            # greedy score: sum of log-probabilities of every decision (N2, A19)


def _decide(model: Transducer, f_t, g):
    y, d, _ = _decide_scored(model, f_t, g)
    return y, d


def _decide_scored(model: Transducer, f_t, g):
    """(y, d, log-probability of the decision): token log-softmax at y, plus,
    for TDT, the duration log-softmax at the chosen duration (the joint
    probability of the (token, duration) pair; reading A19)."""
    logits, dl = model.joint(f_t, g)
    y = argmax_lowest(logits)
    lp = log_prob(logits, y)
    d = None
    if dl is not None:
        j = argmax_lowest(dl)
        d = model.durations[j]
        lp += log_prob(dl, j)
    return y, d, lp


def decode_sequential(model: Transducer, enc_row: np.ndarray, L: int, max_symbols: int,
                      f: Optional[np.ndarray] = None, keep_trace: bool = False) -> DecodeResult:
    """Alg. 1 "Inference of Transducer" for one utterance.

    `enc_row` is [T, D_e] (frames >= L are never read); `f` may pass the
    already-projected rows.  Returns tokens/timestamps(/durations)."""
    if f is None:
        f = model.enc_proj(enc_row[:L]) if L > 0 else np.zeros((0, model.H))
    tdt = model.durations is not None
    m = max_symbols
    res = DecodeResult([], [], [] if tdt else None, trace=[] if keep_trace else None)
    state = model.pred_init()                               # Alg. 1 line 3
    dec, state = model.pred_step(state, model.blank)         # line 65: predictor(state, BOS)
    g = model.pred_proj(dec)                                 # §3.4 projection
    res.predictor_calls = 1
    t, k = 0, 0
    while t < L:                                             # line 63
        y, d, lp = _decide_scored(model, f[t], g)            # lines 69-70
        res.joint_evals += 1
        res.score += lp                                      # every argmax step, blanks included
        if keep_trace:
            res.trace.append((t, y) if not tdt else (t, y, d))
        if y == model.blank:                                 # line 75-76: t = t + 1
            t += max(d, 1) if tdt else 1                     # TDT: A13 anti-stall
            k = 0
            continue
        res.tokens.append(y)                                 # line 72
        res.timestamps.append(t)
        if tdt:
            res.durations.append(d)
        dec, state = model.pred_step(state, y)               # line 74 (state = new_state)
        g = model.pred_proj(dec)
        res.predictor_calls += 1
        if tdt and d > 0:                                    # A13: label with d > 0
            t += d
            k = 0
        else:                                                # A6/A14 guard on zero-duration labels
            k += 1
            if k == m:
                t += 1
                k = 0
    return res


def decode_frame_looping(model: Transducer, enc: np.ndarray, lengths, max_symbols: int):
    """Alg. 2 "Batched Inference of Transducer", RNN-T.

    Per utterance state follows Alg. 1: `states` holds the predictor state
    before the last label and `last` that label (A20), so line 6/17
    `predictor(states, predictions)` recomputes dec for every evaluation and
    lines 10/21 keep new_states only for rows that emitted a non-blank.
    Finished utterances (t >= L_b) are permanently blank-masked.
    Returns (results, counters) where counters count BATCHED predictor and
    joint invocations (Fig. 2)."""
    assert model.durations is None
    B = enc.shape[0]
    lengths = [int(x) for x in lengths]
    T = max(lengths) if B else 0
    f = [model.enc_proj(enc[b, :lengths[b]]) for b in range(B)]
    res = [DecodeResult([], []) for _ in range(B)]
    states = [model.pred_init() for _ in range(B)]           # line 3
    last = [model.blank] * B                                 # line 4: predictions = [BOS * B]
    cnt = {"predictor_calls": 0, "joint_calls": 0}

    def predictor_all():
        cnt["predictor_calls"] += 1
        return [model.pred_step(states[b], last[b]) for b in range(B)]

    def joint_argmax(t, decs, mask):
        cnt["joint_calls"] += 1
        out = []
        for b in range(B):
            if mask[b]:
                out.append(model.blank)
                continue
            g = model.pred_proj(decs[b][0])
            y, _ = _decide(model, f[b][t], g)
            res[b].joint_evals += 1
            out.append(y)
        return out

    t = 0
    while t < T:                                             # line 5
        done = [t >= lengths[b] for b in range(B)]
        new = predictor_all()                                # line 6
        preds = joint_argmax(t, new, done)                   # lines 7-8
        blank_mask = [done[b] or preds[b] == model.blank for b in range(B)]   # line 9
        k = [0] * B
        while not all(blank_mask):                           # line 11
            for b in range(B):                               # lines 12-16 (and line 10)
                if not blank_mask[b]:
                    res[b].tokens.append(preds[b])
                    res[b].timestamps.append(t)
                    states[b] = new[b][1]
                    last[b] = preds[b]
                    k[b] += 1
                    if k[b] == max_symbols:                  # guard (A6): no blank eval
                        blank_mask[b] = True
            if all(blank_mask):
                break
            new = predictor_all()                            # line 17
            preds = joint_argmax(t, new, blank_mask)         # lines 18-19
            blank_mask = [blank_mask[b] or preds[b] == model.blank for b in range(B)]  # line 20
        t += 1                                               # line 22
    return res, cnt


def decode_label_looping(model: Transducer, enc: np.ndarray, lengths, max_symbols: int):
    """Alg. 3 "Label-looping Algorithm", RNN-T and TDT.

    Corrected per DESIGN.md readings: predictions start at SOS (A1); active
    is t < L (A2); the inner-loop mask uses the NEW predictions (A3); only
    rows that FOUND a non-blank at a valid frame are appended (A4); the
    predictor runs only for rows that found a label and stay active (A5, A21);
    guard per A6/A14; TDT time update per A13 (lines 10 and 18
    add the predicted duration).
    Returns (results, counters): outer steps, predictor (batched) calls, joint
    rounds (batched invocations) and joint row evaluations."""
    tdt = model.durations is not None
    B = enc.shape[0]
    m = max_symbols
    lengths = [int(x) for x in lengths]
    f = [model.enc_proj(enc[b, :lengths[b]]) if lengths[b] > 0 else None for b in range(B)]
    res = [DecodeResult([], [], [] if tdt else None) for _ in range(B)]
    cnt = {"outer_steps": 0, "predictor_calls": 0, "joint_rounds": 0, "joint_row_evals": 0}
    t = [0] * B                                              # line 4: b2time
    k = [0] * B                                              # labels emitted at the current frame
    active = [lengths[b] > 0 for b in range(B)]              # line 4: b2active (A2: t < L)
    state = [model.pred_init() for _ in range(B)]            # line 3
    g: List[Optional[np.ndarray]] = [None] * B
    need_pred = list(active)
    labels = [model.blank] * B                               # A1: predictions = SOS
    while any(active):                                       # line 5
        cnt["outer_steps"] += 1
        if any(need_pred):                                   # line 6 (only rows that need it, A5)
            cnt["predictor_calls"] += 1
            for b in range(B):
                if need_pred[b]:
                    dec, state[b] = model.pred_step(state[b], labels[b])
                    g[b] = model.pred_proj(dec)
                    res[b].predictor_calls += 1
        found = [False] * B
        found_t = [0] * B
        found_d = [0] * B
        scanning = list(active)
        while any(scanning):                                 # lines 7-8 then 12-19
            cnt["joint_rounds"] += 1
            for b in range(B):
                if not scanning[b]:
                    continue
                cnt["joint_row_evals"] += 1
                res[b].joint_evals += 1
                y, d = _decide(model, f[b][t[b]], g[b])
                if y == model.blank:                         # lines 9-11 / 15-19
                    t[b] += max(d, 1) if tdt else 1
                    k[b] = 0
                    if t[b] >= lengths[b]:
                        active[b] = False
                        scanning[b] = False
                else:                                        # row found its next label
                    found[b], labels[b] = True, y
                    found_t[b], found_d[b] = t[b], (d if tdt else 0)
                    scanning[b] = False
        for b in range(B):                                   # line 21 (masked append, A4)
            need_pred[b] = False
            if not found[b]:
                continue
            res[b].tokens.append(labels[b])
            res[b].timestamps.append(found_t[b])
            if tdt:
                res[b].durations.append(found_d[b])
            if tdt and found_d[b] > 0:
                t[b] += found_d[b]
                k[b] = 0
            else:
                k[b] += 1
                if k[b] == m:
                    t[b] += 1
                    k[b] = 0
            active[b] = t[b] < lengths[b]
            need_pred[b] = active[b]
    return res, cnt
