"""Brute-force enumeration of greedy-consistent alignments (TEST INFRASTRUCTURE).

Pin for the decoders' control logic (time rules, guard, TDT durations) on tiny
inputs, independent of the loops in decode.py: enumerate EVERY well-formed
alignment of an utterance of L frames, then keep those in which every choice
is the lowest-index float64 argmax of the joint at that point.
Greedy decoding (Alg. 1) must return the unique survivor.

Well-formed alignments (SURVEY.md §8(c) "Brute force"):
  RNN-T: per frame, j labels (0 <= j <= m) followed by a blank iff j < m
         (guard A6: after m labels go to t+1 without evaluating).
  TDT:   a chain of events (y, d) from t=0: blank -> t += max(d,1);
         label with d=0 -> k += 1 (k == m -> t += 1); label with d>0 -> t += d;
         ending when t >= L (A13/A14).
"""
from __future__ import annotations

import itertools
from typing import List, Tuple

import numpy as np

from .model import Transducer, argmax_lowest


def rnnt_alignments(L: int, tokens: List[int], m: int):
    """All per-frame label lists (a tuple of L tuples)."""
    per_frame = []
    for j in range(m + 1):
        per_frame.extend(itertools.product(tokens, repeat=j))
    return itertools.product(per_frame, repeat=L)


def tdt_alignments(L: int, symbols: List[int], blank: int, durations: List[int], m: int):
    """All event chains [(t, y, d), ...] starting at t=0 (generator)."""
    def rec(t, k, prefix):
        if t >= L:
            yield list(prefix)
            return
        for y in symbols:
            for d in durations:
                if y == blank:
                    nt, nk = t + max(d, 1), 0
                elif d > 0:
                    nt, nk = t + d, 0
                else:
                    nt, nk = (t + 1, 0) if k + 1 == m else (t, k + 1)
                prefix.append((t, y, d))
                yield from rec(nt, nk, prefix)
                prefix.pop()
    yield from rec(0, 0, [])


class _Memo:
    """Caches predictor outputs by label prefix so enumeration stays cheap."""

    def __init__(self, model: Transducer, f):
        self.model, self.f = model, f
        self.pred = {}
        self.logit = {}

    def g(self, prefix: Tuple[int, ...]):
        if prefix not in self.pred:
            if not prefix:
                dec, st = self.model.pred_step(self.model.pred_init(), self.model.blank)
            else:
                _, st_prev = self._state(prefix[:-1])
                dec, st = self.model.pred_step(st_prev, prefix[-1])
            self.pred[prefix] = (self.model.pred_proj(dec), st)
        return self.pred[prefix][0]

    def _state(self, prefix):
        self.g(prefix)
        return self.pred[prefix]

    def decide(self, prefix, t):
        key = (prefix, t)
        if key not in self.logit:
            logits, dl = self.model.joint(self.f[t], self.g(prefix))
            y = argmax_lowest(logits)
            di = None if dl is None else argmax_lowest(dl)
            self.logit[key] = (y, di)
        return self.logit[key]


def brute_force_rnnt(model: Transducer, enc_row, L: int, m: int):
    """Returns (survivors, n_alignments); survivors are (tokens, timestamps)."""
    f = model.enc_proj(enc_row[:L])
    memo = _Memo(model, f)
    toks = [v for v in range(model.num_tokens) if v != model.blank]
    survivors, n = [], 0
    for align in rnnt_alignments(L, toks, m):
        n += 1
        prefix: Tuple[int, ...] = ()
        ok = True
        for t, labels in enumerate(align):
            for y in labels:
                if memo.decide(prefix, t)[0] != y:
                    ok = False
                    break
                prefix = prefix + (y,)
            if not ok:
                break
            if len(labels) < m and memo.decide(prefix, t)[0] != model.blank:
                ok = False
                break
        if ok:
            survivors.append((list(prefix), [t for t, ls in enumerate(align) for _ in ls]))
    return survivors, n


def brute_force_tdt(model: Transducer, enc_row, L: int, m: int):
    """Returns (survivors, n_alignments); survivors are (tokens, timestamps, durations)."""
    f = model.enc_proj(enc_row[:L])
    memo = _Memo(model, f)
    D = model.durations
    survivors, n = [], 0
    for chain in tdt_alignments(L, list(range(model.num_tokens)), model.blank, D, m):
        n += 1
        prefix: Tuple[int, ...] = ()
        ok = True
        for t, y, d in chain:
            yy, di = memo.decide(prefix, t)
            if yy != y or D[di] != d:
                ok = False
                break
            if y != model.blank:
                prefix = prefix + (y,)
        if ok:
            ev = [(t, y, d) for t, y, d in chain if y != model.blank]
            survivors.append(([e[1] for e in ev], [e[0] for e in ev], [e[2] for e in ev]))
    return survivors, n
