"""Helpers shared by the GPU parity tests: run the CUDA path through the C ABI
(paper_2406_06220_b200.decoder -> ll.py -> libll.so) and check it against the
float64 oracle with the teacher-forced verifier."""
import numpy as np
import torch

import synth
from oracle import Transducer, decode_sequential
from oracle.verify import verify_rnnt, verify_tdt
from paper_2406_06220_b200 import build as llbuild
from paper_2406_06220_b200.decoder import LabelLoopingDecoder, Model, debug_joint

TOL = 1e-3  # north_star: decisions with a float64 top-2 gap below 1e-3 are near-ties


def gpu_model(spec, weights, dtype="bf16"):
    llbuild.build()
    return Model(weights, pred_kind=spec.pred_kind, context=spec.context, blank_id=spec.blank_id,
                 durations=spec.durations, dtype=dtype)


def gpu_decode(spec, weights, enc, lengths, dtype="bf16", cap=None, model=None, B_max=None, T_max=None):
    model = model or gpu_model(spec, weights, dtype)
    B, T = enc.shape[0], enc.shape[1]
    dec = LabelLoopingDecoder(model, spec.max_symbols, B_max or max(B, 1), T_max or max(T, 1), cap=cap)
    enc_d = torch.from_numpy(np.ascontiguousarray(enc)).to("cuda", model.tdtype)
    len_d = torch.from_numpy(np.asarray(lengths, dtype=np.int32)).cuda()
    out = dec.decode(enc_d, len_d)
    return out.hypotheses(), dec


def verify_all(spec, weights, enc, lengths, hyps, tol=TOL, rows=None):
    """Teacher-forced float64 verification of every (or the listed) row.
    Returns (near_ties, decisions)."""
    model = Transducer.from_spec(spec, weights)
    ties = dec = 0
    for b in (range(len(hyps)) if rows is None else rows):
        L = int(lengths[b])
        h = hyps[b]
        if spec.is_tdt:
            r = verify_tdt(model, enc[b], L, spec.max_symbols, h[0], h[1], h[2], tol=tol)
        else:
            r = verify_rnnt(model, enc[b], L, spec.max_symbols, h[0], h[1], tol=tol)
        assert r.ok, f"row {b}: {r.message}"
        ties += r.near_ties
        dec += r.decisions
    return ties, dec


def oracle_hyps(spec, weights, enc, lengths, rows=None):
    model = Transducer.from_spec(spec, weights)
    out = {}
    for b in (range(enc.shape[0]) if rows is None else rows):
        r = decode_sequential(model, enc[b], int(lengths[b]), spec.max_symbols)
        out[b] = (r.tokens, r.timestamps) + ((r.durations,) if spec.is_tdt else ())
    return out
