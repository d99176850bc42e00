"""Seeded synthetic workloads for label-looping Transducer decoding.

This module is the ONLY code shared by the CUDA path's callers (tests, bench)
and the float64 oracle (`oracle/`).  It holds no arithmetic of the method
(no projection, predictor, joint, argmax or time rule): it only draws seeded
random numbers, rounds them once to bf16, and lays them out in the tensor
shapes of the C ABI (`include/ll.h`).  The planted-alignment family builds
weights whose greedy decode is known in closed form; the
planted alignment it returns is a construction, not a decode.

Readings:
  * weights ~ U[-1/2, 1/2]/sqrt(fan_in), embeddings ~ N(0, 0.5^2),
    rounded once to bf16; those bf16 values are the truth for BOTH paths
    (SURVEY.md §8(c) A24).  f32 runs reuse the same values.
  * encoder outputs ~ N(0, 1), bf16-rounded.
  * blank id is 0 unless stated; SOS = blank.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence

import numpy as np

__all__ = [
    "ModelSpec", "bf16_round", "make_weights", "make_inputs", "make_planted_rnnt",
    "make_planted_tdt", "cat_dog_fixture", "tdt_forced_fixture", "guard_after_blank_fixture",
    "guard_after_blank_tdt_fixture", "CONFIGS",
    "sweep_lengths", "frame_seconds", "planted_weights", "planted_utterance", "SWEEPS",
]

frame_seconds = 0.08  # 8x subsampling of 10 ms frames


def bf16_round(x) -> np.ndarray:
    """Round float64 values to the nearest bf16 (round-to-nearest-even),
    returned as float32 (every bf16 value is exactly representable in f32)."""
    x32 = np.ascontiguousarray(np.asarray(x, dtype=np.float64).astype(np.float32))
    u = x32.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(x32.shape)


@dataclasses.dataclass(frozen=True)
class ModelSpec:
    """Shapes of one Transducer decoding problem (ABI names in brackets)."""
    num_tokens: int            # V+1, blank included            [num_tokens]
    enc_dim: int               # D_e                             [enc_dim]
    pred_dim: int              # P                               [hidden]
    joint_dim: int             # H                               [joint_dim]
    pred_kind: str = "lstm"    # "lstm" | "stateless"
    context: int = 1           # stateless context size c
    durations: Optional[Sequence[int]] = None  # TDT duration set D (None: RNN-T)
    blank_id: int = 0
    max_symbols: int = 10
    num_layers: int = 1        # LSTM layers ("more layers"; layers >= 2: *_rest arrays)

    @property
    def is_tdt(self) -> bool:
        return self.durations is not None


def _uniform(rng, shape, fan_in):
    return rng.uniform(-0.5, 0.5, size=shape) / math.sqrt(fan_in)


def make_weights(spec: ModelSpec, seed: int = 0, blank_bias: float = 0.0) -> Dict[str, np.ndarray]:
    """Random-init weights in ABI layout, bf16-rounded, as float32 arrays.

    LSTM: embedding [V+1,P], w_ih/w_hh [4P,P] (gate rows i,f,g,o), b_ih/b_hh [4P];
    layers 2..L (spec.num_layers > 1): w_ih_rest/w_hh_rest [L-1,4P,P], b_ih_rest/b_hh_rest [L-1,4P].
    Stateless: embedding [c, V+1, P/c].  Joint: w_enc [H,D_e], b_enc [H],
    w_pred [H,P], b_pred [H], w_out [V+1,H], b_out [V+1]; TDT w_dur [|D|,H], b_dur [|D|].
    `blank_bias` is added to b_out[blank] before rounding.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    V1, De, P, H = spec.num_tokens, spec.enc_dim, spec.pred_dim, spec.joint_dim
    w: Dict[str, np.ndarray] = {}
    if spec.pred_kind == "lstm":
        w["embedding"] = rng.normal(0.0, 0.5, size=(V1, P))
        w["w_ih"] = _uniform(rng, (4 * P, P), P)
        w["w_hh"] = _uniform(rng, (4 * P, P), P)
        w["b_ih"] = _uniform(rng, (4 * P,), P)
        w["b_hh"] = _uniform(rng, (4 * P,), P)
    elif spec.pred_kind == "stateless":
        assert P % spec.context == 0
        w["embedding"] = rng.normal(0.0, 0.5, size=(spec.context, V1, P // spec.context))
    else:
        raise ValueError(spec.pred_kind)
    w["w_enc"] = _uniform(rng, (H, De), De)
    w["b_enc"] = _uniform(rng, (H,), De)
    w["w_pred"] = _uniform(rng, (H, P), P)
    w["b_pred"] = _uniform(rng, (H,), P)
    w["w_out"] = _uniform(rng, (V1, H), H)
    b_out = _uniform(rng, (V1,), H)
    b_out[spec.blank_id] += blank_bias
    w["b_out"] = b_out
    if spec.is_tdt:
        nd = len(spec.durations)
        w["w_dur"] = _uniform(rng, (nd, H), H)
        w["b_dur"] = _uniform(rng, (nd,), H)
    if spec.pred_kind == "lstm" and spec.num_layers > 1:   # drawn last: 1-layer weights unchanged per seed
        Lr = spec.num_layers - 1
        w["w_ih_rest"] = _uniform(rng, (Lr, 4 * P, P), P)
        w["w_hh_rest"] = _uniform(rng, (Lr, 4 * P, P), P)
        w["b_ih_rest"] = _uniform(rng, (Lr, 4 * P), P)
        w["b_hh_rest"] = _uniform(rng, (Lr, 4 * P), P)
    return {k: bf16_round(v) for k, v in w.items()}


def make_inputs(seed: int, B: int, T_max: int, enc_dim: int, len_lo: int, len_hi: int,
                pad_value: Optional[float] = None):
    """Encoder outputs [B,T_max,D_e] ~ N(0,1) (bf16-rounded, f32 array) and
    lengths int32[B] ~ U{len_lo..len_hi} (clipped to T_max).  Frames at
    t >= len are filled with `pad_value` if given (e.g. NaN to prove that
    padding is never read)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    enc = bf16_round(rng.normal(0.0, 1.0, size=(B, T_max, enc_dim)))
    lengths = rng.integers(len_lo, len_hi + 1, size=B).clip(0, T_max).astype(np.int32)
    if pad_value is not None:
        for b in range(B):
            enc[b, lengths[b]:, :] = pad_value
    return enc, lengths


def sweep_lengths(seed: int, n: int, median_s: float = 5.5, sigma_ln: float = 0.65,
                  lo_s: float = 1.0, hi_s: float = 35.0) -> np.ndarray:
    """LibriSpeech-like utterance lengths in frames (assumed profile,
    SURVEY.md §8(d) config 5): log-normal seconds, clipped, frames = ceil(s/0.08)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    s = np.exp(rng.normal(math.log(median_s), sigma_ln, size=n)).clip(lo_s, hi_s)
    return np.ceil(s / frame_seconds).astype(np.int32)


# ---------------------------------------------------------------------------
# Planted-alignment family.  Random init everywhere except a
# few joint dims that implement a planted alignment:
#   dim 0        blank channel: f[0] = +1 on blank frames, -1 on token frames;
#                W_out[blank,0] = 4, W_out[v!=blank,0] = 0, g[0] = 0.
#   dims 1..64   code channel: token frames carry code(y_t) (16-of-64 binary);
#                g[1..64] = -code(last label); W_out[v,1..64] = 0.5(2code(v)-1).
#   (TDT) 5 dims duration channel: one-hot of the planted duration index,
#                read by W_dur with gain 4.
# Blank bias 2.0: the planted token wins once at its frame, then blank wins.
# ---------------------------------------------------------------------------
_CODE_DIMS = 64
_CODE_BITS = 16


def _codes(rng, V1, blank_id):
    codes = np.zeros((V1, _CODE_DIMS))
    for v in range(V1):
        if v == blank_id:
            continue
        codes[v, rng.choice(_CODE_DIMS, size=_CODE_BITS, replace=False)] = 1.0
    return codes


def _planted_base(spec: ModelSpec, seed: int, n_extra: int):
    V1, De, P, H = spec.num_tokens, spec.enc_dim, spec.pred_dim, spec.joint_dim
    nd = 1 + _CODE_DIMS + n_extra
    assert De >= nd and H >= nd, "planted family needs D_e, H >= 1+64+extra"
    rng = np.random.Generator(np.random.PCG64(seed))
    w = {k: v.astype(np.float64) for k, v in make_weights(spec, seed).items()}
    codes = _codes(rng, V1, spec.blank_id)
    # encoder projection: planted rows copy planted input dims exactly
    w["w_enc"][:nd, :] = 0.0
    w["b_enc"][:nd] = 0.0
    for j in range(nd):
        w["w_enc"][j, j] = 1.0
    # predictor projection: g[0] = 0, g[1..64] = -code(last), g[extra] = 0
    w["w_pred"][:nd, :] = 0.0
    w["b_pred"][:nd] = 0.0
    if spec.pred_kind == "stateless":
        assert P // spec.context >= _CODE_DIMS
        w["embedding"][0, :, :_CODE_DIMS] = codes       # slot 0 = most recent label
        for j in range(_CODE_DIMS):
            w["w_pred"][1 + j, j] = -1.0
    else:
        assert P >= _CODE_DIMS
        # units 0..63 copy the input code: i,o saturated open, f closed,
        # cell input g = 30(2 code - 1)  =>  h_j = +-tanh(1)
        w["embedding"][:, :_CODE_DIMS] = codes
        for gate in range(4):
            rows = slice(gate * P, gate * P + _CODE_DIMS)
            w["w_ih"][rows, :] = 0.0
            w["w_hh"][rows, :] = 0.0
            w["b_hh"][rows] = 0.0
        for j in range(_CODE_DIMS):
            w["b_ih"][0 * P + j] = 30.0          # input gate open
            w["b_ih"][1 * P + j] = -30.0         # forget gate closed
            w["w_ih"][2 * P + j, j] = 60.0       # cell input +-30
            w["b_ih"][2 * P + j] = -30.0
            w["b_ih"][3 * P + j] = 30.0          # output gate open
            w["w_pred"][1 + j, j] = -1.0 / (2.0 * math.tanh(1.0))
            w["b_pred"][1 + j] = -0.5
    # output layer
    w["w_out"][:, :nd] = 0.0
    w["w_out"][spec.blank_id, 0] = 4.0
    for v in range(V1):
        if v != spec.blank_id:
            w["w_out"][v, 1:1 + _CODE_DIMS] = 0.5 * (2.0 * codes[v] - 1.0)
        else:
            w["w_out"][v, 1:1 + _CODE_DIMS] = -0.5
    w["b_out"][:] = 0.0
    w["b_out"][spec.blank_id] = 2.0
    return rng, w, codes, nd


def _planted_tokens(rng, n, V1, blank_id, codes, prev=None, max_overlap=4):
    """Draw n non-blank tokens; each differs from the previous planted token and
    shares at most `max_overlap` code bits with it, so that z = ReLU(code(y) -
    code(last)) keeps >= 12 active code dims and y wins by a wide margin."""
    out = []
    for _ in range(n):
        while True:
            y = int(rng.integers(0, V1))
            if y == blank_id or y == prev:
                continue
            if prev is not None and float(codes[y] @ codes[prev]) > max_overlap:
                continue
            break
        out.append(y)
        prev = y
    return out


def make_planted_rnnt(spec: ModelSpec, seed: int, B: int, T_max: int, len_lo: int, len_hi: int,
                      rho: float = 0.28):
    """Planted RNN-T workload: each frame is a token frame with prob `rho`
    (one token, then blank) else a blank frame.  Returns (weights, enc,
    lengths, planted) with planted[b] = (tokens, timestamps)."""
    assert not spec.is_tdt
    rng, w, codes, nd = _planted_base(spec, seed, 0)
    enc = rng.normal(0.0, 1.0, size=(B, T_max, spec.enc_dim))
    enc[:, :, :nd] = 0.0
    enc[:, :, 0] = 1.0
    lengths = rng.integers(len_lo, len_hi + 1, size=B).clip(0, T_max).astype(np.int32)
    planted = []
    for b in range(B):
        L = int(lengths[b])
        frames = [t for t in range(L) if rng.random() < rho]
        toks = _planted_tokens(rng, len(frames), spec.num_tokens, spec.blank_id, codes)
        for t, y in zip(frames, toks):
            enc[b, t, 0] = -1.0
            enc[b, t, 1:1 + _CODE_DIMS] = codes[y]
        planted.append((toks, frames))
    return ({k: bf16_round(v) for k, v in w.items()}, bf16_round(enc), lengths, planted)


def make_planted_tdt(spec: ModelSpec, seed: int, B: int, T_max: int, len_lo: int, len_hi: int,
                     p_token: float = 0.55,
                     token_dur_p=(0.45, 0.30, 0.15, 0.10), blank_dur_p=(0.2, 0.3, 0.3, 0.2)):
    """Planted TDT workload: a chain of events from t=0, each (token or blank,
    duration in {1..4}) landing at t+d.  `spec.durations` must contain 1..4.
    Returns (weights, enc, lengths, planted) with planted[b] =
    (tokens, timestamps, durations)."""
    assert spec.is_tdt
    D = list(spec.durations)
    nD = len(D)
    rng, w, codes, nd = _planted_base(spec, seed, nD)
    dur0 = 1 + _CODE_DIMS
    w["w_dur"][:, :nd] = 0.0
    w["b_dur"][:] = 0.0
    for i in range(nD):
        w["w_dur"][i, dur0 + i] = 4.0
    w["w_out"][:, dur0:dur0 + nD] = 0.0
    enc = rng.normal(0.0, 1.0, size=(B, T_max, spec.enc_dim))
    enc[:, :, :nd] = 0.0
    lengths = rng.integers(len_lo, len_hi + 1, size=B).clip(0, T_max).astype(np.int32)
    planted = []
    for b in range(B):
        L = int(lengths[b])
        t, prev = 0, None
        toks, stamps, durs = [], [], []
        while t < L:
            is_tok = rng.random() < p_token
            d = int(rng.choice([1, 2, 3, 4], p=token_dur_p if is_tok else blank_dur_p))
            di = D.index(d)
            enc[b, t, dur0 + di] = 1.0
            if is_tok:
                y = _planted_tokens(rng, 1, spec.num_tokens, spec.blank_id, codes, prev)[0]
                prev = y
                enc[b, t, 0] = -1.0
                enc[b, t, 1:1 + _CODE_DIMS] = codes[y]
                toks.append(y); stamps.append(t); durs.append(d)
            else:
                enc[b, t, 0] = 1.0
            t += d
        planted.append((toks, stamps, durs))
    return ({k: bf16_round(v) for k, v in w.items()}, bf16_round(enc), lengths, planted)


def planted_weights(spec: ModelSpec, seed: int):
    """The planted-family weights alone (RNN-T or TDT), identical to the ones
    make_planted_rnnt / make_planted_tdt return for the same seed."""
    nD = len(spec.durations) if spec.is_tdt else 0
    rng, w, codes, nd = _planted_base(spec, seed, nD)
    if spec.is_tdt:
        dur0 = 1 + _CODE_DIMS
        w["w_dur"][:, :nd] = 0.0
        w["b_dur"][:] = 0.0
        for i in range(nD):
            w["w_dur"][i, dur0 + i] = 4.0
        w["w_out"][:, dur0:dur0 + nD] = 0.0
    return {k: bf16_round(v) for k, v in w.items()}, codes


def planted_utterance(spec: ModelSpec, codes, seed: int, uid: int, L: int, rho: float = 0.28,
                      p_token: float = 0.55, token_dur_p=(0.45, 0.30, 0.15, 0.10),
                      blank_dur_p=(0.2, 0.3, 0.3, 0.2)):
    """One planted utterance of the sweep workload (BASELINE config 5), drawn
    from its own seeded stream (seed, uid) so that any subset of a large sweep
    can be regenerated independently.  Same planted recipe as
    make_planted_rnnt / make_planted_tdt.  Returns (enc [L, D_e] bf16-rounded
    float32, planted alignment)."""
    rng = np.random.Generator(np.random.PCG64([seed, uid]))
    nD = len(spec.durations) if spec.is_tdt else 0
    nd = 1 + _CODE_DIMS + nD
    enc = rng.normal(0.0, 1.0, size=(L, spec.enc_dim)).astype(np.float32)
    enc[:, :nd] = 0.0
    if not spec.is_tdt:
        enc[:, 0] = 1.0
        frames = [t for t in range(L) if rng.random() < rho]
        toks = _planted_tokens(rng, len(frames), spec.num_tokens, spec.blank_id, codes)
        for t, y in zip(frames, toks):
            enc[t, 0] = -1.0
            enc[t, 1:1 + _CODE_DIMS] = codes[y]
        return bf16_round(enc), (toks, frames)
    D = list(spec.durations)
    dur0 = 1 + _CODE_DIMS
    t, prev = 0, None
    toks, stamps, durs = [], [], []
    while t < L:
        is_tok = rng.random() < p_token
        d = int(rng.choice([1, 2, 3, 4], p=token_dur_p if is_tok else blank_dur_p))
        enc[t, dur0 + D.index(d)] = 1.0
        if is_tok:
            y = _planted_tokens(rng, 1, spec.num_tokens, spec.blank_id, codes, prev)[0]
            prev = y
            enc[t, 0] = -1.0
            enc[t, 1:1 + _CODE_DIMS] = codes[y]
            toks.append(y); stamps.append(t); durs.append(d)
        else:
            enc[t, 0] = 1.0
        t += d
    return bf16_round(enc), (toks, stamps, durs)


# ---------------------------------------------------------------------------
# Paper worked example, Fig. 2: B=2, T=4, transcripts
# "CAT" / "DOG", alignments  C b b A T b b  /  b D b b O G b.
# Encoded as real weights of a stateless (context 1) ReLU-joint Transducer:
#   enc one-hot over (utt, t); Emb one-hot over labels; b_pred = -1 so that
#   z = ReLU(f + g) is one-hot at joint dim (utt, t, last label);
#   W_out[next, (utt,t,last)] = 10 where `next` is the alignment's next symbol.
# All values are in {0, +-1, 10}: exact in bf16.
# ---------------------------------------------------------------------------
CAT_DOG_VOCAB = ["<b>", "C", "A", "T", "D", "O", "G"]


def _table_fixture(alignments, T, V1, durations=None, De=16, P=16):
    """Weights of a table model realising per-utterance alignments.

    alignments[u] is a list of (t, last_label, next_symbol[, dur_index]) steps.
    """
    B = len(alignments)
    n_states = B * T * V1
    H = ((n_states + 15) // 16) * 16
    assert B * T <= De and V1 <= P
    spec = ModelSpec(num_tokens=V1, enc_dim=De, pred_dim=P, joint_dim=H, pred_kind="stateless",
                     context=1, durations=durations, blank_id=0, max_symbols=10)
    w = {
        "embedding": np.zeros((1, V1, P)), "w_enc": np.zeros((H, De)), "b_enc": np.zeros(H),
        "w_pred": np.zeros((H, P)), "b_pred": -np.ones(H), "w_out": np.zeros((V1, H)),
        "b_out": np.zeros(V1),
    }
    for v in range(V1):
        w["embedding"][0, v, v] = 1.0
    enc = np.zeros((B, T, De))
    for u in range(B):
        for t in range(T):
            enc[u, t, u * T + t] = 1.0
            for l in range(V1):
                j = (u * T + t) * V1 + l
                w["w_enc"][j, u * T + t] = 1.0
                w["w_pred"][j, l] = 1.0
    if durations is not None:
        w["w_dur"] = np.zeros((len(durations), H))
        w["b_dur"] = np.zeros(len(durations))
    for u, steps in enumerate(alignments):
        for st in steps:
            t, last, nxt = st[0], st[1], st[2]
            j = (u * T + t) * V1 + last
            w["w_out"][nxt, j] = 10.0
            if durations is not None:
                w["w_dur"][st[3], j] = 10.0
    lengths = np.full(B, T, dtype=np.int32)
    return spec, {k: bf16_round(v) for k, v in w.items()}, bf16_round(enc), lengths


def cat_dog_fixture():
    """Fig. 2 as real weights.  Returns (spec, weights, enc,
    lengths, vocab).  Replaying the caption's alignments under Alg. 1 gives
    CAT @ [0,2,2] and DOG @ [1,3,3]."""
    C, A, T_, D, O, G = 1, 2, 3, 4, 5, 6
    b = 0
    # (t, last, next): last = most recent emitted label (SOS = blank)
    cat = [(0, b, C), (0, C, b), (1, C, b), (2, C, A), (2, A, T_), (2, T_, b), (3, T_, b)]
    dog = [(0, b, b), (1, b, D), (1, D, b), (2, D, b), (3, D, O), (3, O, G), (3, G, b)]
    spec, w, enc, lengths = _table_fixture([cat, dog], 4, 7)
    return spec, w, enc, lengths, CAT_DOG_VOCAB


GUARD_VOCAB = ["<b>", "A", "B", "C", "D", "E", "F"]


def guard_after_blank_fixture():
    """Max-symbols guard (reading A6) after a frame advance, m = 3, one RNN-T
    utterance and one TDT utterance-equivalent, as table weights.

    RNN-T alignment over T=4: frame 0 emits A then blank; frame 1 emits B, C,
    D (the guard fires after the 3rd label at frame 1, no blank evaluation);
    frames 2, 3 blank.  The label counter must restart at the frame advance
    (the blank at frame 0), so all three labels at frame 1 are emitted:
    A,B,C,D @ [0,1,1,1].  Returns (spec, weights, enc, lengths, vocab)."""
    A, B_, C, D, b = 1, 2, 3, 4, 0
    steps = [(0, b, A), (0, A, b), (1, A, B_), (1, B_, C), (1, C, D), (2, D, b), (3, D, b)]
    spec, w, enc, lengths = _table_fixture([steps], 4, 7)
    spec = dataclasses.replace(spec, max_symbols=3)
    return spec, w, enc, lengths, GUARD_VOCAB


def guard_after_blank_tdt_fixture():
    """TDT form of guard_after_blank_fixture (durations {0,1,2}, m = 3): frame 0
    emits (A,0) then (blank,1); frame 1 emits (B,0), (C,0), (D,0) -- the guard
    fires after the third zero-duration label at frame 1 -- then (blank,1) at
    frames 2 and 3.  Expected A,B,C,D @ [0,1,1,1], durations [0,0,0,0]."""
    A, B_, C, D, b = 1, 2, 3, 4, 0
    steps = [(0, b, A, 0), (0, A, b, 1), (1, A, B_, 0), (1, B_, C, 0), (1, C, D, 0), (2, D, b, 1),
             (3, D, b, 1)]
    spec, w, enc, lengths = _table_fixture([steps], 4, 7, durations=[0, 1, 2])
    spec = dataclasses.replace(spec, max_symbols=3)
    return spec, w, enc, lengths, GUARD_VOCAB


def tdt_forced_fixture():
    """SPEC.md:311 TDT forced alignment [(D,1),(O,2),(G,1),(b,1)] over T=5
    (one utterance, durations {0,1,2,3,4}).  Replay gives D,O,G @ [0,1,3]."""
    D, O, G, b = 4, 5, 6, 0
    steps = [(0, b, D, 1), (1, D, O, 2), (3, O, G, 1), (4, G, b, 1)]
    spec, w, enc, lengths = _table_fixture([steps], 5, 7, durations=[0, 1, 2, 3, 4])
    return spec, w, enc, lengths, CAT_DOG_VOCAB


# ---------------------------------------------------------------------------
# BASELINE.json configs.
# ---------------------------------------------------------------------------
CONFIGS = {
    # (1) tiny RNN-T: B=4, T<=50, dims 16, stateless, vocab 8+blank, m=3
    "tiny": dict(spec=ModelSpec(9, 16, 16, 16, "stateless", 1, None, 0, 3), B=4, T_max=50,
                 len_lo=0, len_hi=50),
    # (3) TDT variant of config 1, durations {0..4}
    "tiny-tdt": dict(spec=ModelSpec(9, 16, 16, 16, "stateless", 1, (0, 1, 2, 3, 4), 0, 3), B=4,
                     T_max=50, len_lo=0, len_hi=50),
    # (2) FastConformer RNN-T: B=32, T~250 (U{225..275}), enc 512, LSTM 640, joint 640, V=1024+blank
    "fc-rnnt": dict(spec=ModelSpec(1025, 512, 640, 640, "lstm", 1, None, 0, 10), B=32, T_max=275,
                    len_lo=225, len_hi=275),
    # (3) TDT at FastConformer shapes, durations {0..4}
    "fc-tdt": dict(spec=ModelSpec(1025, 512, 640, 640, "lstm", 1, (0, 1, 2, 3, 4), 0, 10), B=32,
                   T_max=275, len_lo=225, len_hi=275),
    # (2') 4x subsampling variant of config 2 (40 ms frames, Table 4
    # :322-339): the same ~20 s utterances are twice as many frames; planted
    # token rate halved per frame (same tokens per second)
    "fc-rnnt-4x": dict(spec=ModelSpec(1025, 512, 640, 640, "lstm", 1, None, 0, 10), B=32, T_max=550,
                       len_lo=450, len_hi=550, frame_s=0.04, rho=0.14),
    # (4) large-batch stateless (context 2): B=512, lengths 50..1500, enc 1024
    "stateless-b512": dict(spec=ModelSpec(1025, 1024, 640, 640, "stateless", 2, None, 0, 10), B=512,
                           T_max=1500, len_lo=50, len_hi=1500),
}

def random_family_blank_bias(spec: ModelSpec) -> float:
    """Blank bias of the RANDOM family at FastConformer scale (H = 640,
    V+1 = 1025), calibrated on the float64 oracle (calibration batch: weights
    seed 61, inputs seed 62, 3 x 60 frames; SURVEY.md §8(d) "blank bias
    calibrated closed-loop"): the token rate is steep in the bias (RNN-T LSTM
    0.25 -> 1.75, 0.30 -> 0.67, 0.35 -> 0.11 tokens/frame; bias >= 0.5 emits
    nothing), so each family gets the bias that lands at ~0.3-0.7
    tokens/frame, where labels, blanks and near-ties all occur.  Small models
    keep 0.5."""
    if spec.joint_dim <= 64:
        return 0.5
    if spec.is_tdt:
        return 0.2          # 0.59 tokens/frame
    if spec.pred_kind == "stateless":
        return 0.28         # ~0.5 tokens/frame (context 2)
    return 0.3              # 0.67 tokens/frame


__all__.append("random_family_blank_bias")


# (5) batch-sharded sweep: 8192 utterances with LibriSpeech-like lengths (seed
# 2024), FastConformer shapes, RNN-T and TDT; batches of 32.
SWEEPS = {
    "sweep-rnnt": dict(spec=CONFIGS["fc-rnnt"]["spec"], n_utt=8192, batch=32, length_seed=2024),
    "sweep-tdt": dict(spec=CONFIGS["fc-tdt"]["spec"], n_utt=8192, batch=32, length_seed=2024),
}
