"""Transducer model pieces in float64 (TEST INFRASTRUCTURE, see oracle/__init__.py).

Fig. 1: encoder -> joiner <- predictor.  The encoder itself is
out of scope: its outputs `enc[t]` are the inputs.  Two linear projections map
encoder and predictor outputs into the joint space (§3.4):
    f[t] = W_enc enc[t] + b_enc          (precomputed once, Alg. 3 line 2)
    g    = W_pred dec + b_pred           (once per predictor call, Alg. 3 line 6)
Joiner (reading A11, north_star): logits = W_out ReLU(f[t] + g) + b_out,
TDT duration head sharing z (A12): dur_logits = W_dur ReLU(f[t] + g) + b_dur.
Predictor (Alg. 1 lines 6-8, `dec, new_state = predictor(state, label)`):
  LSTM (A9): PyTorch nn.LSTM convention, gate rows i,f,g,o, two biases,
      x = Emb[label]; c' = s(f) c + s(i) tanh(g); h' = s(o) tanh(c'); dec = h'.
  stateless (A10): state = last c labels (most recent first),
      dec = concat_k Emb_k[state'[k]], no nonlinearity.
Initial state (A8): h = c = 0, stateless context = [blank]*c; SOS = blank (A7).
"""
from __future__ import annotations

import numpy as np


def argmax_lowest(v: np.ndarray) -> int:
    """argmax with the lowest index among ties (PAPER.md:141 `argmax`; tie rule A16)."""
    v = np.asarray(v)
    m = v.max()
    return int(np.flatnonzero(v == m)[0])


def log_prob(v: np.ndarray, i: int) -> float:
    """log softmax(v)[i] = v[i] - log sum_j exp(v[j]) (the greedy score term of
    one argmax step; BatchedHyps "scores", read per SPEC.md:239 /
    :266 as the log-probability of every argmax step, blanks included).  The
    max is subtracted before exp for range only (exact identity)."""
    v = np.asarray(v, dtype=np.float64)
    m = v.max()
    return float(v[i] - (m + np.log(np.exp(v - m).sum())))


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


class Transducer:
    """A Transducer with weights given in the C-ABI layout (synth.make_weights).

    All arrays are converted to float64; the values are the exact bf16 (or
    f32) values the GPU receives (reading A24)."""

    def __init__(self, weights: dict, blank_id: int = 0, pred_kind: str = "lstm",
                 context: int = 1, durations=None):
        self.w = {k: np.asarray(v, dtype=np.float64) for k, v in weights.items()}
        self.blank = int(blank_id)
        self.kind = pred_kind
        self.context = int(context)
        self.durations = None if durations is None else [int(d) for d in durations]
        self.num_tokens = self.w["w_out"].shape[0]
        self.H = self.w["w_out"].shape[1]
        if pred_kind == "lstm":
            self.P = self.w["w_hh"].shape[1]
            self.layers = 1 + (self.w["w_ih_rest"].shape[0] if "w_ih_rest" in self.w else 0)
        else:
            self.P = self.context * self.w["embedding"].shape[2]

    @classmethod
    def from_spec(cls, spec, weights):
        return cls(weights, spec.blank_id, spec.pred_kind, spec.context, spec.durations)

    # -- encoder projection, PAPER.md:219 / Alg. 3 line 2 (:134) -----------------
    def enc_proj(self, enc_rows: np.ndarray) -> np.ndarray:
        """f[t] = W_enc enc[t] + b_enc for every given frame ([T, D_e] -> [T, H])."""
        enc_rows = np.asarray(enc_rows, dtype=np.float64)
        return enc_rows @ self.w["w_enc"].T + self.w["b_enc"]

    # -- predictor, Alg. 1 lines 62-68 (:62-68) ----------------------------------
    def pred_init(self):
        """predictor.init_state() (Alg. 1 line 3): zeros / context of blanks (A8)."""
        if self.kind == "lstm":
            return (np.zeros((self.layers, self.P)), np.zeros((self.layers, self.P)))
        return tuple([self.blank] * self.context)

    def pred_step(self, state, label: int):
        """dec, new_state = predictor(state, label) (Alg. 1 line 65/67)."""
        if self.kind == "lstm":
            # a stack of `layers` cells (PyTorch nn.LSTM, num_layers = L; reading
            # A9): layer 0 reads the embedding, layer l the new h of layer l-1
            hs, cs = state
            x = self.w["embedding"][label]
            P = self.P
            h_new, c_new = np.empty_like(hs), np.empty_like(cs)
            for layer in range(self.layers):
                if layer == 0:
                    w_ih, w_hh, b_ih, b_hh = self.w["w_ih"], self.w["w_hh"], self.w["b_ih"], self.w["b_hh"]
                else:
                    w_ih, w_hh = self.w["w_ih_rest"][layer - 1], self.w["w_hh_rest"][layer - 1]
                    b_ih, b_hh = self.w["b_ih_rest"][layer - 1], self.w["b_hh_rest"][layer - 1]
                gates = (w_ih @ x + b_ih) + (w_hh @ hs[layer] + b_hh)
                i = _sigmoid(gates[0:P])
                f = _sigmoid(gates[P:2 * P])
                g = np.tanh(gates[2 * P:3 * P])
                o = _sigmoid(gates[3 * P:4 * P])
                c_new[layer] = f * cs[layer] + i * g
                h_new[layer] = o * np.tanh(c_new[layer])
                x = h_new[layer]
            return h_new[-1], (h_new, c_new)
        new_state = (int(label),) + tuple(state[:-1])
        dec = np.concatenate([self.w["embedding"][k][new_state[k]] for k in range(self.context)])
        return dec, new_state

    def pred_proj(self, dec: np.ndarray) -> np.ndarray:
        """g = W_pred dec + b_pred."""
        return self.w["w_pred"] @ dec + self.w["b_pred"]

    # -- joiner, PAPER.md:41 / Alg. 3 lines 7, 13 --------------------------------
    def joint_z(self, f_t: np.ndarray, g: np.ndarray) -> np.ndarray:
        return np.maximum(f_t + g, 0.0)

    def joint(self, f_t: np.ndarray, g: np.ndarray):
        """Token logits [V+1] (and TDT duration logits [|D|], else None)."""
        z = self.joint_z(f_t, g)
        logits = self.w["w_out"] @ z + self.w["b_out"]
        dur = None
        if self.durations is not None:
            dur = self.w["w_dur"] @ z + self.w["b_dur"]
        return logits, dur
