"""User-facing wrapper over the C ABI: device-resident model + decode calls.

PyTorch is used only for device memory and streams; all decoding runs in
libll.so through the functions of `ll.py`.  Typical use:

    model = Model(weights, pred_kind="lstm", blank_id=0)              # numpy/torch weights
    dec = LabelLoopingDecoder(model, max_symbols=10, B_max=32, T_max=275)
    out = dec.decode(enc_dev, lengths_dev)                            # device tensors in/out
    toks = out.hypotheses()                                           # list of (tokens, timestamps[, durations])
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import ll

_DT = {"bf16": (ll.LL_BF16, torch.bfloat16), "f32": (ll.LL_F32, torch.float32)}


def _dev(x, dtype, device):
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    return x.to(device=device, dtype=dtype).contiguous()


class Model:
    """Transducer decoding weights on the device, in the ABI layout of ll.h."""

    def __init__(self, weights: Dict[str, object], pred_kind: str = "lstm", context: int = 1,
                 blank_id: int = 0, durations: Optional[Sequence[int]] = None, dtype: str = "bf16",
                 device: str = "cuda"):
        self.dtype_code, tdtype = _DT[dtype]
        self.dtype = dtype
        self.tdtype = tdtype
        self.device = device
        self.blank_id = int(blank_id)
        self.durations = None if durations is None else [int(d) for d in durations]
        self.t = {k: _dev(v, tdtype, device) for k, v in weights.items()}
        w = self.t
        V1, H = w["w_out"].shape
        P = w["w_pred"].shape[1]
        De = w["w_enc"].shape[1]
        self.V1, self.H, self.P, self.De = int(V1), int(H), int(P), int(De)
        ptr = lambda k: w[k].data_ptr() if k in w else None
        self.pred = ll.ll_predictor(
            ll.LL_PRED_LSTM if pred_kind == "lstm" else ll.LL_PRED_STATELESS, self.V1, self.P,
            int(context), ptr("embedding"), ptr("w_ih"), ptr("w_hh"), ptr("b_ih"), ptr("b_hh"),
            1 + (int(w["w_ih_rest"].shape[0]) if "w_ih_rest" in w else 0),   # LSTM layers (ll.h)
            ptr("w_ih_rest"), ptr("w_hh_rest"), ptr("b_ih_rest"), ptr("b_hh_rest"))
        self.joint = ll.ll_joint(self.De, self.P, self.H, self.V1, ptr("w_enc"), ptr("b_enc"),
                                 ptr("w_pred"), ptr("b_pred"), ptr("w_out"), ptr("b_out"),
                                 ptr("w_dur"), ptr("b_dur"))

    @property
    def num_durations(self) -> int:
        return 0 if self.durations is None else len(self.durations)


@dataclasses.dataclass
class DecodeOutput:
    tokens: torch.Tensor        # [B, cap] int32
    timestamps: torch.Tensor    # [B, cap] int32
    durations: Optional[torch.Tensor]
    lengths: torch.Tensor       # [B] int32
    scores: Optional[torch.Tensor] = None   # [B] f32 greedy scores (decoders built with scores=True)

    def hypotheses(self) -> List[tuple]:
        """Per-utterance python lists (copies to the host)."""
        L = self.lengths.cpu().tolist()
        tk, ts = self.tokens.cpu(), self.timestamps.cpu()
        du = self.durations.cpu() if self.durations is not None else None
        out = []
        for b, n in enumerate(L):
            n = min(n, tk.shape[1])
            h = (tk[b, :n].tolist(), ts[b, :n].tolist())
            if du is not None:
                h = h + (du[b, :n].tolist(),)
            out.append(h)
        return out


class LabelLoopingDecoder:
    """Owns the workspace and output buffers for batches up to (B_max, T_max)."""

    def __init__(self, model: Model, max_symbols: int, B_max: int, T_max: int, cap: Optional[int] = None,
                 prec: int = ll.LL_PREC_FAST, frame_looping: bool = False, scores: bool = False):
        """frame_looping=True runs the Alg. 2 baseline (ll_decode_rnnt_frame_looping,
        RNN-T only) instead of label-looping."""
        if frame_looping and model.durations is not None:
            raise ValueError("frame-looping baseline: RNN-T only")
        self.frame_looping = bool(frame_looping)
        if scores and frame_looping:
            raise ValueError("greedy scores: label-looping only")
        self.with_scores = bool(scores)
        self.model = model
        self.max_symbols = int(max_symbols)
        self.B_max, self.T_max = int(B_max), int(T_max)
        self.cap = int(cap) if cap is not None else max(1, self.T_max * self.max_symbols)
        self.prec = prec
        nD = model.num_durations
        self.ws_bytes = ll.ll_workspace_size(self.B_max, self.T_max, model.pred, model.joint,
                                             model.dtype_code, prec, nD)
        if self.ws_bytes == 0:
            raise ll.LLError(ll.LL_ERR_INVALID_ARGUMENT, "ll_workspace_size")
        dev = model.device
        self.workspace = torch.empty(self.ws_bytes + 256, dtype=torch.uint8, device=dev)
        base = self.workspace.data_ptr()
        self.ws_ptr = (base + 255) // 256 * 256
        self.tokens = torch.zeros(self.B_max, self.cap, dtype=torch.int32, device=dev)
        self.timestamps = torch.zeros_like(self.tokens)
        self.durs = torch.zeros_like(self.tokens) if nD else None
        self.lengths_out = torch.zeros(self.B_max, dtype=torch.int32, device=dev)
        self.scores = torch.zeros(self.B_max, dtype=torch.float32, device=dev) if self.with_scores else None

    def release(self) -> None:
        """ll_release: drop the library's ll_prepare record of this workspace
        (called before the workspace memory goes back to the allocator)."""
        if getattr(self, "ws_ptr", None):
            ll.ll_release(self.ws_ptr)

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass

    def prepare(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """ll_prepare: build the weight-only model tables into this decoder's
        workspace once; later decodes skip them while the weights (pointers)
        and shapes stay the same."""
        m = self.model
        st = (stream or torch.cuda.current_stream()).cuda_stream
        s = ll.ll_prepare(m.pred, m.joint, m.dtype_code, self.prec, self.B_max, self.T_max, m.durations,
                          m.num_durations, self.ws_ptr, self.ws_bytes, st)
        if s != ll.LL_OK:
            raise ll.LLError(s, "ll_prepare")

    def launch(self, enc: torch.Tensor, lengths: torch.Tensor, stream: Optional[torch.cuda.Stream] = None,
               out: Optional[tuple] = None) -> int:
        """Enqueue a decode of enc [B, T, D_e] (device, model dtype) with lengths [B] int32 (device).
        out: optional (tokens, timestamps, durations or None, lengths) device int32 tensors of
        [>= B, self.cap] / [>= B] to write instead of this decoder's own buffers (e.g. row
        slices of one large buffer: the rows of a [N, cap] tensor are contiguous)."""
        m = self.model
        B, T = int(enc.shape[0]), int(enc.shape[1])
        assert B <= self.B_max and T <= self.T_max and enc.is_contiguous() and lengths.dtype == torch.int32
        tok, ts, du, ln = out[:4] if out is not None else (self.tokens, self.timestamps, self.durs, self.lengths_out)
        if out is not None:
            assert tok.shape[1] == self.cap and ts.shape[1] == self.cap and tok.is_contiguous() and ts.is_contiguous()
        st = (stream or torch.cuda.current_stream()).cuda_stream
        if self.with_scores:   # ll_decode_*_scores (N2)
            sc = (out[4] if out is not None and len(out) > 4 else self.scores).data_ptr()
            if m.durations is None:
                return ll.ll_decode_rnnt_scores(enc.data_ptr(), m.dtype_code, self.prec, B, T, lengths.data_ptr(),
                                                m.pred, m.joint, m.blank_id, self.max_symbols, tok.data_ptr(),
                                                ts.data_ptr(), ln.data_ptr(), self.cap, sc, self.ws_ptr,
                                                self.ws_bytes, st)
            return ll.ll_decode_tdt_scores(enc.data_ptr(), m.dtype_code, self.prec, B, T, lengths.data_ptr(),
                                           m.pred, m.joint, m.blank_id, self.max_symbols, m.durations,
                                           m.num_durations, tok.data_ptr(), ts.data_ptr(),
                                           None if du is None else du.data_ptr(), ln.data_ptr(), self.cap, sc,
                                           self.ws_ptr, self.ws_bytes, st)
        if m.durations is None:
            fn = ll.ll_decode_rnnt_frame_looping if self.frame_looping else ll.ll_decode_rnnt
            return fn(enc.data_ptr(), m.dtype_code, self.prec, B, T, lengths.data_ptr(),
                      m.pred, m.joint, m.blank_id, self.max_symbols, tok.data_ptr(),
                      ts.data_ptr(), ln.data_ptr(), self.cap, self.ws_ptr, self.ws_bytes, st)
        return ll.ll_decode_tdt(enc.data_ptr(), m.dtype_code, self.prec, B, T, lengths.data_ptr(), m.pred,
                                m.joint, m.blank_id, self.max_symbols, m.durations, m.num_durations,
                                tok.data_ptr(), ts.data_ptr(), None if du is None else du.data_ptr(),
                                ln.data_ptr(), self.cap, self.ws_ptr, self.ws_bytes, st)

    def decode(self, enc: torch.Tensor, lengths: torch.Tensor, stream=None, check: bool = True) -> DecodeOutput:
        B = int(enc.shape[0])
        s = self.launch(enc, lengths, stream)
        if s != ll.LL_OK:
            raise ll.LLError(s, "decode")
        if check:
            s = self.sync(stream)
            if s != ll.LL_OK:
                raise ll.LLError(s, "ll_sync")
        return DecodeOutput(self.tokens[:B], self.timestamps[:B],
                            None if self.durs is None else self.durs[:B], self.lengths_out[:B],
                            None if self.scores is None else self.scores[:B])

    def sync(self, stream=None) -> int:
        st = (stream or torch.cuda.current_stream()).cuda_stream
        return ll.ll_sync(self.ws_ptr, st)

    def stats(self, stream=None) -> Dict[str, int]:
        st = (stream or torch.cuda.current_stream()).cuda_stream
        s, v = ll.ll_stats(self.ws_ptr, st)
        if s != ll.LL_OK:
            raise ll.LLError(s, "ll_stats")
        keys = ["outer_steps", "joint_rounds", "joint_evals", "predictor_steps", "predictor_rows",
                "labels", "groups", "cluster_size", "joint_rows_computed", "window", "group_rows", "chain",
                "launches"]
        d = dict(zip(keys, v))
        c = d.pop("chain")
        d["chain_rounds"], d["chain_pred_steps"] = (c >> 20) & 0xFFFFF, c & 0xFFFFF
        return d


def debug_joint(model: Model, enc_rows: torch.Tensor, g_rows: torch.Tensor, want_logits: bool = True,
                prec: int = ll.LL_PREC_FAST):
    """ll_debug_joint on n rows: returns (logits [n, V+1+|D|] or None, argmax [n], dur_argmax [n] or None)."""
    n = int(enc_rows.shape[0])
    nD = model.num_durations
    pred = ll.ll_predictor(ll.LL_PRED_STATELESS, model.V1, model.P, 1, None, None, None, None, None)
    ws_bytes = ll.ll_workspace_size(n, 1, pred, model.joint, model.dtype_code, prec, nD)
    ws = torch.empty(ws_bytes + 256, dtype=torch.uint8, device=model.device)
    ws_ptr = (ws.data_ptr() + 255) // 256 * 256
    logits = torch.empty(n, model.V1 + nD, dtype=torch.float32, device=model.device) if want_logits else None
    am = torch.empty(n, dtype=torch.int32, device=model.device)
    dam = torch.empty(n, dtype=torch.int32, device=model.device) if nD else None
    st = torch.cuda.current_stream().cuda_stream
    s = ll.ll_debug_joint(enc_rows.data_ptr(), g_rows.data_ptr(), n, model.joint, model.dtype_code,
                          prec, nD, logits.data_ptr() if logits is not None else None,
                          am.data_ptr(), dam.data_ptr() if dam is not None else None, ws_ptr, ws_bytes, st)
    if s != ll.LL_OK:
        raise ll.LLError(s, "ll_debug_joint")
    torch.cuda.current_stream().synchronize()
    return logits, am, dam


def probe_decode(dec: "LabelLoopingDecoder", enc: torch.Tensor, lengths: torch.Tensor, rows: int = 8192,
                 regions: int = 8, **opts):
    """Decode through the production FastConformer kernel instantiation with its
    probe hook (ll.h ll_options): returns (DecodeOutput, joint rows, g rows) where
    joint rows = list of (b, t, n_labels, logits [V+1+|D|]) and g rows = list of
    (b, n_labels, g [H]) as numpy arrays (parity tests only).  opts: further
    ll_options fields (e.g. group_rows)."""
    m = dec.model
    NV = m.V1 + m.num_durations
    dev = m.device
    pl = torch.full((regions, rows, NV), float("nan"), dtype=torch.float32, device=dev)
    lm = torch.zeros(regions, rows, 4, dtype=torch.int32, device=dev)
    pg = torch.full((regions, rows, m.H), float("nan"), dtype=torch.float32, device=dev)
    gm = torch.zeros(regions, rows, 4, dtype=torch.int32, device=dev)
    cnt = torch.zeros(regions, 2, dtype=torch.int32, device=dev)
    with ll.options(probe_logits=pl.data_ptr(), probe_lmeta=lm.data_ptr(), probe_g=pg.data_ptr(),
                    probe_gmeta=gm.data_ptr(), probe_counts=cnt.data_ptr(), probe_rows=rows,
                    probe_regions=regions, **opts):
        out = dec.decode(enc, lengths)
    torch.cuda.synchronize()
    cnt = cnt.cpu().numpy()
    if (cnt > rows).any():
        raise RuntimeError(f"probe truncated: {cnt.max()} rows > {rows}")
    pl, lm, pg, gm = pl.cpu().numpy(), lm.cpu().numpy(), pg.cpu().numpy(), gm.cpu().numpy()
    joint = [(int(lm[r, i, 0]), int(lm[r, i, 1]), int(lm[r, i, 2]), pl[r, i]) for r in range(regions)
             for i in range(cnt[r, 0])]
    gro = [(int(gm[r, i, 0]), int(gm[r, i, 1]), pg[r, i]) for r in range(regions) for i in range(cnt[r, 1])]
    return out, joint, gro
