"""Small decodes of every kernel family, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
    compute-sanitizer --tool synccheck python tools/sanitize_run.py

Covers: the generic cluster kernel (tiny RNN-T / TDT, stateless), the
FastConformer-shape kernels (LSTM predictor with W_hh in TMEM, tcgen05 GEMM
projections, tick schedule; RNN-T and TDT, planted family so every row emits
labels), the stateless FC-shape kernel, the frame-looping baseline, the
batched Alg. 3 schedule (ll_options.schedule = 0), the on-the-fly projection
kernels (ll_options.projections = 1), LL_PREC_EXACT (widening + fp32 kernels)
and the native ragged gather (world size 1).  Each decode's hypotheses are compared
with the planted alignment / checked for well-formedness; the point of the run
is the sanitizer's report."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2406_06220_b200 import ll, shard  # noqa: E402
from paper_2406_06220_b200.decoder import LabelLoopingDecoder, Model  # noqa: E402


def run_tiny(cfg):
    c = synth.CONFIGS[cfg]
    spec = c["spec"]
    w = synth.make_weights(spec, 1, blank_bias=0.5)
    enc, lengths = synth.make_inputs(2, c["B"], c["T_max"], spec.enc_dim, c["len_lo"], c["len_hi"])
    model = Model(w, spec.pred_kind, spec.context, spec.blank_id, spec.durations, "bf16")
    dec = LabelLoopingDecoder(model, spec.max_symbols, c["B"], c["T_max"])
    out = dec.decode(torch.from_numpy(enc).to("cuda", torch.bfloat16), torch.from_numpy(lengths).cuda())
    print(cfg, "rows", len(out.hypotheses()), flush=True)


def run_planted(cfg, B, frame_looping=False, gather=False, scores=False, prec=ll.LL_PREC_FAST):
    c = synth.CONFIGS[cfg]
    spec = c["spec"]
    w, codes = synth.planted_weights(spec, 1000)
    L = np.array([40 + 7 * i for i in range(B)])
    T = int(L.max())
    enc = np.zeros((B, T, spec.enc_dim), dtype=np.float32)
    planted = []
    for i in range(B):
        e, pl = synth.planted_utterance(spec, codes, 77, i, int(L[i]))
        enc[i, :e.shape[0]] = e
        planted.append(pl)
    model = Model(w, spec.pred_kind, spec.context, spec.blank_id, spec.durations, "bf16")
    dec = LabelLoopingDecoder(model, spec.max_symbols, B, T, frame_looping=frame_looping, scores=scores, prec=prec)
    lengths = torch.from_numpy(L.astype(np.int32)).cuda()
    out = dec.decode(torch.from_numpy(enc).to("cuda", torch.bfloat16), lengths)
    hy = out.hypotheses()
    ok = all(tuple(hy[i][:len(planted[i])]) == tuple(planted[i]) for i in range(B))
    print(cfg, "frame-looping" if frame_looping else "label-looping", "B", B, "planted equal:", ok, flush=True)
    if gather:
        g = shard.NcclGather()
        ids = torch.arange(B, dtype=torch.int32, device="cuda")
        rec = g.gather(ids, out.lengths, out.tokens, out.timestamps, out.durations)
        g.close()
        got = shard.unpack_records(rec.cpu().numpy(), spec.is_tdt)
        print("gather records equal:", all(got[i] == tuple(hy[i]) for i in range(B)), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:   # one case: tiny | fc | fc-batched
        {"tiny": lambda: run_tiny("tiny"), "fc": lambda: run_planted("fc-rnnt", 6)}.get(sys.argv[1], lambda: None)()
        if sys.argv[1] == "fc-batched":
            with ll.options(schedule=0):
                run_planted("fc-rnnt", 6)
        torch.cuda.synchronize()
        sys.exit(0)
    run_tiny("tiny")
    run_tiny("tiny-tdt")
    run_planted("fc-rnnt", 6, gather=True)
    run_planted("fc-tdt", 6, gather=True)
    run_planted("fc-rnnt", 4, frame_looping=True)
    run_planted("stateless-b512", 20)
    run_planted("fc-rnnt", 6, scores=True)   # greedy scores (N2): the SC kernels
    run_planted("fc-tdt", 6, scores=True)
    with ll.options(schedule=0):   # the paper's batched outer loop (Alg. 3 as listed)
        run_tiny("tiny")
        run_planted("fc-rnnt", 6)
        run_planted("fc-tdt", 6)
    with ll.options(projections=1):   # on-the-fly projections (Table 3 arm): the LM = 4 kernels
        run_planted("fc-rnnt", 6)
        run_planted("fc-tdt", 6)
    run_planted("fc-rnnt", 3, prec=ll.LL_PREC_EXACT)   # widening kernels + the fp32 kernels
    torch.cuda.synchronize()
    print("sanitize_run done", flush=True)
