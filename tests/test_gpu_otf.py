"""GPU parity of the on-the-fly projection arm (ll_options.projections = 1):
the ablation of the paper's Table 3 ("Decoding RTFx between
precomputation of projections and on-the-fly projections").  The decode kernel
applies W_enc and W_pred at every joint evaluation instead of reading the
precomputed f / g.  Same bar as the precompute path: every row
passes the float64 teacher-forced verifier (1e-3 near-ties), the planted family
decodes to its planted alignment exactly, and the algorithmic decisions (joint
evaluations, labels) equal the precompute path's.
"""
import numpy as np
import pytest

import synth
from gpu_helpers import gpu_decode, gpu_model, verify_all
from paper_2406_06220_b200 import ll

pytestmark = pytest.mark.gpu


def _decode(spec, w, enc, lengths, model=None, otf=True, **kw):
    with ll.options(projections=1 if otf else 0, **kw):
        return gpu_decode(spec, w, enc, lengths, model=model)


@pytest.mark.parametrize("cfg", ["fc-rnnt", "fc-tdt"])
def test_otf_planted_full_batch(cfg):
    """Config 2 / 3 at full size, planted family: the on-the-fly decode equals the
    planted alignment and the precompute decode, with identical joint-evaluation
    and label counts; sampled rows pass the float64 verifier."""
    c = synth.CONFIGS[cfg]
    spec = c["spec"]
    if spec.is_tdt:
        w, enc, lengths, planted = synth.make_planted_tdt(spec, 6, c["B"], c["T_max"], c["len_lo"], c["len_hi"])
    else:
        w, enc, lengths, planted = synth.make_planted_rnnt(spec, 5, c["B"], c["T_max"], c["len_lo"], c["len_hi"])
    model = gpu_model(spec, w)
    h_otf, d_otf = _decode(spec, w, enc, lengths, model)
    h_pre, d_pre = _decode(spec, w, enc, lengths, model, otf=False)
    for b in range(c["B"]):
        if spec.is_tdt:
            assert h_otf[b] == planted[b], b
        else:
            assert (h_otf[b][0], h_otf[b][1]) == (planted[b][0], planted[b][1]), b
    assert h_otf == h_pre
    s_otf, s_pre = d_otf.stats(), d_pre.stats()
    for k in ("joint_evals", "labels"):
        assert s_otf[k] == s_pre[k], k
    verify_all(spec, w, enc, lengths, h_otf, rows=[0, 11, 31])


@pytest.mark.parametrize("cfg", ["fc-rnnt", "fc-tdt"])
def test_otf_random_family_full_batch(cfg):
    """Random family at config 2 / 3 (near-ties present): all 32 rows of the
    on-the-fly decode pass the teacher-forced float64 verifier."""
    c = synth.CONFIGS[cfg]
    spec = c["spec"]
    w = synth.make_weights(spec, 21, blank_bias=synth.random_family_blank_bias(spec))
    enc, lengths = synth.make_inputs(22, c["B"], c["T_max"], spec.enc_dim, c["len_lo"], c["len_hi"])
    hyps, _ = _decode(spec, w, enc, lengths)
    ties, decs = verify_all(spec, w, enc, lengths, hyps)
    labels = sum(len(h[0]) for h in hyps)
    print(f"otf {cfg}: {labels} labels, {decs} decisions, {ties} near-ties")
    assert labels > 32 * 50
    assert ties <= decs * 0.02


@pytest.mark.parametrize("B", [1, 4, 9])
def test_otf_table3_batch_sizes(B):
    """Table 3's batch sizes (1, 4, 32; 9: a ragged group count): every row
    verified, lengths ragged, including a zero-length utterance at B = 9."""
    c = synth.CONFIGS["fc-rnnt"]
    spec = c["spec"]
    w = synth.make_weights(spec, 31, blank_bias=synth.random_family_blank_bias(spec))
    enc, lengths = synth.make_inputs(32 + B, B, c["T_max"], spec.enc_dim, c["len_lo"], c["len_hi"])
    if B == 9:
        lengths[3] = 0
        lengths[7] = 1
    hyps, _ = _decode(spec, w, enc, lengths)
    verify_all(spec, w, enc, lengths, hyps)
    if B == 9:
        assert hyps[3][0] == []


def test_otf_determinism():
    """Bit-identical repeat runs (fixed reduction orders; 11 runs) and
    batch-composition independence (a row decodes the same alone and inside the
    batch)."""
    c = synth.CONFIGS["fc-rnnt"]
    spec = c["spec"]
    w = synth.make_weights(spec, 51, blank_bias=synth.random_family_blank_bias(spec))
    enc, lengths = synth.make_inputs(52, 12, c["T_max"], spec.enc_dim, c["len_lo"], c["len_hi"])
    model = gpu_model(spec, w)
    a, _ = _decode(spec, w, enc, lengths, model)
    for _ in range(10):   # a race on the cross-CTA z exchange would show as run-to-run differences
        b, _ = _decode(spec, w, enc, lengths, model)
        assert a == b
    one, _ = _decode(spec, w, enc[5:6], lengths[5:6], model)
    assert one[0] == a[5]


@pytest.mark.parametrize("case", ["stateless", "f32", "batched", "scores", "tiny"])
def test_otf_unsupported(case):
    """Outside the FC LSTM tick kernel the option is refused (LL_ERR_UNSUPPORTED),
    before any work is enqueued."""
    c = synth.CONFIGS["tiny" if case == "tiny" else "fc-rnnt"]
    spec = c["spec"]
    dtype = "f32" if case == "f32" else "bf16"
    if case == "stateless":
        spec = synth.ModelSpec(1025, 512, 640, 640, "stateless", 2, None, 0, 10)
    w = synth.make_weights(spec, 7)
    enc, lengths = synth.make_inputs(8, 2, 20, spec.enc_dim, 5, 20)
    model = gpu_model(spec, w, dtype)
    opts = {"schedule": 0} if case == "batched" else {}
    with pytest.raises(ll.LLError) as e:
        with ll.options(projections=1, **opts):
            if case == "scores":
                import torch
                from paper_2406_06220_b200.decoder import LabelLoopingDecoder
                dec = LabelLoopingDecoder(model, spec.max_symbols, 2, 20, scores=True)
                dec.decode(torch.from_numpy(enc).to("cuda", model.tdtype),
                           torch.from_numpy(np.asarray(lengths, np.int32)).cuda())
            else:
                gpu_decode(spec, w, enc, lengths, dtype, model=model)
    assert e.value.status == ll.LL_ERR_UNSUPPORTED
