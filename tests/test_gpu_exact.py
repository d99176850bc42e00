"""GPU parity of LL_PREC_EXACT with bf16 inputs and of bf16 multi-layer LSTM
predictors (ll.h: both run the fp32 kernels on fp32 copies of the bf16 values).

Every bf16 value is an fp32 value, so a bf16 model decoded under LL_PREC_EXACT
must equal, bit for bit, the same values given as LL_F32 weights (the fp32
path), and its joint logits must meet the fp32 tolerance of north_star (1e-5
absolute against float64).  Rows are also teacher-forced against the float64
oracle (1e-3 near-ties)."""
import numpy as np
import pytest
import torch

import synth
from gpu_helpers import gpu_model, verify_all
from oracle import Transducer
from paper_2406_06220_b200 import ll
from paper_2406_06220_b200.decoder import LabelLoopingDecoder, debug_joint

pytestmark = pytest.mark.gpu


def _decode(spec, model, enc, lengths, prec, scores=False, frame_looping=False):
    B, T = enc.shape[0], enc.shape[1]
    dec = LabelLoopingDecoder(model, spec.max_symbols, B, T, prec=prec, scores=scores, frame_looping=frame_looping)
    out = dec.decode(torch.from_numpy(np.ascontiguousarray(enc)).to("cuda", model.tdtype),
                     torch.from_numpy(np.asarray(lengths, np.int32)).cuda())
    return out.hypotheses(), (None if out.scores is None else out.scores.cpu().numpy())


@pytest.mark.parametrize("cfg", ["tiny", "tiny-tdt", "fc-rnnt", "fc-tdt"])
def test_exact_equals_f32_path(cfg):
    """bf16 model + LL_PREC_EXACT == the same values as fp32 weights (bit-exact
    hypotheses); rows verified against float64."""
    c = synth.CONFIGS[cfg]
    spec = c["spec"]
    fam = synth.random_family_blank_bias(spec) if spec.joint_dim >= 70 else 0.5
    w = synth.make_weights(spec, 61, blank_bias=fam)
    B = c["B"] if spec.joint_dim < 70 else 8
    enc, lengths = synth.make_inputs(62, B, c["T_max"], spec.enc_dim, c["len_lo"], c["len_hi"])
    h_exact, _ = _decode(spec, gpu_model(spec, w, "bf16"), enc, lengths, ll.LL_PREC_EXACT)
    h_f32, _ = _decode(spec, gpu_model(spec, w, "f32"), enc, lengths, ll.LL_PREC_FAST)
    assert h_exact == h_f32
    verify_all(spec, w, enc, lengths, h_exact, rows=None if B <= 8 else list(range(0, B, 3)))


@pytest.mark.parametrize("shape", ["fc", "tiny"])
@pytest.mark.parametrize("tdt", [False, True])
def test_exact_joint_logits(shape, tdt):
    """ll_debug_joint with bf16 inputs under LL_PREC_EXACT: logits within the fp32
    tolerance (1e-5) of float64; argmax equal except at float64 near-ties."""
    durs = (0, 1, 2, 3, 4) if tdt else None
    if shape == "fc":
        spec = synth.ModelSpec(1025, 512, 640, 640, "lstm", 1, durs, 0, 10)
    else:
        spec = synth.ModelSpec(9, 16, 16, 16, "stateless", 1, durs, 0, 3)
    w = synth.make_weights(spec, 71, blank_bias=0.3)
    rng = np.random.default_rng(71)
    n = 45
    enc = synth.bf16_round(rng.normal(0, 1, size=(n, spec.enc_dim)))
    g = rng.normal(0, 0.5, size=(n, spec.joint_dim)).astype(np.float32)
    model = gpu_model(spec, w, "bf16")
    logits, am, dam = debug_joint(model, torch.from_numpy(enc).to("cuda", torch.bfloat16),
                                  torch.from_numpy(g).cuda(), prec=ll.LL_PREC_EXACT)
    o = Transducer.from_spec(spec, w)
    f = o.enc_proj(enc)
    ref = []
    for i in range(n):
        l, dl = o.joint(f[i], g[i].astype(np.float64))
        ref.append(np.concatenate([l, dl]) if tdt else l)
    ref = np.array(ref)
    err = np.abs(logits.cpu().numpy().astype(np.float64) - ref).max()
    assert err < 1e-5, err
    am = am.cpu().numpy()
    V1 = spec.num_tokens
    for i in range(n):
        assert am[i] == int(np.argmax(ref[i, :V1])) or ref[i, :V1].max() - ref[i, am[i]] < 1e-3


@pytest.mark.parametrize("cfg", ["tiny", "tiny-tdt"])
@pytest.mark.parametrize("layers", [2, 3])
def test_multilayer_lstm_bf16(cfg, layers):
    """N4 "more layers" with bf16 weights: identical to the fp32
    path on the same values (bit-exact), every row verified against the float64
    L-layer oracle."""
    c = synth.CONFIGS[cfg]
    spec = c["spec"]
    for seed in range(4):
        sp = synth.ModelSpec(spec.num_tokens, spec.enc_dim, spec.pred_dim, spec.joint_dim, "lstm", 1,
                             spec.durations, spec.blank_id, spec.max_symbols, num_layers=layers)
        w = synth.make_weights(sp, 5000 + seed, blank_bias=0.5)
        enc, lengths = synth.make_inputs(6000 + seed, c["B"], c["T_max"], sp.enc_dim, c["len_lo"], c["len_hi"])
        h_bf, _ = _decode(sp, gpu_model(sp, w, "bf16"), enc, lengths, ll.LL_PREC_FAST)
        h_32, _ = _decode(sp, gpu_model(sp, w, "f32"), enc, lengths, ll.LL_PREC_FAST)
        assert h_bf == h_32
        verify_all(sp, w, enc, lengths, h_bf)


def test_multilayer_lstm_bf16_fc_shape():
    """A 2-layer LSTM predictor at the FastConformer shape (P = H = 640) with
    bf16 weights: decodes, equals the fp32 path, sampled rows verified."""
    c = synth.CONFIGS["fc-rnnt"]
    spec = c["spec"]
    sp = synth.ModelSpec(spec.num_tokens, spec.enc_dim, spec.pred_dim, spec.joint_dim, "lstm", 1,
                         None, spec.blank_id, spec.max_symbols, num_layers=2)
    w = synth.make_weights(sp, 81, blank_bias=synth.random_family_blank_bias(spec))
    enc, lengths = synth.make_inputs(82, 6, c["T_max"], sp.enc_dim, c["len_lo"], c["len_hi"])
    h_bf, _ = _decode(sp, gpu_model(sp, w, "bf16"), enc, lengths, ll.LL_PREC_FAST)
    h_32, _ = _decode(sp, gpu_model(sp, w, "f32"), enc, lengths, ll.LL_PREC_FAST)
    assert h_bf == h_32
    verify_all(sp, w, enc, lengths, h_bf, rows=[0, 5])


def test_exact_scores_and_frame_looping():
    """The EXACT path carries the other entry points: greedy scores equal the fp32
    path's, and the frame-looping baseline gives the label-looping hypotheses."""
    c = synth.CONFIGS["tiny"]
    spec = c["spec"]
    w = synth.make_weights(spec, 91, blank_bias=0.5)
    enc, lengths = synth.make_inputs(92, c["B"], c["T_max"], spec.enc_dim, c["len_lo"], c["len_hi"])
    mb, m32 = gpu_model(spec, w, "bf16"), gpu_model(spec, w, "f32")
    h1, s1 = _decode(spec, mb, enc, lengths, ll.LL_PREC_EXACT, scores=True)
    h2, s2 = _decode(spec, m32, enc, lengths, ll.LL_PREC_FAST, scores=True)
    assert h1 == h2 and np.array_equal(s1, s2)
    h3, _ = _decode(spec, mb, enc, lengths, ll.LL_PREC_EXACT, frame_looping=True)
    assert h3 == h1


def test_exact_refuses_otf():
    c = synth.CONFIGS["fc-rnnt"]
    spec = c["spec"]
    w = synth.make_weights(spec, 7)
    enc, lengths = synth.make_inputs(8, 2, 20, spec.enc_dim, 5, 20)
    with pytest.raises(ll.LLError) as e:
        with ll.options(projections=1):
            _decode(spec, gpu_model(spec, w, "bf16"), enc, lengths, ll.LL_PREC_EXACT)
    assert e.value.status == ll.LL_ERR_UNSUPPORTED
