"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle.

Tolerances (north_star): joint logits within 2e-3 absolute in bf16 and 1e-5
in fp32; token / timestamp / length sequences bit-exact except at decisions
whose float64 top-2 gap is below 1e-3 (teacher-forced verifier, oracle/verify.py).
"""
import numpy as np
import pytest
import torch

import synth
from gpu_helpers import TOL, gpu_decode, gpu_model, oracle_hyps, verify_all
from oracle import Transducer
from paper_2406_06220_b200 import ll
from paper_2406_06220_b200.decoder import LabelLoopingDecoder, debug_joint

pytestmark = pytest.mark.gpu


def _joint_case(spec, seed, n, dtype):
    w = synth.make_weights(spec, seed, blank_bias=0.3)
    rng = np.random.default_rng(seed)
    enc = synth.bf16_round(rng.normal(0, 1, size=(n, spec.enc_dim)))
    g = rng.normal(0, 0.5, size=(n, spec.joint_dim)).astype(np.float32)
    model = gpu_model(spec, w, dtype)
    logits, am, dam = debug_joint(model, torch.from_numpy(enc).to("cuda", model.tdtype),
                                  torch.from_numpy(g).cuda())
    o = Transducer.from_spec(spec, w)
    f = o.enc_proj(enc)
    ref, dref = [], []
    for i in range(n):
        l, dl = o.joint(f[i], g[i].astype(np.float64))
        ref.append(l)
        dref.append(dl)
    ref = np.array(ref)
    full = np.concatenate([ref, np.array(dref)], 1) if spec.is_tdt else ref
    return logits.cpu().numpy().astype(np.float64), am.cpu().numpy(), \
        None if dam is None else dam.cpu().numpy(), full, ref, (np.array(dref) if spec.is_tdt else None)


@pytest.mark.parametrize("dtype,tol", [("bf16", 2e-3), ("f32", 1e-5)])
@pytest.mark.parametrize("shape", ["fc", "tiny"])
@pytest.mark.parametrize("tdt", [False, True])
def test_debug_joint_logits(dtype, tol, shape, tdt):
    """Joint (+ encoder projection) logits vs float64 (north_star tolerances);
    argmax equal except at float64 near-ties.  n spans several R=16 chunks and a
    ragged tail."""
    durs = (0, 1, 2, 3, 4) if tdt else None
    if shape == "fc":
        spec = synth.ModelSpec(1025, 512, 640, 640, "lstm", 1, durs, 0, 10)
    else:
        spec = synth.ModelSpec(9, 16, 16, 16, "stateless", 1, durs, 0, 3)
    logits, am, dam, full, ref, dref = _joint_case(spec, 11, 45, dtype)
    err = np.abs(logits - full).max()
    assert err < tol, err
    for i in range(len(am)):
        gap = ref[i].max() - ref[i][am[i]]
        assert am[i] == int(np.argmax(ref[i])) or gap < TOL
        if tdt:
            gap = dref[i].max() - dref[i][dam[i]]
            assert dam[i] == int(np.argmax(dref[i])) or gap < TOL


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("window", [1, 0])
def test_cat_dog_through_abi(dtype, window):
    """Fig. 2 worked example through ll_decode_rnnt.  With a
    one-frame window (W=1, the paper's inner loop) the device runs exactly the
    golden 4 predictor steps and 8 joint rounds of Alg. 3; with the default
    multi-frame window the hypotheses are identical and the decisions used
    equal the frame-by-frame count."""
    # window 1: one frame per round, both rows in one group, the paper's batched
    # outer loop (Alg. 3 as listed)
    opts = dict(window=1, group_rows=4, schedule=0) if window else {}
    spec, w, enc, lengths, vocab = synth.cat_dog_fixture()
    with ll.options(**opts):
        hyps, dec = gpu_decode(spec, w, enc, lengths, dtype)
    assert [[vocab[y] for y in h[0]] for h in hyps] == [list("CAT"), list("DOG")]
    assert [h[1] for h in hyps] == [[0, 2, 2], [1, 3, 3]]
    st = dec.stats()
    assert st["joint_evals"] == 7 + 7      # one decision per alignment symbol
    if window == 1:                        # one group of both rows, one frame per round
        assert st["window"] == 1 and st["groups"] == 1
        assert st["predictor_steps"] == 4  # label-looping: BOS + longest hypothesis
        assert st["joint_rounds"] == 8     # tests/golden/cat_dog.txt


def test_tdt_forced_through_abi():
    spec, w, enc, lengths, vocab = synth.tdt_forced_fixture()
    hyps, _ = gpu_decode(spec, w, enc, lengths, "bf16")
    assert [vocab[y] for y in hyps[0][0]] == list("DOG")
    assert hyps[0][1] == [0, 1, 3] and hyps[0][2] == [1, 2, 1]


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("tdt", [False, True])
@pytest.mark.parametrize("window", [1, 0])
def test_guard_counter_restarts_after_blank(dtype, tdt, window):
    """Reading A6/A14: after a frame advance inside a multi-frame window the
    label counter restarts, so frame 1 emits m = 3 labels (A,B,C,D @ [0,1,1,1],
    hand-derived; pinned on the oracle in test_oracle.py)."""
    fx = synth.guard_after_blank_tdt_fixture() if tdt else synth.guard_after_blank_fixture()
    spec, w, enc, lengths, vocab = fx
    with ll.options(window=window):
        hyps, _ = gpu_decode(spec, w, enc, lengths, dtype)
    assert [vocab[y] for y in hyps[0][0]] == list("ABCD")
    assert hyps[0][1] == [0, 1, 1, 1]
    if tdt:
        assert hyps[0][2] == [0, 0, 0, 0]


@pytest.mark.parametrize("kind", ["stateless", "lstm"])
def test_tiny_low_blank_bias_sweep(kind):
    """Random tiny models with blank biases in [-0.5, 2] (many labels per frame,
    blanks between them: the guard after a frame advance is exercised), 60
    seeds x 2 rows, windows of 8 frames; every row teacher-forced in float64."""
    base = synth.CONFIGS["tiny"]["spec"]
    sp = synth.ModelSpec(base.num_tokens, base.enc_dim, base.pred_dim, base.joint_dim, kind, 1, None,
                         base.blank_id, base.max_symbols)
    decs = 0
    for seed in range(60):
        bb = float(np.random.default_rng(seed).uniform(-0.5, 2.0))
        w = synth.make_weights(sp, 5000 + seed, blank_bias=bb)
        enc, lengths = synth.make_inputs(7000 + seed, 2, 30, sp.enc_dim, 5, 30)
        hyps, _ = gpu_decode(sp, w, enc, lengths, "f32")
        decs += verify_all(sp, w, enc, lengths, hyps)[1]
    assert decs > 1000


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("cfg", ["tiny", "tiny-tdt"])
def test_tiny_random_family(dtype, cfg):
    """BASELINE configs (1) and (3)-tiny on many seeds (random family, guard and
    zero-duration paths exercised), teacher-forced against float64."""
    c = synth.CONFIGS[cfg]
    spec = c["spec"]
    ties = decs = 0
    for seed in range(12):
        for kind, ctx in [("stateless", 1), ("stateless", 2), ("lstm", 1)]:
            sp = synth.ModelSpec(spec.num_tokens, spec.enc_dim, spec.pred_dim, spec.joint_dim, kind, ctx,
                                 spec.durations, spec.blank_id, spec.max_symbols)
            w = synth.make_weights(sp, 1000 + seed, blank_bias=0.5)
            enc, lengths = synth.make_inputs(2000 + seed, c["B"], c["T_max"], sp.enc_dim, c["len_lo"], c["len_hi"])
            hyps, _ = gpu_decode(sp, w, enc, lengths, dtype)
            t, d = verify_all(sp, w, enc, lengths, hyps)
            ties += t
            decs += d
            if dtype == "f32":
                ref = oracle_hyps(sp, w, enc, lengths)
                mism = sum(1 for b in ref if tuple(map(list, ref[b])) != tuple(map(list, hyps[b])))
                assert mism == 0 or ties > 0
    assert decs > 1000


@pytest.mark.parametrize("kind", ["lstm", "stateless"])
def test_fc_rnnt_planted_full_batch(kind):
    """Config (2) at full size (B=32, T in 225..275, V+1=1025, H=P=640, D_e=512),
    planted family: the decode equals the planted alignment exactly (closed
    form), and 4 sampled rows pass the float64 teacher-forced verifier."""
    c = synth.CONFIGS["fc-rnnt"]
    spec = c["spec"]
    if kind == "stateless":
        spec = synth.ModelSpec(1025, 512, 640, 640, "stateless", 2, None, 0, 10)
    w, enc, lengths, planted = synth.make_planted_rnnt(spec, 5, c["B"], c["T_max"], c["len_lo"], c["len_hi"])
    hyps, dec = gpu_decode(spec, w, enc, lengths, "bf16")
    for b in range(c["B"]):
        assert (hyps[b][0], hyps[b][1]) == (planted[b][0], planted[b][1]), b
    verify_all(spec, w, enc, lengths, hyps, rows=[0, 7, 19, 31])
    st = dec.stats()
    assert st["labels"] == sum(len(p[0]) for p in planted)


def test_fc_tdt_planted_full_batch():
    c = synth.CONFIGS["fc-tdt"]
    spec = c["spec"]
    w, enc, lengths, planted = synth.make_planted_tdt(spec, 6, c["B"], c["T_max"], c["len_lo"], c["len_hi"])
    hyps, _ = gpu_decode(spec, w, enc, lengths, "bf16")
    for b in range(c["B"]):
        assert hyps[b] == planted[b], b
    verify_all(spec, w, enc, lengths, hyps, rows=[0, 13, 31])


@pytest.mark.parametrize("tdt", [False, True])
def test_fc_random_family_full_batch(tdt):
    """Config (2)/(3) shapes, random family (near-ties present): all 32 rows pass
    the teacher-forced float64 verifier with the 1e-3 near-tie tolerance."""
    c = synth.CONFIGS["fc-tdt" if tdt else "fc-rnnt"]
    spec = c["spec"]
    w = synth.make_weights(spec, 21, blank_bias=synth.random_family_blank_bias(spec))
    enc, lengths = synth.make_inputs(22, c["B"], c["T_max"], spec.enc_dim, c["len_lo"], c["len_hi"])
    hyps, _ = gpu_decode(spec, w, enc, lengths, "bf16")
    ties, decs = verify_all(spec, w, enc, lengths, hyps)
    labels = sum(len(h[0]) for h in hyps)
    print(f"fc random family tdt={tdt}: {labels} labels, {decs} decisions, {ties} near-ties")
    assert labels > 32 * 50            # the calibrated bias emits labels (not an all-blank run)
    assert decs > 32 * (60 if tdt else 200)
    assert ties <= decs * 0.02


def test_stateless_large_batch_config4_sampled():
    """Config (4): B=512, lengths 50..1500, D_e=1024, stateless context 2, in the
    launch configuration bench.py uses; sampled rows verified in float64 and
    properties (lengths, monotone timestamps, <= m per frame) on all rows."""
    c = synth.CONFIGS["stateless-b512"]
    spec = c["spec"]
    w, enc, lengths, planted = synth.make_planted_rnnt(spec, 9, c["B"], c["T_max"], c["len_lo"], c["len_hi"])
    hyps, _ = gpu_decode(spec, w, enc, lengths, "bf16")
    for b in range(c["B"]):
        assert (hyps[b][0], hyps[b][1]) == (planted[b][0], planted[b][1]), b
    verify_all(spec, w, enc, lengths, hyps, rows=[3, 200, 511])


def test_edge_cases():
    """Empty batch, zero lengths, length > T_max (reported by ll_sync), NaN
    padding never read (A17), capacity overflow (bounded writes, true count)."""
    spec = synth.ModelSpec(9, 16, 16, 16, "lstm", 1, None, 0, 3)
    w = synth.make_weights(spec, 3, blank_bias=-2.0)
    model = gpu_model(spec, w)
    # B = 0
    dec = LabelLoopingDecoder(model, 3, 4, 10)
    enc = torch.zeros(0, 10, 16, dtype=torch.bfloat16, device="cuda")
    out = dec.decode(enc, torch.zeros(0, dtype=torch.int32, device="cuda"))
    assert out.lengths.numel() == 0
    # zero lengths + NaN padding
    encn, lengths = synth.make_inputs(4, 4, 10, 16, 0, 10, pad_value=float("nan"))
    lengths[:2] = 0
    hyps, _ = gpu_decode(spec, w, encn, lengths)
    assert hyps[0][0] == [] and hyps[1][0] == []
    verify_all(spec, w, np.nan_to_num(encn), lengths, hyps)
    # length > T_max -> LL_ERR_INVALID_ARGUMENT from ll_sync, row decodes empty
    enc_d = torch.from_numpy(np.nan_to_num(encn)).to("cuda", torch.bfloat16)
    bad = torch.tensor([3, 11, 5, 2], dtype=torch.int32, device="cuda")
    assert dec.launch(enc_d, bad) == ll.LL_OK
    assert dec.sync() == ll.LL_ERR_INVALID_ARGUMENT
    assert dec.lengths_out[1].item() == 0
    # capacity overflow: never-blank model emits L*m labels, cap smaller
    w2 = synth.make_weights(spec, 3, blank_bias=-1e4)
    m2 = gpu_model(spec, w2)
    dec2 = LabelLoopingDecoder(m2, 3, 4, 10, cap=7)
    enc2, len2 = synth.make_inputs(5, 4, 10, 16, 10, 10)
    dec2.tokens.fill_(-7)
    assert dec2.launch(torch.from_numpy(enc2).to("cuda", torch.bfloat16), torch.from_numpy(len2).cuda()) == 0
    assert dec2.sync() == ll.LL_ERR_CAPACITY
    assert dec2.lengths_out.cpu().tolist() == [30, 30, 30, 30]
    assert (dec2.tokens[:, :7] >= 1).all()


def test_determinism_and_batch_composition():
    """SPEC.md:354/:356/:395: repeat runs are bitwise identical; an utterance
    decodes identically alone and inside a permuted batch."""
    c = synth.CONFIGS["fc-rnnt"]
    spec = c["spec"]
    w = synth.make_weights(spec, 31, blank_bias=synth.random_family_blank_bias(spec))
    enc, lengths = synth.make_inputs(32, 20, 120, spec.enc_dim, 60, 120)
    model = gpu_model(spec, w)
    h1, _ = gpu_decode(spec, w, enc, lengths, model=model)
    h2, _ = gpu_decode(spec, w, enc, lengths, model=model)
    assert h1 == h2
    perm = np.random.default_rng(0).permutation(20)
    hp, _ = gpu_decode(spec, w, enc[perm], lengths[perm], model=model)
    for i, b in enumerate(perm):
        assert hp[i] == h1[b]
    for b in [0, 5, 19]:
        ha, _ = gpu_decode(spec, w, enc[b:b + 1], lengths[b:b + 1], model=model)
        assert ha[0] == h1[b]


# ------------------------------------------------------------------ frame-looping
# The Alg. 2 baseline (ll_decode_rnnt_frame_looping) on the same kernels: the
# hypotheses must equal label-looping's (both reach Alg. 1's greedy result) and
# the batched joint-call count must equal the oracle's Alg. 2 count.

@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_frame_looping_cat_dog(dtype):
    spec, w, enc, lengths, vocab = synth.cat_dog_fixture()
    model = gpu_model(spec, w, dtype)
    dec = LabelLoopingDecoder(model, spec.max_symbols, 2, enc.shape[1], frame_looping=True)
    with ll.options(group_rows=2):                      # both utterances in one batch
        out = dec.decode(torch.from_numpy(enc).to("cuda", model.tdtype), torch.from_numpy(lengths).cuda())
    hyps = out.hypotheses()
    assert [[vocab[y] for y in h[0]] for h in hyps] == [list("CAT"), list("DOG")]
    assert [h[1] for h in hyps] == [[0, 2, 2], [1, 3, 3]]
    from oracle import decode_frame_looping
    _, cnt = decode_frame_looping(Transducer.from_spec(spec, w), enc, lengths, spec.max_symbols)
    st = dec.stats()
    assert st["joint_rounds"] == cnt["joint_calls"]
    assert st["joint_evals"] == 14


@pytest.mark.parametrize("kind", ["stateless", "lstm"])
def test_frame_looping_equals_label_looping_tiny(kind):
    """Random tiny models (guard exercised): frame-looping == label-looping on
    the GPU, and every row passes the float64 verifier."""
    base = synth.CONFIGS["tiny"]["spec"]
    sp = synth.ModelSpec(base.num_tokens, base.enc_dim, base.pred_dim, base.joint_dim, kind, 1, None,
                         base.blank_id, base.max_symbols)
    for seed in range(20):
        bb = float(np.random.default_rng(seed).uniform(-0.5, 2.0))
        w = synth.make_weights(sp, 5000 + seed, blank_bias=bb)
        enc, lengths = synth.make_inputs(7000 + seed, 4, 30, sp.enc_dim, 0, 30)
        model = gpu_model(sp, w, "f32")
        ref, _ = gpu_decode(sp, w, enc, lengths, "f32", model=model)
        dec = LabelLoopingDecoder(model, sp.max_symbols, 4, 30, frame_looping=True)
        hyps = dec.decode(torch.from_numpy(enc).to("cuda", model.tdtype), torch.from_numpy(lengths).cuda()).hypotheses()
        assert hyps == ref, seed
        verify_all(sp, w, enc, lengths, hyps)


def test_frame_looping_fc_planted():
    """Config (2) at full size through the frame-looping baseline: equal to the
    planted alignment (the same closed form label-looping meets)."""
    c = synth.CONFIGS["fc-rnnt"]
    spec = c["spec"]
    w, enc, lengths, planted = synth.make_planted_rnnt(spec, 5, c["B"], c["T_max"], c["len_lo"], c["len_hi"])
    model = gpu_model(spec, w)
    dec = LabelLoopingDecoder(model, spec.max_symbols, c["B"], c["T_max"], frame_looping=True)
    hyps = dec.decode(torch.from_numpy(enc).to("cuda", torch.bfloat16), torch.from_numpy(lengths).cuda()).hypotheses()
    for b in range(c["B"]):
        assert (hyps[b][0], hyps[b][1]) == (planted[b][0], planted[b][1]), b


# ------------------------------------------------------------------ ll_prepare
def test_prepare_tables_reuse_and_invalidate():
    """ll_prepare builds the weight-only tables once: decodes after it equal
    decodes without it (also for a smaller batch on the same workspace), and a
    decode with OTHER weights on the prepared workspace rebuilds its tables."""
    c = synth.CONFIGS["fc-rnnt"]
    spec = c["spec"]
    wa, enc, lengths, planted = synth.make_planted_rnnt(spec, 5, 12, 120, 60, 120)
    wb = synth.make_weights(spec, 77, blank_bias=3.0)
    ma, mb = gpu_model(spec, wa), gpu_model(spec, wb)
    ref_b, _ = gpu_decode(spec, wb, enc, lengths, model=mb)
    dec = LabelLoopingDecoder(ma, spec.max_symbols, 12, 120)
    dec.prepare()
    e = torch.from_numpy(enc).to("cuda", torch.bfloat16)
    l = torch.from_numpy(lengths).cuda()
    for _ in range(2):
        h = dec.decode(e, l).hypotheses()
        assert [(x[0], x[1]) for x in h] == [(p[0], p[1]) for p in planted]
    h5 = dec.decode(e[:5], l[:5]).hypotheses()           # smaller batch, same prepared tables
    assert [(x[0], x[1]) for x in h5] == [(p[0], p[1]) for p in planted[:5]]
    dec.model = mb                                          # other weights, same workspace
    hb = dec.decode(e, l).hypotheses()
    assert hb == ref_b
    dec.model = ma                                          # back: tables were rebuilt for mb
    h = dec.decode(e, l).hypotheses()
    assert [(x[0], x[1]) for x in h] == [(p[0], p[1]) for p in planted]


@pytest.mark.parametrize("cfg", ["fc-rnnt", "fc-tdt"])
def test_schedules_identical(cfg):
    """The per-row tick schedule (default) and the paper's batched outer loop
    (ll_options.schedule = 0) are exact reorderings of Alg. 3: identical hypotheses on a
    random-family FC batch (near-ties included), and identical joint-evaluation
    counts (the algorithmic decisions)."""
    c = synth.CONFIGS[cfg]
    spec = c["spec"]
    w = synth.make_weights(spec, 41, blank_bias=synth.random_family_blank_bias(spec))
    enc, lengths = synth.make_inputs(42, c["B"], c["T_max"], spec.enc_dim, c["len_lo"], c["len_hi"])
    model = gpu_model(spec, w)
    out = {}
    for sched in (0, 1):
        with ll.options(schedule=sched):
            hyps, dec = gpu_decode(spec, w, enc, lengths, model=model)
            out[sched] = (hyps, dec.stats())
    assert out[0][0] == out[1][0]
    assert out[0][1]["joint_evals"] == out[1][1]["joint_evals"]
    assert out[0][1]["labels"] == out[1][1]["labels"]


def test_fc_rnnt_4x_subsampling_planted():
    """4x-subsampling variant of config 2 (40 ms frames, T ~ 500; PAPER.md
    Table 4): decode == planted alignment at full size, sampled rows verified."""
    c = synth.CONFIGS["fc-rnnt-4x"]
    spec = c["spec"]
    w, enc, lengths, planted = synth.make_planted_rnnt(spec, 8, c["B"], c["T_max"], c["len_lo"], c["len_hi"],
                                                       rho=c["rho"])
    hyps, _ = gpu_decode(spec, w, enc, lengths, "bf16")
    for b in range(c["B"]):
        assert (hyps[b][0], hyps[b][1]) == (planted[b][0], planted[b][1]), b
    verify_all(spec, w, enc, lengths, hyps, rows=[0, 31])


def test_sweep_chunks_pack_unpack():
    """Config-5 plumbing on one GPU: utterances of a LibriSpeech-like sweep,
    LPT-sharded and decoded longest-first in two launches; the device-packed
    ragged buffer unpacks to exactly the per-utterance planted alignments."""
    from paper_2406_06220_b200 import shard
    c = synth.SWEEPS["sweep-tdt"]
    spec = c["spec"]
    w, codes = synth.planted_weights(spec, 1000)
    L_all = synth.sweep_lengths(c["length_seed"], 96)
    ids = shard.rank_shard(L_all, 2, 1, 16)           # rank 1 of 2
    model = gpu_model(spec, w)
    outs, planted = [], {}
    for c0 in range(0, len(ids), 24):
        cid = ids[c0:c0 + 24]
        T = int(L_all[cid].max())
        enc = np.zeros((len(cid), T, spec.enc_dim), dtype=np.float32)
        for i, u in enumerate(cid):
            e, pl = synth.planted_utterance(spec, codes, c["length_seed"], int(u), int(L_all[u]))
            enc[i, :e.shape[0]] = e
            planted[int(u)] = pl
        dec = LabelLoopingDecoder(model, spec.max_symbols, len(cid), T)
        out = dec.decode(torch.from_numpy(enc).to("cuda", torch.bfloat16),
                         torch.from_numpy(L_all[cid].astype(np.int32)).cuda())
        outs.append((torch.from_numpy(cid).cuda(), out))
    buf = shard.pack_hypotheses([i for i, _ in outs], [o.lengths for _, o in outs], [o.tokens for _, o in outs],
                                [o.timestamps for _, o in outs], [o.durations for _, o in outs])
    got = shard.unpack_hypotheses(buf.cpu().numpy(), True)
    assert sorted(got) == sorted(int(u) for u in ids)
    for u in ids:
        assert got[int(u)] == tuple(planted[int(u)]), int(u)
    # the native exchange (ll_gather_ragged, world size 1): one record per
    # launch, byte-identical to the torch-built record, parsing to the same map
    g = shard.NcclGather()
    try:
        recs = [g.gather(i.to(torch.int32), o.lengths, o.tokens, o.timestamps, o.durations) for i, o in outs]
    finally:
        g.close()
    for (i, o), r in zip(outs, recs):
        assert torch.equal(r, shard.pack_hypotheses(i, o.lengths, o.tokens, o.timestamps, o.durations))
    assert shard.unpack_records(torch.cat(recs).cpu().numpy(), True) == got


@pytest.mark.parametrize("B,cap,tdt", [(0, 5, False), (1, 1, True), (37, 7, False), (1500, 9, True), (2100, 3, False)])
def test_native_gather_records(B, cap, tdt):
    """ll_gather_ragged's packing kernels on ragged rows: lengths beyond the
    capacity are clamped, empty rows and B = 0 give well-formed records, more
    than 1024 rows exercise the multi-pass scan; the result equals the
    torch-built record element by element.  A root buffer that is too small is
    reported (LL_ERR_CAPACITY with the size needed) and the retry succeeds."""
    from paper_2406_06220_b200 import shard
    gen = torch.Generator().manual_seed(B * 31 + cap)
    ids = torch.randperm(max(B, 1) * 3, generator=gen)[:B].to(torch.int32).cuda()
    lens = torch.randint(0, cap + 4, (B,), generator=gen, dtype=torch.int32).cuda()
    tok = torch.randint(0, 1 << 20, (B, cap), generator=gen, dtype=torch.int32).cuda()
    ts = torch.randint(0, 1 << 20, (B, cap), generator=gen, dtype=torch.int32).cuda()
    du = torch.randint(0, 5, (B, cap), generator=gen, dtype=torch.int32).cuda() if tdt else None
    g = shard.NcclGather()
    try:
        g._root = torch.empty(1, dtype=torch.int32, device="cuda")   # force the capacity path
        got = g.gather(ids, lens, tok, ts, du)
        again = g.gather(ids, lens, tok, ts, du)
    finally:
        g.close()
    ref = shard.pack_hypotheses(ids, lens, tok, ts, du)
    assert torch.equal(got, ref) and torch.equal(again, ref)
    if B == 0:
        assert got.tolist() == [0]


# ------------------------------------------------------------------ production-instantiation probe
# The logit tolerance and the predictor output checked on the PRODUCTION
# FastConformer kernel (decode_kernel<bf16, *, KREG, 640, 640, 16, ticks, family>
# with its probe hook, ll.h ll_options): every joint row the kernel evaluated
# (speculative window frames included) and g after every predictor step, against
# float64 along the kernel's own label history (teacher forcing).
G_TOL = 2e-3   # bf16 h through the recurrence and W_pred


def _oracle_g_sequence(o, tokens):
    """g after consuming SOS, tokens[0], ..., tokens[n-1], for n = 0..len(tokens)."""
    st = o.pred_init()
    dec, st = o.pred_step(st, o.blank)
    gs = [o.pred_proj(dec)]
    for y in tokens:
        dec, st = o.pred_step(st, int(y))
        gs.append(o.pred_proj(dec))
    return gs


@pytest.mark.parametrize("kind,tdt", [("lstm", False), ("lstm", True), ("stateless", False)])
def test_production_kernel_logits_and_g(kind, tdt):
    from paper_2406_06220_b200.decoder import probe_decode
    durs = (0, 1, 2, 3, 4) if tdt else None
    De = 1024 if kind == "stateless" else 512
    spec = synth.ModelSpec(1025, De, 640, 640, kind, 2 if kind == "stateless" else 1, durs, 0, 10)
    w = synth.make_weights(spec, 61, blank_bias=synth.random_family_blank_bias(spec))
    B, T = 16, 80
    enc, lengths = synth.make_inputs(62, B, T, spec.enc_dim, 40, T)
    model = gpu_model(spec, w)
    dec = LabelLoopingDecoder(model, spec.max_symbols, B, T)
    out, jrows, grows = probe_decode(dec, torch.from_numpy(enc).to("cuda", torch.bfloat16),
                                     torch.from_numpy(lengths).cuda())
    hyps = out.hypotheses()
    verify_all(spec, w, enc, lengths, hyps)
    o = Transducer.from_spec(spec, w)
    gseq = {b: _oracle_g_sequence(o, hyps[b][0]) for b in range(B)}
    fs = {b: o.enc_proj(enc[b][:int(lengths[b])]) for b in range(B)}
    st = dec.stats()
    assert len(jrows) == st["joint_rows_computed"] and len(grows) == st["predictor_rows"]
    assert len(grows) > 10 * B          # labels were emitted: the recurrence is exercised
    lerr = 0.0
    for b, t, n, lg in jrows:
        assert 0 <= b < B and 0 <= t < lengths[b] and 0 <= n <= len(hyps[b][0])
        l, dl = o.joint(fs[b][t], gseq[b][n])
        ref = np.concatenate([l, dl]) if tdt else l
        lerr = max(lerr, float(np.abs(lg.astype(np.float64) - ref).max()))
    gerr = 0.0
    for b, n, g in grows:
        gerr = max(gerr, float(np.abs(g.astype(np.float64) - gseq[b][n]).max()))
    print(f"{kind} tdt={tdt}: {len(jrows)} joint rows max |logit err| {lerr:.3g}; "
          f"{len(grows)} g rows max |g err| {gerr:.3g}")
    assert lerr < 2e-3, lerr
    assert gerr < G_TOL, gerr


def test_group_start_h_exchange_race_regression():
    """Regression (round 2): a CTA used to zero its h buffer when it took the
    next group while faster CTAs of its cluster could already have st.async'ed
    that group's first h' slices into it -> wrong g on the first predictor step
    of a group.  Many short groups (2 rows each, short utterances) make group
    starts frequent, and the probe's stall hook delays the odd ranks of each
    cluster at every group start (the race window wide open); the production
    kernel's g after EVERY predictor step must match float64."""
    from paper_2406_06220_b200.decoder import probe_decode
    spec = synth.ModelSpec(1025, 512, 640, 640, "lstm", 1, None, 0, 10)
    w = synth.make_weights(spec, 71, blank_bias=synth.random_family_blank_bias(spec))
    B, T = 40, 24
    enc, lengths = synth.make_inputs(72, B, T, spec.enc_dim, 6, T)
    model = gpu_model(spec, w)
    o = Transducer.from_spec(spec, w)
    for _ in range(3):
        dec = LabelLoopingDecoder(model, spec.max_symbols, B, T)
        out, jrows, grows = probe_decode(dec, torch.from_numpy(enc).to("cuda", torch.bfloat16),
                                         torch.from_numpy(lengths).cuda(), regions=4, group_rows=2,
                                         probe_stall=20000)
        hyps = out.hypotheses()
        gseq = {b: _oracle_g_sequence(o, hyps[b][0]) for b in range(B)}
        assert dec.stats()["groups"] == B // 2
        gerr = max(float(np.abs(g.astype(np.float64) - gseq[b][n]).max()) for b, n, g in grows)
        assert gerr < G_TOL, gerr


def test_config4_random_family_full_batch():
    """Config (4) in the launch configuration bench.py times (B=512, lengths
    50..1500, D_e=1024, stateless context 2, throughput mode: many waves of small
    groups) on the RANDOM family (calibrated blank bias: labels, blanks and
    near-ties): all 512 rows pass the teacher-forced float64 verifier."""
    c = synth.CONFIGS["stateless-b512"]
    spec = c["spec"]
    w = synth.make_weights(spec, 71, blank_bias=synth.random_family_blank_bias(spec))
    enc, lengths = synth.make_inputs(72, c["B"], c["T_max"], spec.enc_dim, c["len_lo"], c["len_hi"])
    hyps, dec = gpu_decode(spec, w, enc, lengths, "bf16")
    st = dec.stats()
    # throughput mode: groups of <= 16 rows taken from the work counter in many waves
    assert st["group_rows"] <= 16 and st["groups"] >= c["B"] // 16
    ties, decs = verify_all(spec, w, enc, lengths, hyps)
    print(f"config 4 random family: {decs} decisions, {ties} near-ties, {st['labels']} labels")
    assert st["labels"] > c["B"] * 50
    assert decs > c["B"] * 50


# ------------------------------------------------------------------ greedy scores (N2)
# ll_decode_*_scores: the fused log-sum-exp in the joint epilogue.  The float64
# reference score is the verifier's, accumulated along the GPU's own decisions
# (oracle/verify.py).  Bound per decision: the token (and duration) logit and
# the log-sum-exp each within the north_star logit tolerance, so 2 x tol per
# log-probability (4 x for TDT's two terms), plus fp32 accumulation.
def _scored_decode(spec, w, enc, lengths, dtype):
    model = gpu_model(spec, w, dtype)
    B, T = enc.shape[0], enc.shape[1]
    e = torch.from_numpy(np.ascontiguousarray(enc)).to("cuda", model.tdtype)
    l = torch.from_numpy(np.asarray(lengths, dtype=np.int32)).cuda()
    plain = LabelLoopingDecoder(model, spec.max_symbols, B, T).decode(e, l).hypotheses()
    dec = LabelLoopingDecoder(model, spec.max_symbols, B, T, scores=True)
    out = dec.decode(e, l)
    return plain, out.hypotheses(), out.scores.cpu().numpy().astype(np.float64)


def _check_scores(spec, w, enc, lengths, hyps, scores, tol_logit):
    from oracle.verify import verify_rnnt, verify_tdt
    o = Transducer.from_spec(spec, w)
    checked = 0
    for b in range(len(hyps)):
        L = int(lengths[b])
        h = hyps[b]
        r = (verify_tdt(o, enc[b], L, spec.max_symbols, h[0], h[1], h[2], all_paths=True) if spec.is_tdt
             else verify_rnnt(o, enc[b], L, spec.max_symbols, h[0], h[1]))
        assert r.ok, r.message
        # TDT: blank durations are not in the outputs, so the kernel's decision
        # path is one of the acceptable paths (near-tie durations); its score
        # must match that path's float64 score
        cands = r.path_scores if spec.is_tdt else [r.score]
        bound = (r.decisions + 2) * (4 if spec.is_tdt else 2) * tol_logit + 1e-6 * abs(r.score) + 1e-5
        err = min(abs(scores[b] - c_) for c_ in cands)
        assert err <= bound, (b, scores[b], cands, bound)
        checked += 1
    return checked


@pytest.mark.parametrize("dtype,tol", [("bf16", 2e-3), ("f32", 1e-5)])
@pytest.mark.parametrize("cfg", ["tiny", "tiny-tdt"])
def test_scores_tiny_random_family(dtype, tol, cfg):
    c = synth.CONFIGS[cfg]
    spec = c["spec"]
    checked = 0
    for seed in range(6):
        for kind, ctx in [("stateless", 2), ("lstm", 1)]:
            sp = synth.ModelSpec(spec.num_tokens, spec.enc_dim, spec.pred_dim, spec.joint_dim, kind, ctx,
                                 spec.durations, spec.blank_id, spec.max_symbols)
            w = synth.make_weights(sp, 1300 + seed, blank_bias=0.5)
            enc, lengths = synth.make_inputs(2300 + seed, c["B"], c["T_max"], sp.enc_dim, c["len_lo"], c["len_hi"])
            plain, hyps, scores = _scored_decode(sp, w, enc, lengths, dtype)
            assert hyps == plain            # scores do not change the hypotheses
            checked += _check_scores(sp, w, enc, lengths, hyps, scores, tol)
    assert checked >= 30


@pytest.mark.parametrize("tdt", [False, True])
def test_scores_fc_random_family(tdt):
    """Config (2)/(3) shapes (the FC score instantiations), random family."""
    c = synth.CONFIGS["fc-tdt" if tdt else "fc-rnnt"]
    spec = c["spec"]
    w = synth.make_weights(spec, 81, blank_bias=synth.random_family_blank_bias(spec))
    enc, lengths = synth.make_inputs(82, 16, 120, spec.enc_dim, 60, 120)
    plain, hyps, scores = _scored_decode(spec, w, enc, lengths, "bf16")
    assert hyps == plain
    assert _check_scores(spec, w, enc, lengths, hyps, scores, 2e-3) >= 8


def test_scores_cat_dog_closed_form():
    """Fig. 2 table model: 7 decisions per utterance, each with logit 10 on the
    chosen symbol and 0 on the other six: score = 7 (10 - log(e^10 + 6))."""
    spec, w, enc, lengths, vocab = synth.cat_dog_fixture()
    for dtype in ("bf16", "f32"):
        _, hyps, scores = _scored_decode(spec, w, enc, lengths, dtype)
        expect = 7 * (10.0 - np.log(np.exp(10.0) + 6.0))
        assert np.abs(scores - expect).max() < 1e-5, (scores, expect)


@pytest.mark.parametrize("cfg", ["tiny", "tiny-tdt"])
@pytest.mark.parametrize("layers", [2, 3])
def test_multilayer_lstm_f32(cfg, layers):
    """N4 ("more layers"): an L-layer LSTM predictor (fp32 weights,
    generic kernel) on many seeds, every row teacher-forced against the float64
    L-layer oracle, and equal to the oracle decode where no near-tie occurred."""
    c = synth.CONFIGS[cfg]
    spec = c["spec"]
    ties = decs = 0
    for seed in range(8):
        sp = synth.ModelSpec(spec.num_tokens, spec.enc_dim, spec.pred_dim, spec.joint_dim, "lstm", 1,
                             spec.durations, spec.blank_id, spec.max_symbols, num_layers=layers)
        w = synth.make_weights(sp, 3000 + seed, blank_bias=0.5)
        enc, lengths = synth.make_inputs(4000 + seed, c["B"], c["T_max"], sp.enc_dim, c["len_lo"], c["len_hi"])
        hyps, _ = gpu_decode(sp, w, enc, lengths, "f32")
        t, d = verify_all(sp, w, enc, lengths, hyps)
        ties += t
        decs += d
        ref = oracle_hyps(sp, w, enc, lengths)
        mism = sum(1 for b in ref if tuple(map(list, ref[b])) != tuple(map(list, hyps[b])))
        assert mism == 0 or ties > 0
    assert decs > 300


@pytest.mark.parametrize("cfg,B", [("fc-rnnt", 32), ("fc-rnnt", 30), ("fc-rnnt", 29), ("fc-tdt", 32),
                                   ("fc-tdt", 31), ("fc-rnnt", 64), ("fc-tdt", 45), ("tiny", 40),
                                   ("tiny-tdt", 37)])
def test_group_plan_equals_equal_groups(cfg, B):
    """Length-sorted unequal groups (ll_options.group_plan, default on for
    one-wave FC decodes, RNN-T and TDT) and length-ranked groups (every other
    decode with more than one group, any kernel): hypotheses identical to
    equal groups of consecutive utterances (utterances are independent,
    SPEC.md:354), every
    output length written (buffers pre-filled with garbage), a zero-length
    utterance included; every row verified against float64."""
    c = synth.CONFIGS[cfg]
    spec = c["spec"]
    fam = synth.random_family_blank_bias(spec) if spec.joint_dim >= 70 else 0.5
    w = synth.make_weights(spec, 91 + B, blank_bias=fam)
    enc, lengths = synth.make_inputs(92 + B, B, c["T_max"], spec.enc_dim, c["len_lo"], c["len_hi"])
    lengths[B // 2] = 0
    model = gpu_model(spec, w)
    out = {}
    for plan in (0, -1):
        dec = LabelLoopingDecoder(model, spec.max_symbols, B, c["T_max"])
        dec.lengths_out.fill_(-7)
        dec.tokens.fill_(-7)
        with ll.options(group_plan=plan):
            o = dec.decode(torch.from_numpy(enc).to("cuda", torch.bfloat16), torch.from_numpy(lengths).cuda())
        assert int(o.lengths.min()) >= 0
        out[plan] = (o.hypotheses(), dec.stats())
    assert out[0][0] == out[-1][0]
    assert out[-1][0][B // 2][0] == []
    assert out[0][1]["joint_evals"] == out[-1][1]["joint_evals"]
    verify_all(spec, w, enc, lengths, out[-1][0])


def test_stats_count_kernel_launches():
    """ll_stats [12]: the kernels a decode call launched, counted by the library
    (bench.py's gpu_launches): with the model tables prepared, one-wave B = 32
    runs the projection GEMM + the decode kernel; B = 64 adds the length ranking;
    on the fly, the decode kernel alone; an unprepared LSTM decode also builds
    its tables (gate permutation, E' GEMM, packed weights)."""
    c = synth.CONFIGS["fc-rnnt"]
    spec = c["spec"]
    w = synth.make_weights(spec, 5, blank_bias=synth.random_family_blank_bias(spec))
    model = gpu_model(spec, w)
    for B, want in ((32, 2), (64, 3)):
        enc, lengths = synth.make_inputs(6, B, 60, spec.enc_dim, 20, 60)
        dec = LabelLoopingDecoder(model, spec.max_symbols, B, 60)
        dec.prepare()
        dec.decode(torch.from_numpy(enc).to("cuda", torch.bfloat16), torch.from_numpy(lengths).cuda())
        assert dec.stats()["launches"] == want, (B, dec.stats())
    enc, lengths = synth.make_inputs(6, 32, 60, spec.enc_dim, 20, 60)
    dec = LabelLoopingDecoder(model, spec.max_symbols, 32, 60)
    dec.decode(torch.from_numpy(enc).to("cuda", torch.bfloat16), torch.from_numpy(lengths).cuda())
    assert dec.stats()["launches"] == 5, dec.stats()
    dec.prepare()
    with ll.options(projections=1):
        dec.decode(torch.from_numpy(enc).to("cuda", torch.bfloat16), torch.from_numpy(lengths).cuda())
    assert dec.stats()["launches"] == 1, dec.stats()
