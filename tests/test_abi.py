"""The C-ABI library loads, exports every symbol include/ll.h declares, and
validates its arguments on the host (nothing enqueued, no GPU needed)."""
import ctypes
import os
import re

import pytest

from paper_2406_06220_b200 import ll
from paper_2406_06220_b200 import build as llbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    llbuild.build()
    return ll.load_library()


def test_exports_every_declared_symbol(lib):
    header = open(os.path.join(ROOT, "include", "ll.h")).read()
    declared = set(re.findall(r"\b(ll_[a-z_]+)\s*\(", header))
    assert declared == set(ll.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name


def test_status_strings_and_version(lib):
    assert ll.ll_status_string(ll.LL_OK) == "LL_OK"
    assert ll.ll_status_string(ll.LL_ERR_CAPACITY) == "LL_ERR_CAPACITY"
    assert ll.ll_status_string(99) == "LL_ERR_UNKNOWN"
    assert "sm_100a" in ll.ll_version()


FAKE = 0x10000  # never dereferenced: validation fails first


def _model(kind=ll.LL_PRED_LSTM, V1=1025, P=640, H=640, De=512, ctx=1, tdt=False):
    pred = ll.ll_predictor(kind, V1, P, ctx, FAKE, FAKE, FAKE, FAKE, FAKE)
    joint = ll.ll_joint(De, P, H, V1, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE,
                        FAKE if tdt else None, FAKE if tdt else None)
    return pred, joint


def _rnnt(pred, joint, **kw):
    a = dict(enc=FAKE, dtype=ll.LL_BF16, prec=ll.LL_PREC_FAST, B=32, T_max=275, lengths=FAKE, blank=0, m=10,
             tok=FAKE, ts=FAKE, lens=FAKE, cap=2750, ws=0x100000, ws_bytes=1 << 40)
    a.update(kw)
    return ll.ll_decode_rnnt(a["enc"], a["dtype"], a["prec"], a["B"], a["T_max"], a["lengths"], pred, joint,
                             a["blank"], a["m"], a["tok"], a["ts"], a["lens"], a["cap"], a["ws"],
                             a["ws_bytes"], None)


def test_workspace_size(lib):
    pred, joint = _model()
    n = ll.ll_workspace_size(32, 275, pred, joint, ll.LL_BF16, ll.LL_PREC_FAST, 0)
    # f [B*T*H] bf16 + E' [V1*4P] f32 + h [2*B*P] bf16 + g [B*H] f32 + header
    assert n >= 32 * 275 * 640 * 2 + 1025 * 2560 * 4 + 2 * 32 * 640 * 2 + 32 * 640 * 4
    assert ll.ll_workspace_size(-1, 275, pred, joint, ll.LL_BF16, ll.LL_PREC_FAST, 0) == 0
    assert ll.ll_workspace_size(32, 275, pred, joint, 7, ll.LL_PREC_FAST, 0) == 0


@pytest.mark.parametrize("kw,status", [
    (dict(B=-1), ll.LL_ERR_INVALID_ARGUMENT),
    (dict(T_max=-1), ll.LL_ERR_INVALID_ARGUMENT),
    (dict(enc=None), ll.LL_ERR_INVALID_ARGUMENT),
    (dict(lengths=None), ll.LL_ERR_INVALID_ARGUMENT),
    (dict(tok=None), ll.LL_ERR_INVALID_ARGUMENT),
    (dict(lens=None), ll.LL_ERR_INVALID_ARGUMENT),
    (dict(blank=1025), ll.LL_ERR_INVALID_ARGUMENT),
    (dict(blank=-1), ll.LL_ERR_INVALID_ARGUMENT),
    (dict(m=0), ll.LL_ERR_INVALID_ARGUMENT),
    (dict(cap=-1), ll.LL_ERR_INVALID_ARGUMENT),
    (dict(ws=None), ll.LL_ERR_INVALID_ARGUMENT),
    (dict(ws=0x100010), ll.LL_ERR_INVALID_ARGUMENT),      # not 256-byte aligned
    (dict(ws_bytes=1024), ll.LL_ERR_WORKSPACE),
    (dict(dtype=5), ll.LL_ERR_INVALID_ARGUMENT),
    (dict(prec=7), ll.LL_ERR_INVALID_ARGUMENT),
])
def test_rnnt_validation(lib, kw, status):
    pred, joint = _model()
    assert _rnnt(pred, joint, **kw) == status


def test_exact_workspace(lib):
    """LL_PREC_EXACT with bf16 inputs (ll.h): the fp32 call's workspace plus fp32
    copies of every weight and of the encoder output; too small -> LL_ERR_WORKSPACE
    before anything is enqueued."""
    pred, joint = _model()
    fast = ll.ll_workspace_size(32, 275, pred, joint, ll.LL_BF16, ll.LL_PREC_FAST, 0)
    exact = ll.ll_workspace_size(32, 275, pred, joint, ll.LL_BF16, ll.LL_PREC_EXACT, 0)
    f32 = ll.ll_workspace_size(32, 275, pred, joint, ll.LL_F32, ll.LL_PREC_FAST, 0)
    V1, P, H, De = 1025, 640, 640, 512
    weights = (H * De + H + H * P + H + V1 * H + V1 + V1 * P + 2 * 4 * P * P + 2 * 4 * P) * 4
    assert exact >= f32 + weights + 32 * 275 * De * 4
    assert exact < f32 + weights + 32 * 275 * De * 4 + 24 * 256 + 512
    assert ll.ll_workspace_size(32, 275, pred, joint, ll.LL_F32, ll.LL_PREC_EXACT, 0) == f32
    assert _rnnt(pred, joint, prec=ll.LL_PREC_EXACT, ws_bytes=fast) == ll.LL_ERR_WORKSPACE
    assert _rnnt(pred, joint, prec=ll.LL_PREC_EXACT, ws_bytes=exact - 1) == ll.LL_ERR_WORKSPACE


def test_model_validation(lib):
    pred, joint = _model()
    pred.hidden = 320                      # predictor / joint dims inconsistent
    assert _rnnt(pred, joint) == ll.LL_ERR_INVALID_ARGUMENT
    pred, joint = _model(H=632, P=640)     # joint dim not a multiple of 16
    assert _rnnt(pred, joint) == ll.LL_ERR_UNSUPPORTED
    pred, joint = _model()
    pred.w_hh = None
    assert _rnnt(pred, joint) == ll.LL_ERR_INVALID_ARGUMENT
    pred, joint = _model(kind=ll.LL_PRED_STATELESS, ctx=0)
    assert _rnnt(pred, joint) == ll.LL_ERR_INVALID_ARGUMENT
    pred, joint = _model(kind=ll.LL_PRED_STATELESS, ctx=5)
    assert _rnnt(pred, joint) == ll.LL_ERR_UNSUPPORTED
    pred, joint = _model(kind=7)
    assert _rnnt(pred, joint) == ll.LL_ERR_INVALID_ARGUMENT


def test_tdt_validation(lib):
    pred, joint = _model(tdt=True)
    call = lambda durs, n, **kw: ll.ll_decode_tdt(FAKE, ll.LL_BF16, ll.LL_PREC_FAST, 32, 275, FAKE, pred, joint,
                                                  0, 10, durs, n, FAKE, FAKE, None, FAKE, 2750, 0x100000,
                                                  kw.get("ws_bytes", 1 << 40), None)
    assert call([0, 1, 2], 0) == ll.LL_ERR_INVALID_ARGUMENT      # empty duration set
    assert call(None, 3) == ll.LL_ERR_INVALID_ARGUMENT
    assert call([0, -1, 2], 3) == ll.LL_ERR_INVALID_ARGUMENT     # negative duration
    assert call(list(range(17)), 17) == ll.LL_ERR_INVALID_ARGUMENT
    joint.w_dur = None
    assert call([0, 1, 2], 3) == ll.LL_ERR_INVALID_ARGUMENT      # TDT needs the duration head
    joint.w_dur = FAKE
    assert call([0, 1, 2], 3, ws_bytes=100) == ll.LL_ERR_WORKSPACE


def test_debug_joint_validation(lib):
    _, joint = _model()
    assert ll.ll_debug_joint(FAKE, FAKE, -1, joint, ll.LL_BF16, 0, 0, None, FAKE, None, 0x100000, 1 << 40,
                             None) == ll.LL_ERR_INVALID_ARGUMENT
    assert ll.ll_debug_joint(FAKE, FAKE, 4, joint, ll.LL_BF16, 0, 0, None, None, None, 0x100000, 1 << 40,
                             None) == ll.LL_ERR_INVALID_ARGUMENT
    assert ll.ll_debug_joint(FAKE, FAKE, 4, joint, ll.LL_BF16, 0, 0, None, FAKE, None, 0x100000, 10,
                             None) == ll.LL_ERR_WORKSPACE


def test_no_oracle_in_product_path():
    """The product package never imports or loads the oracle (test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_2406_06220_b200")
    pat = re.compile(r"^\s*(from\s+oracle|import\s+oracle)|oracle/", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                assert not pat.search(open(os.path.join(dirpath, f)).read()), f


def test_gather_validation(lib):
    """ll_gather_ragged / NCCL helpers: host-side argument checks return before
    any NCCL or CUDA call."""
    F = FAKE
    assert ll.ll_gather_workspace_size(-1, 5, False) == 0
    assert ll.ll_gather_workspace_size(0, 5, False) > 0
    assert ll.ll_gather_workspace_size(100, 5, True) > ll.ll_gather_workspace_size(100, 5, False)
    assert lib.ll_nccl_unique_id(None) == ll.LL_ERR_INVALID_ARGUMENT
    assert ll.ll_nccl_comm_init(0, b"\0" * 128, 0)[0] == ll.LL_ERR_INVALID_ARGUMENT
    assert ll.ll_nccl_comm_init(2, b"\0" * 128, 2)[0] == ll.LL_ERR_INVALID_ARGUMENT
    assert ll.ll_nccl_comm_destroy(None) == ll.LL_OK
    args = dict(comm=F, root=0, B=4, utt_ids=F, lengths=F, tokens=F, timestamps=F, durations=None,
                out_capacity=8, root_buf=F, root_capacity=1000, workspace=F, workspace_bytes=1 << 30, stream=None)
    for bad in [dict(comm=None), dict(B=-1), dict(workspace=None), dict(out_capacity=-1), dict(root_capacity=-1),
                dict(utt_ids=None), dict(lengths=None), dict(tokens=None), dict(timestamps=None)]:
        kw = {**args, **bad}
        assert ll.ll_gather_ragged(*kw.values())[0] == ll.LL_ERR_INVALID_ARGUMENT, bad


def test_options_validation_and_release(lib):
    """ll_set_options: explicit knobs (no environment variables on the
    production path), validated on the host; NULL restores the defaults.
    ll_release of an unknown / NULL workspace is a no-op."""
    assert ll.ll_set_options(None) == ll.LL_OK
    for bad in [dict(window=9), dict(group_rows=33), dict(cluster_size=17), dict(schedule=2),
                dict(spec_prefetch=-2), dict(max_clusters=-1), dict(probe_rows=-1), dict(projections=2),
                dict(projections=-1)]:
        o = ll.default_options()
        for k, v in bad.items():
            setattr(o, k, v)
        assert ll.ll_set_options(o) == ll.LL_ERR_INVALID_ARGUMENT, bad
    with ll.options(window=2, group_rows=4, schedule=0):
        pass
    with ll.options(projections=1):   # on-the-fly projections (Table 3's ablation arm)
        pass
    assert ll.ll_set_options(None) == ll.LL_OK
    assert ll.ll_release(None) == ll.LL_OK
    assert ll.ll_release(0x100000) == ll.LL_OK


def test_no_environment_knobs_in_library():
    """The production library reads no environment variable:
    getenv is not referenced by the C ABI sources."""
    for f in ("ll_api.cu", "ll_gather.cu", "decode.cuh", "common.cuh", "gemm_tc.cuh", "linear.cuh"):
        src = open(os.path.join(ROOT, "paper_2406_06220_b200", "csrc", f)).read()
        assert "getenv" not in src, f
