"""Thin ctypes binding of the C ABI in include/ll.h (argument marshalling only).

Every function here has the name of the C entry point it forwards to and takes
plain integers (device pointers, sizes) and the ctypes structs below; every
step of decoding runs in the library's CUDA kernels.  The library is built
in-tree (`python -m paper_2406_06220_b200.build`); if it is missing or cannot
be loaded, importing the binding raises -- there is no fallback path.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_int32, c_size_t, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LL_LIB_PATH") or os.path.join(HERE, "libll.so")  # override: experiments only

LL_OK, LL_ERR_INVALID_ARGUMENT, LL_ERR_UNSUPPORTED, LL_ERR_WORKSPACE, LL_ERR_CUDA, LL_ERR_CAPACITY = range(6)
LL_BF16, LL_F32 = 0, 1
LL_PREC_FAST, LL_PREC_EXACT = 0, 1
LL_PRED_LSTM, LL_PRED_STATELESS = 0, 1

# Every symbol include/ll.h declares (checked by tests/test_abi.py).
EXPORTED = ["ll_workspace_size", "ll_decode_rnnt", "ll_decode_rnnt_frame_looping", "ll_decode_tdt", "ll_prepare",
            "ll_decode_rnnt_scores", "ll_decode_tdt_scores",
            "ll_sync",
            "ll_status_string",
            "ll_stats", "ll_debug_joint", "ll_set_timing_events", "ll_version", "ll_release", "ll_set_options",
            "ll_nccl_unique_id", "ll_nccl_comm_init", "ll_nccl_comm_destroy", "ll_gather_workspace_size",
            "ll_gather_ragged"]


class ll_predictor(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("num_tokens", c_int32), ("hidden", c_int32), ("context", c_int32),
                ("embedding", c_void_p), ("w_ih", c_void_p), ("w_hh", c_void_p), ("b_ih", c_void_p),
                ("b_hh", c_void_p), ("num_layers", c_int32), ("w_ih_rest", c_void_p), ("w_hh_rest", c_void_p),
                ("b_ih_rest", c_void_p), ("b_hh_rest", c_void_p)]


class ll_joint(ctypes.Structure):
    _fields_ = [("enc_dim", c_int32), ("pred_dim", c_int32), ("joint_dim", c_int32),
                ("num_outputs", c_int32), ("w_enc", c_void_p), ("b_enc", c_void_p), ("w_pred", c_void_p),
                ("b_pred", c_void_p), ("w_out", c_void_p), ("b_out", c_void_p), ("w_dur", c_void_p),
                ("b_dur", c_void_p)]


class ll_options(ctypes.Structure):
    _fields_ = [("cluster_size", c_int32), ("group_rows", c_int32), ("window", c_int32),
                ("max_clusters", c_int32), ("schedule", c_int32), ("spec_prefetch", c_int32),
                ("gemm_mma_sync", c_int32), ("timeline", c_void_p), ("trace", c_void_p),
                ("probe_logits", c_void_p), ("probe_lmeta", c_void_p), ("probe_g", c_void_p),
                ("probe_gmeta", c_void_p), ("probe_counts", c_void_p), ("probe_rows", c_int32),
                ("probe_regions", c_int32), ("projections", c_int32), ("probe_stall", c_int32),
                ("group_plan", c_int32)]


def default_options() -> ll_options:
    o = ll_options()
    o.schedule = -1
    o.spec_prefetch = -1
    o.group_plan = -1
    return o


class LLError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {ll_status_string(status)} ({status})")
        self.status = status


_lib = None


def load_library() -> ctypes.CDLL:
    """Load libll.so (raises if it is missing: no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; build it with `python -m paper_2406_06220_b200.build`")
    lib = ctypes.CDLL(LIB_PATH)
    P, J = POINTER(ll_predictor), POINTER(ll_joint)
    lib.ll_workspace_size.argtypes = [c_int32, c_int32, P, J, c_int32, c_int32, c_int32]
    lib.ll_workspace_size.restype = c_size_t
    lib.ll_decode_rnnt.argtypes = [c_void_p, c_int32, c_int32, c_int32, c_int32, c_void_p, P, J, c_int32,
                                   c_int32, c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_size_t,
                                   c_void_p]
    lib.ll_decode_rnnt.restype = c_int32
    lib.ll_decode_rnnt_frame_looping.argtypes = lib.ll_decode_rnnt.argtypes
    lib.ll_decode_rnnt_frame_looping.restype = c_int32
    lib.ll_decode_tdt.argtypes = [c_void_p, c_int32, c_int32, c_int32, c_int32, c_void_p, P, J, c_int32,
                                  c_int32, POINTER(c_int32), c_int32, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_int32, c_void_p, c_size_t, c_void_p]
    lib.ll_decode_tdt.restype = c_int32
    lib.ll_decode_rnnt_scores.argtypes = lib.ll_decode_rnnt.argtypes[:14] + [c_void_p] + lib.ll_decode_rnnt.argtypes[14:]
    lib.ll_decode_rnnt_scores.restype = c_int32
    lib.ll_decode_tdt_scores.argtypes = lib.ll_decode_tdt.argtypes[:17] + [c_void_p] + lib.ll_decode_tdt.argtypes[17:]
    lib.ll_decode_tdt_scores.restype = c_int32
    lib.ll_prepare.argtypes = [P, J, c_int32, c_int32, c_int32, c_int32, POINTER(c_int32), c_int32, c_void_p,
                               c_size_t, c_void_p]
    lib.ll_prepare.restype = c_int32
    lib.ll_sync.argtypes = [c_void_p, c_void_p]
    lib.ll_sync.restype = c_int32
    lib.ll_status_string.argtypes = [c_int32]
    lib.ll_status_string.restype = c_char_p
    lib.ll_stats.argtypes = [c_void_p, POINTER(c_uint64), c_void_p]
    lib.ll_stats.restype = c_int32
    lib.ll_debug_joint.argtypes = [c_void_p, c_void_p, c_int32, J, c_int32, c_int32, c_int32, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]
    lib.ll_debug_joint.restype = c_int32
    lib.ll_set_timing_events.argtypes = [c_void_p, c_void_p]
    lib.ll_set_timing_events.restype = c_int32
    lib.ll_release.argtypes = [c_void_p]
    lib.ll_release.restype = c_int32
    lib.ll_set_options.argtypes = [POINTER(ll_options)]
    lib.ll_set_options.restype = c_int32
    lib.ll_version.argtypes = []
    lib.ll_version.restype = c_char_p
    lib.ll_nccl_unique_id.argtypes = [c_void_p]
    lib.ll_nccl_unique_id.restype = c_int32
    lib.ll_nccl_comm_init.argtypes = [POINTER(c_void_p), c_int32, c_void_p, c_int32]
    lib.ll_nccl_comm_init.restype = c_int32
    lib.ll_nccl_comm_destroy.argtypes = [c_void_p]
    lib.ll_nccl_comm_destroy.restype = c_int32
    lib.ll_gather_workspace_size.argtypes = [c_int32, c_int32, c_int32]
    lib.ll_gather_workspace_size.restype = c_size_t
    lib.ll_gather_ragged.argtypes = [c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                     c_int32, c_void_p, ctypes.c_int64, POINTER(ctypes.c_int64), c_void_p, c_size_t,
                                     c_void_p]
    lib.ll_gather_ragged.restype = c_int32
    _lib = lib
    return lib


def ll_status_string(status: int) -> str:
    return load_library().ll_status_string(int(status)).decode()


def ll_version() -> str:
    return load_library().ll_version().decode()


def ll_workspace_size(B, T_max, pred: ll_predictor, joint: ll_joint, dtype, prec, num_durations) -> int:
    return int(load_library().ll_workspace_size(B, T_max, ctypes.byref(pred), ctypes.byref(joint), dtype,
                                                prec, num_durations))


def ll_decode_rnnt(enc, dtype, prec, B, T_max, lengths, pred, joint, blank_id, max_symbols, out_tokens,
                   out_timestamps, out_lengths, out_capacity, workspace, workspace_bytes, stream) -> int:
    return int(load_library().ll_decode_rnnt(enc, dtype, prec, B, T_max, lengths, ctypes.byref(pred),
                                             ctypes.byref(joint), blank_id, max_symbols, out_tokens,
                                             out_timestamps, out_lengths, out_capacity, workspace,
                                             workspace_bytes, stream))


def ll_decode_rnnt_scores(enc, dtype, prec, B, T_max, lengths, pred, joint, blank_id, max_symbols, out_tokens,
                          out_timestamps, out_lengths, out_capacity, out_scores, workspace, workspace_bytes,
                          stream) -> int:
    return int(load_library().ll_decode_rnnt_scores(enc, dtype, prec, B, T_max, lengths, ctypes.byref(pred),
                                                    ctypes.byref(joint), blank_id, max_symbols, out_tokens,
                                                    out_timestamps, out_lengths, out_capacity, out_scores,
                                                    workspace, workspace_bytes, stream))


def ll_decode_tdt_scores(enc, dtype, prec, B, T_max, lengths, pred, joint, blank_id, max_symbols, durations,
                         num_durations, out_tokens, out_timestamps, out_durations, out_lengths, out_capacity,
                         out_scores, workspace, workspace_bytes, stream) -> int:
    dur = None
    if durations is not None:
        dur = (c_int32 * max(1, len(durations)))(*[int(d) for d in durations])
    return int(load_library().ll_decode_tdt_scores(enc, dtype, prec, B, T_max, lengths, ctypes.byref(pred),
                                                   ctypes.byref(joint), blank_id, max_symbols, dur, num_durations,
                                                   out_tokens, out_timestamps, out_durations, out_lengths,
                                                   out_capacity, out_scores, workspace, workspace_bytes, stream))


def ll_prepare(pred, joint, dtype, prec, B, T_max, durations, num_durations, workspace, workspace_bytes,
               stream) -> int:
    dur = None
    if durations is not None:
        dur = (c_int32 * len(durations))(*durations)
    return int(load_library().ll_prepare(ctypes.byref(pred), ctypes.byref(joint), dtype, prec, B, T_max, dur,
                                         num_durations, workspace, workspace_bytes, stream))


def ll_decode_rnnt_frame_looping(enc, dtype, prec, B, T_max, lengths, pred, joint, blank_id, max_symbols,
                                 out_tokens, out_timestamps, out_lengths, out_capacity, workspace,
                                 workspace_bytes, stream) -> int:
    return int(load_library().ll_decode_rnnt_frame_looping(
        enc, dtype, prec, B, T_max, lengths, ctypes.byref(pred), ctypes.byref(joint), blank_id, max_symbols,
        out_tokens, out_timestamps, out_lengths, out_capacity, workspace, workspace_bytes, stream))


def ll_decode_tdt(enc, dtype, prec, B, T_max, lengths, pred, joint, blank_id, max_symbols, durations,
                  num_durations, out_tokens, out_timestamps, out_durations, out_lengths, out_capacity,
                  workspace, workspace_bytes, stream) -> int:
    dur = None
    if durations is not None:
        dur = (c_int32 * max(1, len(durations)))(*[int(d) for d in durations])
    return int(load_library().ll_decode_tdt(enc, dtype, prec, B, T_max, lengths, ctypes.byref(pred),
                                            ctypes.byref(joint), blank_id, max_symbols, dur, num_durations,
                                            out_tokens, out_timestamps, out_durations, out_lengths,
                                            out_capacity, workspace, workspace_bytes, stream))


def ll_sync(workspace, stream) -> int:
    return int(load_library().ll_sync(workspace, stream))


def ll_stats(workspace, stream):
    out = (c_uint64 * 13)()
    st = int(load_library().ll_stats(workspace, out, stream))
    return st, list(out)


def ll_debug_joint(enc_rows, g_rows, n, joint, dtype, prec, num_durations, out_logits, out_argmax,
                   out_dur_argmax, workspace, workspace_bytes, stream) -> int:
    return int(load_library().ll_debug_joint(enc_rows, g_rows, n, ctypes.byref(joint), dtype, prec,
                                             num_durations, out_logits, out_argmax, out_dur_argmax,
                                             workspace, workspace_bytes, stream))


def ll_set_timing_events(ev_before_decode, ev_after_decode) -> int:
    return int(load_library().ll_set_timing_events(ev_before_decode, ev_after_decode))


def ll_release(workspace) -> int:
    return int(load_library().ll_release(workspace))


def ll_set_options(opts) -> int:
    """opts: an ll_options struct, or None for the library defaults."""
    return int(load_library().ll_set_options(None if opts is None else ctypes.byref(opts)))


class options:
    """Context manager over ll_set_options (test / debug knobs of ll.h, this host
    thread only): `with ll.options(window=1, schedule=0): ...`."""

    def __init__(self, **kw):
        self.opts = default_options()
        for k, v in kw.items():
            setattr(self.opts, k, v)

    def __enter__(self):
        s = ll_set_options(self.opts)
        if s != LL_OK:
            raise LLError(s, "ll_set_options")
        return self.opts

    def __exit__(self, *exc):
        ll_set_options(None)


def ll_nccl_unique_id():
    """(status, 128-byte NCCL unique id)."""
    buf = ctypes.create_string_buffer(128)
    st = int(load_library().ll_nccl_unique_id(buf))
    return st, buf.raw


def ll_nccl_comm_init(nranks: int, uid: bytes, rank: int):
    """(status, opaque communicator handle)."""
    comm = c_void_p()
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    st = int(load_library().ll_nccl_comm_init(ctypes.byref(comm), nranks, buf, rank))
    return st, comm.value


def ll_nccl_comm_destroy(comm) -> int:
    return int(load_library().ll_nccl_comm_destroy(comm))


def ll_gather_workspace_size(B: int, out_capacity: int, with_durations: bool) -> int:
    return int(load_library().ll_gather_workspace_size(B, out_capacity, int(bool(with_durations))))


def ll_gather_ragged(comm, root, B, utt_ids, lengths, tokens, timestamps, durations, out_capacity, root_buf,
                     root_capacity, workspace, workspace_bytes, stream):
    """(status, elements written on root / needed on LL_ERR_CAPACITY)."""
    used = ctypes.c_int64(0)
    st = int(load_library().ll_gather_ragged(comm, root, B, utt_ids, lengths, tokens, timestamps, durations,
                                             out_capacity, root_buf, root_capacity, ctypes.byref(used),
                                             workspace, workspace_bytes, stream))
    return st, int(used.value)
