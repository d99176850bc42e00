#!/usr/bin/env python
"""Throughput of batched label-looping greedy decoding on B200 (arXiv 2406.06220).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config fc-rnnt] [--impl ours|reference]

One STEP decodes one batch of synthetic encoder outputs through the whole hot
path (encoder projection, model tables, the persistent label-looping kernel)
via the C ABI.  Default workload: BASELINE config (2) "fc-rnnt": B=32
utterances, T in U{225..275} frames (80 ms), D_e=512, LSTM predictor P=640,
joint H=640, V+1=1025, max_symbols=10, bf16, planted-alignment family
(DESIGN.md "Input recipe").  Metric: decoded audio-seconds per second (RTFx,
PAPER.md:234 footnote; 0.08 s per frame) -- plus utterances/s.

Timing: W untimed warm-up steps, then K steps, each bracketed by CUDA events on
the decode stream with a 512 MiB L2 flush between steps (outside the events);
a barrier + synchronize on both sides; the max over ranks.  Multi-GPU (torchrun):
each rank decodes its own batches (utterances are independent, no data-path
collective; weak scaling).

`--impl reference` times the float64 CPU oracle (oracle/, the conventional
sequential greedy decoder, Alg. 1) as it stands on the host cores, on a bounded
sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "decoded audio-sec/sec (RTFx) and utterances/sec at B=32, 1/2/4/8 B200"
UNIT = "audio-s/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="fc-rnnt", choices=list(synth.CONFIGS) + list(synth.SWEEPS))
    ap.add_argument("--chunk", type=int, default=1024, help="sweep: utterances per decode launch")
    ap.add_argument("--streams", type=int, default=1, help="sweep: concurrent decode streams (one workspace each)")
    ap.add_argument("--clock-window", type=float, default=1.0,
                    help="seconds of identical (untimed) steps the clock sampler watches at least")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--family", default="planted", choices=["planted", "random"])
    ap.add_argument("--frame-looping", action="store_true",
                    help="time the Alg. 2 frame-looping baseline (ll_decode_rnnt_frame_looping) instead")
    ap.add_argument("--schedule", default="ticks", choices=["ticks", "batched"],
                    help="label-looping schedule: per-row ticks (default) or the batched outer loop of Alg. 3 as listed")
    ap.add_argument("--projections", default="precompute", choices=["precompute", "on-the-fly"],
                    help="joint input projections precomputed (default, PAPER.md §3.4) or applied at every joint "
                         "evaluation (the ablation arm of Table 3; ll_options.projections = 1)")
    ap.add_argument("--batch", type=int, default=0,
                    help="decode only the first B utterances of the config's batch (Table 3's batch sizes 1 / 4)")
    ap.add_argument("--no-group-plan", action="store_true",
                    help="equal groups of consecutive utterances (ll_options.group_plan = 0) instead of the "
                         "length-sorted unequal groups")
    ap.add_argument("--group-rows", type=int, default=0,
                    help="force the rows per group R (ll_options.group_rows; tuning experiments)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="utterances in the oracle sample (0: auto)")
    return ap.parse_args()


def workload(cfg_name, seed, family="planted"):
    c = synth.CONFIGS[cfg_name]
    spec = c["spec"]
    if family == "planted" and spec.joint_dim >= 70:
        if spec.is_tdt:
            w, enc, lengths, _ = synth.make_planted_tdt(spec, seed, c["B"], c["T_max"], c["len_lo"], c["len_hi"])
        else:
            w, enc, lengths, _ = synth.make_planted_rnnt(spec, seed, c["B"], c["T_max"], c["len_lo"], c["len_hi"],
                                                         rho=c.get("rho", 0.28))
    else:
        w = synth.make_weights(spec, seed, blank_bias=synth.random_family_blank_bias(spec))
        enc, lengths = synth.make_inputs(seed + 1, c["B"], c["T_max"], spec.enc_dim, c["len_lo"], c["len_hi"])
    return spec, w, enc, lengths


def frame_s_of(cfg_name):
    """Seconds of audio per encoder frame (8x subsampling: 80 ms, PAPER.md:233;
    the 4x-subsampling variant: 40 ms)."""
    return synth.CONFIGS.get(cfg_name, {}).get("frame_s", synth.frame_seconds)


spec_name_hint = ["fc-rnnt"]


def algorithmic_flops(spec, stats, total_frames):
    """a1 L*2*D_e*H; a3 E*2*H*(V+1+|D|); a2 S*(2*(P+P)*4P [LSTM] + 2*P*H)."""
    H, P, De = spec.joint_dim, spec.pred_dim, spec.enc_dim
    V = spec.num_tokens + (len(spec.durations) if spec.is_tdt else 0)
    E, S = stats["joint_evals"], stats["predictor_rows"]
    a1 = total_frames * 2 * De * H
    a3 = E * 2 * H * V
    a2 = S * ((2 * (P + P) * 4 * P) if spec.pred_kind == "lstm" else 0) + S * 2 * P * H
    return a1, a2, a3


# Primitive latencies measured on the B200 itself (tools/microbench.cu,
# profiles/r01_microbench.txt), in SM cycles.
LAT_HMMA = 20.8        # dependent mma.sync.m16n8k16 bf16
LAT_LDS = 28.6         # dependent shared-memory load
LAT_BAR = 30.7         # CTA barrier (bar.sync)
LAT_XCTA = 125.7 / 2   # st.async + mbarrier, one way between two CTAs of a 16-CTA cluster


def chain_floor_cycles(spec):
    """Lower bounds (cycles) on one joint round and one predictor step of the
    decode kernel's dependent chain (DESIGN.md §7 "dependency-chain floor"):
    only the latencies no implementation of the cluster decomposition can
    avoid -- the K-chain of the tensor-core contraction (two accumulator chains
    over K), one shared-memory read, the CTA barriers and the one-way DSMEM
    exchanges; no bandwidth term, no control code."""
    H, P = spec.joint_dim, spec.pred_dim
    joint = LAT_LDS + LAT_BAR + (H // 16) / 2 * LAT_HMMA + LAT_XCTA + LAT_BAR
    if spec.pred_kind == "lstm":
        # W_hh h does not depend on the next label (only E'[y] does), so it is off
        # the chain (the FC kernels compute it in the background on tcgen05)
        pred = (LAT_LDS + LAT_XCTA                                     # pre-activation read + cell, h' exchange
                + (P // 16) / 10 * LAT_HMMA + LAT_LDS + LAT_BAR        # W_pred, K split over 10 warps
                + LAT_XCTA + LAT_BAR)                                  # g exchange
    else:
        pred = LAT_LDS + LAT_BAR                                       # table lookup
    return joint, pred


def chain_floor_ms(spec, rounds, pred_steps, sm_mhz):
    j, pr = chain_floor_cycles(spec)
    return (rounds * j + pred_steps * pr) / (sm_mhz * 1e3)


def cpu_info():
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def spawn_ranks(a):
    """`--gpus N` without a torchrun environment: re-launch this command under
    torch.distributed.run with N ranks (one per GPU, 127.0.0.1 rendezvous)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def oracle_worker(args):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    spec, w, enc_row, L = args
    from oracle import Transducer, decode_sequential
    model = Transducer.from_spec(spec, w)
    r = decode_sequential(model, enc_row, L, spec.max_symbols)
    return len(r.tokens)


def cpu_oracle_time(spec, w, enc, lengths, n_utt, cfg_name="fc-rnnt"):
    """Time the float64 oracle (as it stands) on the host cores: one utterance per task."""
    spec_name_hint[0] = cfg_name
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    idx = list(range(min(n_utt, enc.shape[0])))
    tasks = [(spec, w, enc[b], int(lengths[b])) for b in idx]
    ctx = mp.get_context("fork")
    procs = min(cores, len(tasks))
    with ctx.Pool(procs, initializer=_limit_threads) as pool:
        pool.map(oracle_worker, tasks[:procs])  # warm the workers (imports)
        t0 = time.perf_counter()
        pool.map(oracle_worker, tasks, chunksize=1)
        dt = time.perf_counter() - t0
    audio = float(sum(int(lengths[b]) for b in idx)) * frame_s_of(spec_name_hint[0])
    return audio / dt, dt, procs, len(idx), audio


def _limit_threads():
    """One BLAS thread per worker process (the pool supplies the parallelism)."""
    try:
        import threadpoolctl
        threadpoolctl.threadpool_limits(1)
    except Exception:
        pass


def sweep_sample(cfg_name, n):
    """The first n utterances (by id) of a sweep workload: (spec, w, enc, lengths)."""
    c = synth.SWEEPS[cfg_name]
    spec = c["spec"]
    w, codes = synth.planted_weights(spec, 1000)
    L = synth.sweep_lengths(c["length_seed"], c["n_utt"])[:n]
    T = int(L.max())
    enc = np.zeros((n, T, spec.enc_dim), dtype=np.float32)
    for u in range(n):
        enc[u, :L[u]] = synth.planted_utterance(spec, codes, c["length_seed"], u, int(L[u]))[0]
    return spec, w, enc, L.astype(np.int32)


def run_reference(a, rank, world):
    if rank != 0:
        return
    if a.config in synth.SWEEPS:
        spec, w, enc, lengths = sweep_sample(a.config, a.cpu_sample or 64)
    else:
        spec, w, enc, lengths = workload(a.config, 1000, a.family)
    n = a.cpu_sample or enc.shape[0]
    times = []
    for i in range(a.warmup + a.steps):
        v, dt, procs, nutt, audio = cpu_oracle_time(spec, w, enc, lengths, n, a.config)
        if i >= a.warmup:
            times.append((v, dt))
    value = statistics.mean(v for v, _ in times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * statistics.mean(d for _, d in times),
        "higher_is_better": True, "scaling": "strong" if a.config in synth.SWEEPS else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": a.config, "family": a.family, "sample_utts": nutt},
        "cpu_baseline": dict({"value": value, "unit": UNIT, "cores": procs, "kind": "oracle",
                              "impl": "oracle/ Python + numpy float64, sequential greedy (Alg. 1), "
                                      "one process per utterance",
                              "sample": f"{nutt} utterances ({audio:.1f} audio-s) of the {a.config} batch per step"},
                             **cpu_info()),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        sys.exit(spawn_ranks(a))   # one process per GPU under torch.distributed.run
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    if a.impl == "reference":
        return run_reference(a, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2406_06220_b200 import build as llbuild
    from paper_2406_06220_b200 import ll
    from paper_2406_06220_b200.decoder import LabelLoopingDecoder, Model

    llbuild.build()
    if a.schedule == "batched" or a.projections == "on-the-fly" or a.no_group_plan or a.group_rows:
        o = ll.options(schedule=0 if a.schedule == "batched" else -1,   # ll_options of this thread
                       projections=1 if a.projections == "on-the-fly" else 0,
                       group_plan=0 if a.no_group_plan else -1, group_rows=a.group_rows).opts
        if ll.ll_set_options(o) != ll.LL_OK:
            raise RuntimeError("ll_set_options")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    if a.config in synth.SWEEPS:
        return run_sweep(a, rank, world, local, dev)

    # weak scaling: every rank decodes its own batch (seed 1000 + rank)
    spec, w, enc_np, len_np = workload(a.config, 1000 + rank, a.family)
    if a.batch > 0:   # the first B utterances of the seeded batch
        enc_np, len_np = enc_np[:a.batch].copy(), len_np[:a.batch].copy()
    B, T = enc_np.shape[0], enc_np.shape[1]
    model = Model(w, spec.pred_kind, spec.context, spec.blank_id, spec.durations, "bf16", device=f"cuda:{local}")
    dec = LabelLoopingDecoder(model, spec.max_symbols, B, T, frame_looping=a.frame_looping)
    dec.prepare()      # weight-only model tables, once per model (ll_prepare)
    enc = torch.from_numpy(enc_np).to(dev, torch.bfloat16)
    lengths = torch.from_numpy(len_np).to(dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    ev_k0 = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ev_k1 = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ev_s0 = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ev_s1 = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    for e in ev_k0 + ev_k1:      # torch creates CUDA events lazily: force the handles now
        e.record(stream)

    def step():
        s = dec.launch(enc, lengths)
        if s != ll.LL_OK:
            raise ll.LLError(s, "decode")

    for _ in range(a.warmup):
        step()
    if dec.sync() != ll.LL_OK:
        raise RuntimeError("warm-up decode failed")
    stats = dec.stats()
    ref_out = dec.tokens.clone(), dec.lengths_out.clone()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(a.steps):
            flush.zero_()
            ev_s0[i].record(stream)
            ll.ll_set_timing_events(ev_k0[i].cuda_event, ev_k1[i].cuda_event)
            step()
            ll.ll_set_timing_events(None, None)
            ev_s1[i].record(stream)
        torch.cuda.synchronize()
        # the clock record needs a sustained window: identical untimed steps
        # until --clock-window seconds have passed (the timed K steps above are
        # the measurement)
        t_end = time.perf_counter() + a.clock_window
        while time.perf_counter() < t_end:
            for _ in range(20):
                flush.zero_()
                step()
            torch.cuda.synchronize()
    if dec.sync() != ll.LL_OK:
        raise RuntimeError("timed decode failed")
    step_ms = [ev_s0[i].elapsed_time(ev_s1[i]) for i in range(a.steps)]
    kern_ms = [ev_k0[i].elapsed_time(ev_k1[i]) for i in range(a.steps)]
    assert torch.equal(dec.tokens, ref_out[0]) and torch.equal(dec.lengths_out, ref_out[1]), "non-deterministic"
    tot_ms = sum(step_ms)

    # End to end through the public API with host buffers, as a serving loop
    # would run it: every step copies ITS inputs from pinned host memory (H2D)
    # and reads ITS hypotheses back (D2H).  Two decoders (two workspaces) and
    # double-buffered inputs / outputs let step i+1's H2D run on a copy stream
    # while step i decodes; the L2 flush stays before every decode, inside the
    # timed region.  Timed as one region over the K steps (CUDA events).
    dec2 = LabelLoopingDecoder(model, spec.max_symbols, B, T, frame_looping=a.frame_looping)
    dec2.prepare()
    decs = [dec, dec2]
    enc_h = torch.from_numpy(enc_np).to(torch.bfloat16).pin_memory()
    len_h = torch.from_numpy(len_np).pin_memory()
    bufs = [(torch.empty_like(enc), torch.empty_like(lengths)) for _ in range(2)]
    outs = [tuple(torch.empty_like(t, device="cpu").pin_memory() for t in (d.tokens, d.timestamps, d.lengths_out))
            for d in decs]
    h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)   # separate: in-order streams
    ev_in = [torch.cuda.Event() for _ in range(2)]     # inputs of buffer j landed
    ev_dec = [torch.cuda.Event() for _ in range(2)]    # decode on buffer j finished
    ev_out = [torch.cuda.Event() for _ in range(2)]    # results of buffer j read back
    for e in ev_in + ev_dec + ev_out:
        e.record(stream)

    def e2e_steps(n):
        for i in range(n):
            j = i & 1
            with torch.cuda.stream(h2d_s):
                h2d_s.wait_event(ev_dec[j])            # buffer j's previous decode has consumed its inputs
                bufs[j][0].copy_(enc_h, non_blocking=True)
                bufs[j][1].copy_(len_h, non_blocking=True)
                ev_in[j].record(h2d_s)
            stream.wait_event(ev_in[j])
            stream.wait_event(ev_out[j])               # decoder j's previous results were read
            flush.zero_()
            st = decs[j].launch(bufs[j][0], bufs[j][1], stream)
            if st != ll.LL_OK:
                raise ll.LLError(st, "decode")
            ev_dec[j].record(stream)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(ev_dec[j])
                for h, d in zip(outs[j], (decs[j].tokens, decs[j].timestamps, decs[j].lengths_out)):
                    h.copy_(d, non_blocking=True)
                ev_out[j].record(d2h_s)
        stream.wait_event(ev_out[(n - 1) & 1])
        if n > 1:
            stream.wait_event(ev_out[(n - 2) & 1])

    e2e_steps(max(a.warmup, 2))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], ref_out[0].cpu()) and torch.equal(outs[1][0], ref_out[0].cpu()), "e2e results differ"
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_steps(a.steps)
    e1.record(stream)
    e1.synchronize()
    e2e_ms = [e0.elapsed_time(e1)]
    h2d = enc_h.numel() * enc_h.element_size() + len_h.numel() * 4
    d2h = sum(t.numel() * 4 for t in outs[0])

    # single-call latency: the same public call with nothing overlapped -- H2D of
    # the inputs, the decode, D2H of the hypotheses, back to back on one stream
    def single_calls(n):
        for _ in range(n):
            bufs[0][0].copy_(enc_h, non_blocking=True)
            bufs[0][1].copy_(len_h, non_blocking=True)
            flush.zero_()
            st = decs[0].launch(bufs[0][0], bufs[0][1], stream)
            if st != ll.LL_OK:
                raise ll.LLError(st, "decode")
            for h, d in zip(outs[0], (decs[0].tokens, decs[0].timestamps, decs[0].lengths_out)):
                h.copy_(d, non_blocking=True)

    with torch.cuda.stream(stream):
        single_calls(2)
        torch.cuda.synchronize()
        e0.record(stream)
        single_calls(a.steps)
        e1.record(stream)
    e1.synchronize()
    single_ms = e0.elapsed_time(e1) / a.steps

    # whole-job aggregate: the audio / utterances of ALL ranks over the max-over-ranks time
    audio_s = float(len_np.sum()) * frame_s_of(a.config)
    t_all = torch.tensor([tot_ms, sum(e2e_ms)], dtype=torch.float64, device=dev)
    work = torch.tensor([audio_s, float(B)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_all, op=dist.ReduceOp.MAX)
        dist.all_reduce(work, op=dist.ReduceOp.SUM)
        dist.barrier()
    tot_ms_max, e2e_ms_max = float(t_all[0]), float(t_all[1])
    audio_all, utt_all = float(work[0]), float(work[1])
    value = a.steps * audio_all / (tot_ms_max / 1e3)
    utt_s = a.steps * utt_all / (tot_ms_max / 1e3)
    e2e_value = a.steps * audio_all / (e2e_ms_max / 1e3)

    # roofline of the dominant kernel (the persistent decode kernel)
    a1, a2, a3 = algorithmic_flops(spec, stats, int(len_np.sum()))
    kern_mean = statistics.mean(kern_ms)
    peaks = {}
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        peaks = json.load(open(pk_path))
    peak = peaks.get("bf16_tflops", 1590.0)
    if a.projections == "on-the-fly":   # the decode kernel also does the projections (a1 is counted once)
        a2 += a1
    achieved = (a2 + a3) / (kern_mean / 1e3) / 1e12
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        traffic = json.load(open(tr_path)).get(a.config)
    clocks = clk.summary()
    sm_mhz = (clocks or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    floor = chain_floor_ms(spec, stats["chain_rounds"], stats["chain_pred_steps"], sm_mhz)
    jf, pf = chain_floor_cycles(spec)

    rows = stats["joint_evals"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": tot_ms_max / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": a.config, "family": a.family, "B": B, "T_max": T,
                   "algorithm": "frame-looping (Alg. 2 baseline)" if a.frame_looping else
                   ("label-looping (Alg. 3), batched outer loop" if a.schedule == "batched"
                    else "label-looping (Alg. 3), per-row ticks"),
                   "projections": a.projections + (" (W_enc, W_pred applied at every joint evaluation, inside "
                                                   "the decode kernel; no f)" if a.projections == "on-the-fly" else
                                                   " (encoder GEMM over all frames + g once per predictor step)"),
                   "frames": int(len_np.sum()), "audio_s_per_step": audio_s, "l2": "flushed (512 MiB) between steps",
                   "model_tables": "prepared once per model (ll_prepare), outside the step",
                   "parallelism": f"utterance-sharded x{world} (each rank its own B={B} batch)"},
        "utterances_per_s": utt_s,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms_max / a.steps,
                "mode": "serving loop: step i+1's H2D overlaps step i's decode (H2D / D2H streams, 2 workspaces)",
                "single_call": {"ms": single_ms, "value": audio_s / (single_ms / 1e3), "unit": UNIT,
                                "mode": "one call at a time: H2D, decode, D2H back to back on one stream (latency)"}},
        # the library's own count of the call's kernels (ll_stats [12]): encoder projection GEMM (not on
        # the fly), the length ranking (decodes of several groups), the decode kernel; tables prepared once
        "gpu_launches": a.steps * stats["launches"],
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": "decode_kernel",
                     "kernel_ms": kern_mean, "kernel_share_of_step": kern_mean / (tot_ms_max / a.steps),
                     "flops_per_launch": a2 + a3,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)" if peaks else "fallback 1.59 PF"},
        "chain_floor": {"ms": floor, "frac": floor / kern_mean, "kernel_ms": kern_mean,
                        "critical_cluster": {"joint_rounds": stats["chain_rounds"],
                                             "predictor_steps": stats["chain_pred_steps"]},
                        "cycles_per_round": jf, "cycles_per_predictor_step": pf, "sm_mhz": sm_mhz,
                        "basis": "dependent-latency lower bound per phase from measured primitive latencies "
                                 "(profiles/r01_microbench.txt; DESIGN.md §7)"},
        "decode_stats": {"labels": stats["labels"], "tokens_per_frame": stats["labels"] / max(1, int(len_np.sum())),
                         "outer_steps": stats["outer_steps"], "joint_rounds": stats["joint_rounds"],
                         "mean_active_rows": rows / max(1, stats["joint_rounds"]),
                         "predictor_steps": stats["predictor_steps"], "groups": stats["groups"],
                         "cluster_size": stats["cluster_size"], "window": stats["window"],
                         "group_rows": stats["group_rows"]},
        "context": "paper: 5197.2 non-encoder RTFx RNNT-L B=32 with CUDA graphs on one RTX A6000, bf16 (PAPER.md:354)",
    }
    if rank == 0 and not a.no_cpu_baseline:
        n = a.cpu_sample or B
        v, dt, procs, nutt, audio = cpu_oracle_time(spec, w, enc_np, len_np, n, a.config)
        line["cpu_baseline"] = dict({"value": v, "unit": UNIT, "cores": procs, "kind": "oracle",
                                     "impl": "oracle/ Python + numpy float64, sequential greedy (Alg. 1), "
                                             "one process per utterance",
                                     "sample": f"{nutt} utterances ({audio:.1f} audio-s) of the {a.config} batch, "
                                               f"{dt:.1f} s wall"}, **cpu_info())
    if clocks:
        clocks["window"] = f"the {a.steps} timed steps + identical untimed steps to >= {a.clock_window} s"
        line["clocks"] = clocks
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sweep(a, rank, world, local, dev):
    """BASELINE config (5): 8192 utterances with LibriSpeech-like lengths,
    length-bucketed into batches of 32 and assigned to ranks by LPT
    (paper_2406_06220_b200.shard).  Each rank decodes its shard longest-first in
    launches of `--chunk` utterances spread round-robin over `--streams` CUDA
    streams (one workspace each; no host sync between launches), every launch
    writing its rows of the rank's [n, cap] output buffers; then the rank's
    ragged hypotheses are gathered on rank 0 with ll_gather_ragged (NCCL, the
    only collective).  A step = the whole sweep, gather included; strong
    scaling (the total work is fixed)."""
    import torch
    import torch.distributed as dist
    from paper_2406_06220_b200 import ll, shard
    from paper_2406_06220_b200.decoder import LabelLoopingDecoder, Model

    c = synth.SWEEPS[a.config]
    spec = c["spec"]
    tdt = spec.is_tdt
    w, codes = synth.planted_weights(spec, 1000)
    L_all = synth.sweep_lengths(c["length_seed"], c["n_utt"])
    ids = shard.rank_shard(L_all, world, rank, c["batch"])
    n_loc = len(ids)
    T_glob = int(L_all.max())
    model = Model(w, spec.pred_kind, spec.context, spec.blank_id, spec.durations, "bf16", device=f"cuda:{local}")
    nstreams = max(1, a.streams)
    decs = [LabelLoopingDecoder(model, spec.max_symbols, a.chunk, T_glob) for _ in range(nstreams)]
    for d in decs:
        d.prepare()
    cap = decs[0].cap
    # the rank's output buffers: every launch writes its rows (contiguous row slices)
    out_tok = torch.zeros(max(n_loc, 1), cap, dtype=torch.int32, device=dev)
    out_ts = torch.zeros_like(out_tok)
    out_du = torch.zeros_like(out_tok) if tdt else None
    out_len = torch.zeros(max(n_loc, 1), dtype=torch.int32, device=dev)
    # inputs: planted utterances (each from its own seeded stream), laid out per
    # launch as [B_c, T_c, D_e] bf16 on the device; the ragged frames are also
    # kept in pinned host memory for the end-to-end leg
    chunks, planted = [], {}
    for c0 in range(0, n_loc, a.chunk):
        cid = ids[c0:c0 + a.chunk]
        Lc = L_all[cid]
        T = int(Lc.max())
        enc = torch.zeros(len(cid), T, spec.enc_dim, dtype=torch.bfloat16, device=dev)
        host = []
        for i, u in enumerate(cid):
            e, pl = synth.planted_utterance(spec, codes, c["length_seed"], int(u), int(L_all[u]))
            planted[int(u)] = pl
            eh = torch.from_numpy(e).to(torch.bfloat16)
            host.append(eh)
            enc[i, :e.shape[0]] = eh.to(dev)
        frames = torch.cat(host).pin_memory()
        rows = torch.cat([torch.arange(int(l), device=dev) + i * T for i, l in enumerate(Lc)])
        sl = slice(c0, c0 + len(cid))
        chunks.append(dict(enc=enc, lengths=torch.from_numpy(Lc.astype(np.int32)).to(dev), frames=frames, rows=rows,
                           out=(out_tok[sl], out_ts[sl], None if out_du is None else out_du[sl], out_len[sl]),
                           frames_n=int(Lc.sum())))
    ids32 = torch.from_numpy(ids.astype(np.int32)).to(dev)
    stream = torch.cuda.current_stream()
    streams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(nstreams - 1)]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    gather = shard.NcclGather(device=dev)   # ll_gather_ragged on a libll NCCL communicator (world 1 too)

    h2d_s = torch.cuda.Stream(device=dev)
    ev_in = [torch.cuda.Event() for _ in chunks]
    ev_dec = [torch.cuda.Event() for _ in chunks]
    ev_fork, ev_join = torch.cuda.Event(), [torch.cuda.Event() for _ in streams]
    ev_k = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in chunks]
    for e in ev_dec + [x for p in ev_k for x in p]:
        e.record(stream)

    def step(e2e=False, timed=False):
        if e2e:   # H2D of every chunk's ragged frames (scattered into the padded layout) on a copy
            # stream, so chunk k+1's copy overlaps chunk k's decode
            with torch.cuda.stream(h2d_s):
                for k, ch in enumerate(chunks):
                    h2d_s.wait_event(ev_dec[k])     # the chunk's previous decode has read its inputs
                    dst = ch["enc"].view(-1, spec.enc_dim)
                    dst.index_copy_(0, ch["rows"], ch["frames"].to(dev, non_blocking=True))
                    ev_in[k].record(h2d_s)
        ev_fork.record(stream)
        for s_ in streams[1:]:
            s_.wait_event(ev_fork)
        for k, ch in enumerate(chunks):
            j = k % nstreams
            st = streams[j]
            if e2e:
                st.wait_event(ev_in[k])
            if timed:
                ll.ll_set_timing_events(ev_k[k][0].cuda_event, ev_k[k][1].cuda_event)
            s = decs[j].launch(ch["enc"], ch["lengths"], st, out=ch["out"])
            if timed:
                ll.ll_set_timing_events(None, None)
            ev_dec[k].record(st)
            if s != ll.LL_OK:
                raise ll.LLError(s, "decode")
        for j, s_ in enumerate(streams[1:], 1):
            ev_join[j].record(s_)
            stream.wait_event(ev_join[j])
        buf = gather.gather(ids32, out_len[:n_loc], out_tok[:n_loc], out_ts[:n_loc],
                            out_du[:n_loc] if tdt else None)
        if rank != 0:
            return None
        return buf.cpu() if e2e else buf   # e2e: D2H of the gathered hypotheses

    for _ in range(a.warmup):
        gathered = step()
    torch.cuda.synchronize()
    gathered_ok = True
    if rank == 0:   # the gathered records hold every utterance once; this rank's equal their planted alignments
        merged = shard.unpack_records(gathered.cpu().numpy(), tdt)
        gathered_ok = len(merged) == int(c["n_utt"]) and all(merged[u] == tuple(planted[u]) for u in planted)
    for d in decs:
        if d.sync() != ll.LL_OK:
            raise RuntimeError("sweep decode failed")
    # statistics of one sweep (per launch: each decoder's stats are its last launch's)
    agg = dict(joint_evals=0, predictor_rows=0, labels=0, joint_rounds=0, predictor_steps=0, groups=0)
    chain_ms_floor = 0.0
    per_launch = []
    for k, ch in enumerate(chunks):
        d = decs[k % nstreams]
        d.launch(ch["enc"], ch["lengths"], streams[0], out=ch["out"])
        st = d.stats(streams[0])
        per_launch.append(st)
        for key in agg:
            agg[key] += st[key]
    # correctness of the sweep: every utterance of this shard equals its planted alignment
    tok, ts, ln = out_tok[:n_loc].cpu(), out_ts[:n_loc].cpu(), out_len[:n_loc].cpu()
    du = out_du[:n_loc].cpu() if tdt else None
    bad = 0
    for i, u in enumerate(ids.tolist()):
        k = int(ln[i])
        got = (tok[i, :k].tolist(), ts[i, :k].tolist()) + ((du[i, :k].tolist(),) if tdt else ())
        bad += got != tuple(planted[u])
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    kern = []
    with ClockSampler(local) as clk:
        for i in range(a.steps):
            flush.zero_()
            if world > 1:
                dist.barrier()
            ev0[i].record(stream)
            step(timed=True)
            ev1[i].record(stream)
            torch.cuda.synchronize()
            kern.append([ev_k[k][0].elapsed_time(ev_k[k][1]) for k in range(len(chunks))])
        t_end = time.perf_counter() + a.clock_window
        while time.perf_counter() < t_end:
            step()
            torch.cuda.synchronize()
    ms = [ev0[i].elapsed_time(ev1[i]) for i in range(a.steps)]
    e2e_ms, d2h = [], 0
    for i in range(a.steps):
        flush.zero_()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        got = step(e2e=True)
        e1.record(stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
        d2h = got.numel() * 4 if got is not None else 0
    t_all = torch.tensor([sum(ms), sum(e2e_ms), float(bad)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_all, op=dist.ReduceOp.MAX)
    tot_ms, e2e_tot, bad_max = float(t_all[0]), float(t_all[1]), int(t_all[2])
    audio_s = float(L_all.sum()) * synth.frame_seconds
    n_utt = int(c["n_utt"])
    value = a.steps * audio_s / (tot_ms / 1e3)
    h2d = sum(ch["frames"].numel() * 2 + ch["lengths"].numel() * 4 for ch in chunks)
    # roofline of the decode kernel on this rank: algorithmic FLOPs of every
    # launch over that launch's duration (CUDA events on its stream), averaged
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("bf16_tflops", 1590.0)
    kern_mean = [statistics.mean(kern[i][k] for i in range(a.steps)) for k in range(len(chunks))]
    flops = []
    for k, ch in enumerate(chunks):
        _, a2, a3 = algorithmic_flops(spec, per_launch[k], ch["frames_n"])
        flops.append(a2 + a3)
    achieved = sum(flops) / (sum(kern_mean) / 1e3) / 1e12
    clocks = clk.summary()
    sm_mhz = (clocks or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    floor = sum(chain_floor_ms(spec, st["chain_rounds"], st["chain_pred_steps"], sm_mhz) for st in per_launch)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": tot_ms / a.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic",
        "config": {"workload": a.config, "family": "planted", "utterances": n_utt, "batch": c["batch"],
                   "launch_batch": a.chunk, "streams": nstreams, "launches_per_rank": len(chunks),
                   "frames": int(L_all.sum()), "audio_s_per_step": audio_s,
                   "l2": "flushed (512 MiB) between steps", "parallelism": f"LPT length-bucketed x{world}, NCCL gather"},
        "utterances_per_s": a.steps * n_utt / (tot_ms / 1e3),
        "e2e": {"value": a.steps * audio_s / (e2e_tot / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_tot / a.steps},
        # per launch: the library's own count (ll_stats [12]: projection GEMM, length ranking, decode);
        # per step: the two packing kernels of ll_gather_ragged (NCCL's own all-gather / send-recv
        # kernels not counted); model tables prepared once before timing
        "gpu_launches": a.steps * (sum(st["launches"] for st in per_launch) + 2),
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": None, "kernel": "decode_kernel (rank 0, every launch)",
                     "kernel_ms_sum": sum(kern_mean), "flops_per_step": sum(flops),
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)" if peaks else "fallback 1.59 PF"},
        "chain_floor": {"ms": floor, "frac": floor / sum(kern_mean), "kernel_ms_sum": sum(kern_mean),
                        "basis": "sum over launches of the per-launch dependency-chain floor (DESIGN.md §7)"},
        "decode_stats": dict(agg, tokens_per_frame=agg["labels"] / max(1, sum(ch["frames_n"] for ch in chunks))),
        "hypotheses_equal_planted": bad_max == 0,
        "gathered_hypotheses_ok": gathered_ok,
    }
    if rank == 0 and not a.no_cpu_baseline:
        sp, ws_, enc_s, len_s = sweep_sample(a.config, a.cpu_sample or 64)
        v, dt, procs, nutt, audio = cpu_oracle_time(sp, ws_, enc_s, len_s, len(len_s), a.config)
        line["cpu_baseline"] = dict({"value": v, "unit": UNIT, "cores": procs, "kind": "oracle",
                                     "impl": "oracle/ Python + numpy float64, sequential greedy (Alg. 1), "
                                             "one process per utterance",
                                     "sample": f"utterances 0..{nutt - 1} of the sweep ({audio:.1f} audio-s), "
                                               f"{dt:.1f} s wall"}, **cpu_info())
    if clocks:
        clocks["window"] = f"the {a.steps} timed steps + identical untimed steps to >= {a.clock_window} s"
        line["clocks"] = clocks
    if rank == 0:
        print(json.dumps(line), flush=True)
    gather.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
