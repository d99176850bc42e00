"""Host-side multi-GPU logic: LPT partitioning of a
length-bucketed sweep and the ragged all-gather of hypotheses, the latter run
with world_size 2 over gloo on CPU (the GPU path uses NCCL through the same
torch.distributed calls)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2406_06220_b200 import shard


def test_buckets_and_lpt_cover_every_utterance_once():
    L = synth.sweep_lengths(2024, 8192)
    for n in (1, 2, 4, 8):
        ids = np.concatenate([shard.rank_shard(L, n, r, 32) for r in range(n)])
        assert sorted(ids.tolist()) == list(range(8192))
        for r in range(n):   # longest first inside a shard
            s = L[shard.rank_shard(L, n, r, 32)]
            assert (np.diff(s) <= 0).all()


def test_lpt_balance_on_sweep_lengths():
    """LPT max/mean load on the config-5 lengths (SURVEY.md §8(e) reports
    1.000 / 1.000 / 1.0002 / 1.0033 at G = 1/2/4/8)."""
    L = synth.sweep_lengths(2024, 8192)
    batches = shard.length_buckets(L, 32)
    assert len(batches) == 256
    for n, bound in ((1, 1.0), (2, 1.001), (4, 1.002), (8, 1.01)):
        asg = shard.lpt_assign(batches, L, n)
        load = [sum(int(L[batches[i]].max()) for i in a) for a in asg]
        assert max(load) / np.mean(load) <= bound, (n, load)


def test_lpt_small_cases():
    # 3 batches of costs 5, 4, 3 on 2 ranks -> {5}, {4, 3}
    L = [5, 4, 3]
    b = shard.length_buckets(L, 1)
    asg = shard.lpt_assign(b, L, 2)
    loads = sorted(sum(L[int(b[i][0])] for i in a) for a in asg)
    assert loads == [5, 7]
    assert shard.lpt_assign(b, L, 5)[3] == [] and shard.lpt_assign(b, L, 5)[4] == []
    with pytest.raises(ValueError):
        shard.lpt_assign(b, L, 0)


def _fake_results(ids, cap, tdt, seed):
    rng = np.random.default_rng(seed)
    B = len(ids)
    lens = rng.integers(0, cap + 1, size=B)
    tok = rng.integers(1, 1025, size=(B, cap))
    ts = np.sort(rng.integers(0, 500, size=(B, cap)), axis=1)
    du = rng.integers(0, 5, size=(B, cap)) if tdt else None
    return lens, tok, ts, du


@pytest.mark.parametrize("tdt", [False, True])
def test_unpack_records_concatenation(tdt):
    """The root buffer of ll_gather_ragged is a concatenation of records (one
    per rank per call, an empty record being [0]); unpack_records parses it to
    the union of the records' hypotheses."""
    parts, want = [], {}
    for k, ids in enumerate([np.array([5, 2]), np.array([], dtype=np.int64), np.array([9, 1, 4])]):
        lens, tok, ts, du = _fake_results(ids, 6, tdt, 10 + k)
        buf = shard.pack_hypotheses(torch.from_numpy(ids), torch.from_numpy(lens), torch.from_numpy(tok),
                                    torch.from_numpy(ts), None if du is None else torch.from_numpy(du))
        parts.append(buf)
        want.update(shard.unpack_hypotheses(buf.numpy(), tdt))
    assert parts[1].tolist() == [0]
    got = shard.unpack_records(torch.cat(parts).numpy(), tdt)
    assert got == want and sorted(got) == [1, 2, 4, 5, 9]


@pytest.mark.parametrize("tdt", [False, True])
def test_pack_unpack_roundtrip(tdt):
    ids = np.array([7, 3, 11, 0])
    lens, tok, ts, du = _fake_results(ids, 9, tdt, 1)
    lens[1] = 0
    buf = shard.pack_hypotheses(torch.from_numpy(ids), torch.from_numpy(lens), torch.from_numpy(tok),
                                torch.from_numpy(ts), None if du is None else torch.from_numpy(du))
    out = shard.unpack_hypotheses(buf.numpy(), tdt)
    assert sorted(out) == sorted(ids.tolist())
    for i, u in enumerate(ids):
        n = int(lens[i])
        want = (tok[i, :n].tolist(), ts[i, :n].tolist()) + ((du[i, :n].tolist(),) if tdt else ())
        assert out[int(u)] == want


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tdt, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = synth.sweep_lengths(2024, 300)
    ids = shard.rank_shard(L, world, rank, 32)
    lens, tok, ts, du = _fake_results(ids, 12, tdt, 100 + rank)
    buf = shard.pack_hypotheses(torch.from_numpy(ids), torch.from_numpy(lens), torch.from_numpy(tok),
                                torch.from_numpy(ts), None if du is None else torch.from_numpy(du))
    merged = shard.gather_ragged(buf, tdt)
    if rank == 0:
        # rank 0 rebuilds every rank's expected results independently
        want = {}
        for r in range(world):
            rid = shard.rank_shard(L, world, r, 32)
            ln, tk, tss, dd = _fake_results(rid, 12, tdt, 100 + r)
            for i, u in enumerate(rid):
                n = int(ln[i])
                want[int(u)] = (tk[i, :n].tolist(), tss[i, :n].tolist()) + ((dd[i, :n].tolist(),) if tdt else ())
        q.put(merged == want and sorted(merged) == list(range(300)))
    else:
        q.put(merged is None)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("tdt", [False, True])
def test_gather_ragged_world2_gloo(tdt):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, tdt, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(res), res


def test_bench_gpus_spawns_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself with
    2 ranks (torch.distributed.run, 127.0.0.1); the reference arm runs on rank 0
    only and prints one JSON line with n_gpus 2, the other rank exits 0."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                          "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "tiny", "--steps", "1", "--warmup", "0", "--cpu-sample", "2"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["cpu_baseline"]["nproc"] >= 1
