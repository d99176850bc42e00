"""Multi-GPU plumbing for batch-sharded decoding.

Utterances are independent (Alg. 1 decodes each utterance on its own,
PAPER.md:56-81), so a large set of utterances is split across ranks with no
data-path collective; the only exchange is gathering the ragged hypotheses at
the end (north_star: "NCCL is used only to gather the ragged results").

* ``length_buckets`` / ``lpt_assign`` / ``rank_shard``: host-side partitioning.
  Utterances are sorted by length and cut into batches of ``batch`` (a batch
  ends with its longest row, so length-sorted batches waste the fewest
  frames); batches go to ranks by LPT greedy (longest processing time first,
  to the least-loaded rank) on the cost max_len(batch).
* ``NcclGather``: the native exchange -- ``ll_gather_ragged`` of the C ABI
  (packing kernels + ncclAllGather of the record sizes + ncclSend/ncclRecv of
  the records to the root) on a libll NCCL communicator whose unique id is
  broadcast over ``torch.distributed``.  ``unpack_records`` parses the root
  buffer.  This is what bench.py's sweep uses on GPUs.
* ``pack_hypotheses`` / ``gather_ragged``: the same record format built with
  torch ops and all-gathered over ``torch.distributed`` -- the host-side model
  of the exchange, exercised with gloo (world size 2) in the CPU tests.

Everything here is plumbing: no step of the decoding method runs in this file.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch


def length_buckets(lengths: Sequence[int], batch: int) -> List[np.ndarray]:
    """Utterance ids sorted by length (stable, ascending) cut into batches."""
    if batch < 1:
        raise ValueError("batch must be >= 1")
    order = np.argsort(np.asarray(lengths), kind="stable")
    return [order[i:i + batch] for i in range(0, len(order), batch)]


def lpt_assign(batches: Sequence[np.ndarray], lengths: Sequence[int], n_ranks: int) -> List[List[int]]:
    """Longest-processing-time-first assignment of batches to ranks; cost of a
    batch = its longest utterance.  Returns, per rank, the batch indices.
    Deterministic (ties broken by batch index, then by rank index)."""
    if n_ranks < 1:
        raise ValueError("n_ranks must be >= 1")
    lengths = np.asarray(lengths)
    cost = [int(lengths[b].max()) if len(b) else 0 for b in batches]
    order = sorted(range(len(batches)), key=lambda i: (-cost[i], i))
    load = [0] * n_ranks
    out: List[List[int]] = [[] for _ in range(n_ranks)]
    for i in order:
        r = min(range(n_ranks), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += cost[i]
    return out


def rank_shard(lengths: Sequence[int], n_ranks: int, rank: int, batch: int = 32) -> np.ndarray:
    """Utterance ids decoded by `rank`, longest first (the decode kernel takes
    groups from a work counter, so long groups start first)."""
    batches = length_buckets(lengths, batch)
    mine = lpt_assign(batches, lengths, n_ranks)[rank]
    ids = np.concatenate([batches[i] for i in mine]) if mine else np.zeros(0, dtype=np.int64)
    lengths = np.asarray(lengths)
    return ids[np.argsort(-lengths[ids], kind="stable")].astype(np.int64)


def pack_hypotheses(ids, lengths, tokens, timestamps, durations=None) -> torch.Tensor:
    """Flat int32 buffer of one rank's results, built on the results' device:
    [n, ids[n], lens[n], tokens(ragged), timestamps(ragged)(, durations(ragged))].
    Each argument is a tensor or a list of tensors (one per decode launch):
    tokens / timestamps / durations are the decoder's [B, cap] outputs, lengths
    its [B] counts (capped at cap), ids the utterance ids of the rows."""
    if isinstance(ids, torch.Tensor):
        ids, lengths, tokens, timestamps = [ids], [lengths], [tokens], [timestamps]
        durations = None if durations is None else [durations]
    dev = tokens[0].device
    lens, fields = [], [[], [], []]
    for k in range(len(ids)):
        n = ids[k].numel()
        ln = lengths[k][:n].to(torch.int64).clamp(max=tokens[k].shape[1])
        mask = torch.arange(tokens[k].shape[1], device=dev)[None, :] < ln[:, None]
        lens.append(ln.to(torch.int32))
        fields[0].append(tokens[k][:n][mask].to(torch.int32))
        fields[1].append(timestamps[k][:n][mask].to(torch.int32))
        if durations is not None:
            fields[2].append(durations[k][:n][mask].to(torch.int32))
    n_tot = sum(int(i.numel()) for i in ids)
    parts = [torch.tensor([n_tot], dtype=torch.int32, device=dev)] + [i.to(device=dev, dtype=torch.int32) for i in ids]
    parts += lens + fields[0] + fields[1] + fields[2]
    return torch.cat(parts)


def unpack_hypotheses(buf: np.ndarray, with_durations: bool) -> Dict[int, Tuple[list, ...]]:
    """Inverse of pack_hypotheses (host side): {utterance id: (tokens,
    timestamps[, durations])}."""
    n = int(buf[0])
    ids = buf[1:1 + n]
    lens = buf[1 + n:1 + 2 * n].astype(np.int64)
    tot = int(lens.sum())
    off = 1 + 2 * n
    fields = [buf[off + k * tot: off + (k + 1) * tot] for k in range(3 if with_durations else 2)]
    starts = np.concatenate([[0], np.cumsum(lens)])
    out = {}
    for i in range(n):
        a, b = starts[i], starts[i + 1]
        out[int(ids[i])] = tuple(f[a:b].tolist() for f in fields)
    return out


def unpack_records(buf: np.ndarray, with_durations: bool) -> Dict[int, Tuple[list, ...]]:
    """Parse a concatenation of records (the root buffer of ll_gather_ragged:
    one record per rank per call) into {utterance id: hypothesis}."""
    nf = 3 if with_durations else 2
    out: Dict[int, Tuple[list, ...]] = {}
    off = 0
    while off < len(buf):
        n = int(buf[off])
        tot = int(buf[off + 1 + n:off + 1 + 2 * n].astype(np.int64).sum())
        size = 1 + 2 * n + nf * tot
        out.update(unpack_hypotheses(buf[off:off + size], with_durations))
        off += size
    return out


class NcclGather:
    """The C-ABI gather (ll_gather_ragged) on one libll NCCL communicator per
    process group.  Collective: construct and call on every rank."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        from . import ll
        self.ll = ll
        init = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if init else 0
        self.world = dist.get_world_size(group) if init else 1
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        uid = b"\0" * 128
        if self.rank == 0:
            st, uid = ll.ll_nccl_unique_id()
            if st != ll.LL_OK:
                raise ll.LLError(st, "ll_nccl_unique_id")
        if self.world > 1:   # share the id (the process group's own backend carries it)
            t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).clone()
            if dist.get_backend(group) == "nccl":
                t = t.to(self.device)
            dist.broadcast(t, 0, group=group)
            uid = bytes(t.cpu().numpy().tobytes())
        st, self.comm = ll.ll_nccl_comm_init(self.world, uid, self.rank)
        if st != ll.LL_OK:
            raise ll.LLError(st, "ll_nccl_comm_init")
        self._ws = torch.empty(0, dtype=torch.uint8, device=self.device)
        self._root = torch.empty(1 << 16, dtype=torch.int32, device=self.device)

    def gather(self, ids, lengths, tokens, timestamps, durations=None, root: int = 0, stream=None):
        """Gather one set of decoded rows (ids/lengths [B], tokens... [B, cap] int32
        device tensors) on `root`.  Returns the root's int32 device buffer
        (records of all ranks in rank order) on root, None elsewhere."""
        ll = self.ll
        B, cap = int(ids.numel()), int(tokens.shape[1])
        need = ll.ll_gather_workspace_size(B, cap, durations is not None)
        if self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        ptr = lambda t: None if t is None else t.data_ptr()
        for _ in range(2):   # at most one retry: LL_ERR_CAPACITY reports the size needed on every rank
            st, used = ll.ll_gather_ragged(self.comm, root, B, ptr(ids), ptr(lengths), ptr(tokens), ptr(timestamps),
                                           ptr(durations), cap, ptr(self._root), self._root.numel(),
                                           ptr(self._ws), self._ws.numel(), s)
            if st != ll.LL_ERR_CAPACITY:
                break
            self._root = torch.empty(max(used, 2 * self._root.numel()), dtype=torch.int32, device=self.device)
        if st != ll.LL_OK:
            raise ll.LLError(st, "ll_gather_ragged")
        return self._root[:used].clone() if self.rank == root else None

    def close(self):
        if self.comm:
            self.ll.ll_nccl_comm_destroy(self.comm)
            self.comm = None


def gather_ragged(packed: torch.Tensor, with_durations: bool, group=None, unpack: bool = True):
    """All-gather every rank's packed buffer (sizes first, then the buffers
    padded to the largest) over torch.distributed.  On rank 0 returns the
    merged {utterance id: hypothesis} (unpack=True) or the list of per-rank
    packed device buffers (unpack=False); None on the other ranks.  Works with
    the NCCL backend (device tensors) and gloo (host tensors)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    size = torch.tensor([packed.numel()], dtype=torch.int64, device=packed.device)
    sizes = [torch.zeros_like(size) for _ in range(world)]
    dist.all_gather(sizes, size, group=group)
    sz = [int(s.item()) for s in sizes]
    pad = torch.zeros(max(sz), dtype=torch.int32, device=packed.device)
    pad[:packed.numel()] = packed
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    if rank != 0:
        return None
    bufs = [b[:n] for n, b in zip(sz, bufs)]
    if not unpack:
        return bufs
    out: Dict[int, Tuple[list, ...]] = {}
    for b in bufs:
        out.update(unpack_hypotheses(b.cpu().numpy(), with_durations))
    return out
