"""Length-balanced sharding of document pairs across GPUs + record gather.

Documents are independent units (miner.py:158-180) and output order is input
order (miner.py:205-211), so multi-GPU mining is: split the batch into one
shard per rank (LPT over n*m cells plus a per-document overhead), mine each
shard on its own GPU with no collective, then gather the compacted records to
rank 0 (all_gather of counts, gather of fixed-width 24-byte records) and
restore document order there. Over NCCL the gather runs on NVLink/NVSwitch;
the same code runs over gloo for the CPU multi-process tests.
"""

from __future__ import annotations

import heapq

import numpy as np

RECORD_DTYPE = np.dtype([("doc", "<i4"), ("i", "<i4"), ("j", "<i4"), ("pad", "<i4"), ("conf", "<f8")])


def doc_cost(n: np.ndarray, m: np.ndarray, overhead: float = 2000.0) -> np.ndarray:
    """Work estimate of a document: its DP cells plus a fixed per-document term."""
    return n.astype(np.float64) * m.astype(np.float64) + overhead


def lpt_shards(n, m, world: int, overhead: float = 2000.0) -> list[np.ndarray]:
    """Longest-processing-time-first greedy assignment of documents to ranks.

    Deterministic: documents are taken by decreasing cost (ties by index) and
    go to the least-loaded rank (ties by rank id). Each shard is returned in
    input order, so per-rank output stays ordered by document index.
    """
    n = np.asarray(n)
    m = np.asarray(m)
    if world < 1:
        raise ValueError("world must be >= 1")
    cost = doc_cost(n, m, overhead)
    order = np.lexsort((np.arange(cost.size), -cost))
    heap = [(0.0, r) for r in range(world)]
    owner = np.empty(cost.size, dtype=np.int64)
    for d in order:
        load, r = heapq.heappop(heap)
        owner[d] = r
        heapq.heappush(heap, (load + float(cost[d]), r))
    return [np.nonzero(owner == r)[0] for r in range(world)]


def shard_imbalance(shards: list[np.ndarray], n, m, overhead: float = 2000.0) -> float:
    cost = doc_cost(np.asarray(n), np.asarray(m), overhead)
    loads = np.array([cost[s].sum() for s in shards])
    return float(loads.max() / max(loads.mean(), 1e-12))


def restore_order(parts: list[np.ndarray]) -> np.ndarray:
    """Concatenate per-rank records (doc = global index, path order within a
    doc) and order them by document; stable, so path order is kept."""
    allr = np.concatenate(parts) if parts else np.zeros(0, RECORD_DTYPE)
    return allr[np.argsort(allr["doc"], kind="stable")]


def gather_records(recs: np.ndarray, group=None, dst: int = 0, device=None) -> np.ndarray | None:
    """Gather every rank's records (numpy RECORD_DTYPE, doc = global index) on
    rank `dst`, in document order. Returns None on the other ranks."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = device if device is not None else torch.device("cpu")
    raw = np.ascontiguousarray(recs, dtype=RECORD_DTYPE).view(np.uint8)
    count = torch.tensor([recs.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(counts, count, group=group)
    sizes = [int(c.item()) for c in counts]
    width = max(max(sizes), 1) * RECORD_DTYPE.itemsize
    buf = torch.zeros(width, dtype=torch.uint8, device=dev)
    if raw.size:
        buf[: raw.size] = torch.from_numpy(raw).to(dev)
    if rank == dst:
        outs = [torch.zeros(width, dtype=torch.uint8, device=dev) for _ in range(world)]
        dist.gather(buf, outs, dst=dst, group=group)
        parts = [o.cpu().numpy()[: s * RECORD_DTYPE.itemsize].view(RECORD_DTYPE)
                 for o, s in zip(outs, sizes)]
        return restore_order(parts)
    dist.gather(buf, None, dst=dst, group=group)
    return None


def mine_shard(corpus, plex, model, threshold: float, penalty: float, rank: int, world: int,
               swapped=None):
    """Mine this rank's LPT shard of a packed batch on the current GPU; the
    returned records carry global document indices."""
    from . import engine

    shards = lpt_shards(corpus.n, corpus.m, world)
    idx = shards[rank]
    if idx.size == 0:
        return np.zeros(0, RECORD_DTYPE), idx
    dc = engine.DeviceCorpus.upload(corpus)
    dl = engine.DeviceLexicon.upload(plex)
    sw = None if swapped is None else np.asarray(swapped)[idx]
    view = engine.DocView.of(corpus, idx, sw)
    recs, _cost = engine.mine(dc, dl, view, model, threshold, penalty)
    recs = recs.copy()
    recs["doc"] = idx[recs["doc"]]
    return recs, idx


def merge_shards_device(parts, lens, n_docs: int):
    """Rank-0 side of the gather on the device: ``parts`` is a [world, stride, 6]
    int32 CUDA tensor of 24-byte records (doc = global index, each rank's
    records in document order), ``lens`` the int64 CUDA tensor of valid counts.
    Returns the records in global document order as a uint8 CUDA tensor
    (bm_merge_shards)."""
    import torch

    from . import _native as N
    from . import engine

    lib = N.lib()
    world, stride = int(parts.shape[0]), int(parts.shape[1])
    out = torch.empty(max(world * stride, 1) * RECORD_DTYPE.itemsize, dtype=torch.uint8,
                      device=parts.device)
    total = torch.zeros(1, dtype=torch.int64, device=parts.device)
    N.check(lib.bm_merge_shards(engine._ptr(parts), stride, engine._ptr(lens), world, int(n_docs),
                                engine._ptr(out), engine._ptr(total), engine.stream_ptr()))
    return out[: int(total.item()) * RECORD_DTYPE.itemsize]


def reduce_tune_counts(pred, hit, group=None):
    """Sum every rank's per-grid-point (pred, hit) counts (tuner.py:134-145 over
    a dev set split into shards): one all_reduce of a [2, n_pen, n_thr] int64
    tensor -- over NCCL for CUDA tensors, gloo for CPU ones. Returns the summed
    (pred, hit) as numpy arrays on every rank."""
    import torch
    import torch.distributed as dist

    both = torch.stack([torch.as_tensor(pred), torch.as_tensor(hit)]).to(torch.int64)
    if isinstance(pred, torch.Tensor) and pred.is_cuda:
        both = both.to(pred.device)
    dist.all_reduce(both, op=dist.ReduceOp.SUM, group=group)
    out = both.cpu().numpy()
    return out[0], out[1]


def tune_shard(corpus, plex, model, penalties, thresholds, gold_keys, rank: int, world: int,
               group=None):
    """This rank's LPT shard of a dev set through bm_tune, then the counts of all
    ranks summed (reduce_tune_counts over NCCL): every rank returns the whole
    dev set's (pred, hit)."""
    from . import engine

    idx = lpt_shards(corpus.n, corpus.m, world)[rank]
    dev = engine.device()
    import torch

    if idx.size:
        dc = engine.DeviceCorpus.upload(corpus)
        dl = engine.DeviceLexicon.upload(plex)
        view = engine.DocView.of(corpus, idx)
        gold = engine.DeviceGold.of([gold_keys[d] for d in idx])
        pred, hit = engine.tune_counts_device(dc, dl, view, model, penalties, thresholds, gold)
    else:
        pred = torch.zeros((len(penalties), len(thresholds)), dtype=torch.int64, device=dev)
        hit = torch.zeros_like(pred)
    return reduce_tune_counts(pred, hit, group)
