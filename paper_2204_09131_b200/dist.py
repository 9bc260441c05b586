"""Multi-GPU sharding of the hot path (row a8).

One process per GPU (torchrun), torch.distributed for the plumbing.  Work units are independent
(windows of a sweep, series pairs of a search, (pair, chunk) units of a chunked search), so there
is no data-path collective: each rank evaluates its shard through the C ABI, and ONE all_gather
(NCCL over NVLink on B200; gloo in the CPU tests) collects the fixed-size records at the end.

Results never depend on the number of ranks: a sweep's records are per window, a search's windows
are per pair (LAHC streams are keyed by the pair id, not the rank), and the merged output is sorted
by (pair, method, t0).  The compute callables are injectable so the sharding/gather logic can be
exercised on CPU with gloo (tests pass the oracle); the default is the GPU library (no fallback).
"""
from __future__ import annotations

import heapq

import numpy as np

REC_FIELDS = ("mi", "h", "nmi")


def lpt_assign(costs, world: int):
    """Longest-processing-time-first assignment of units to ranks.  Returns a list of index lists."""
    heap = [(0.0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(v) for v in out]


def interleave_by_class(windows, world: int):
    """Sweep windows -> ranks: interleaved within each window size (cost ~ w^2), so every rank gets
    the same mix of sizes.  Returns a list of index arrays."""
    W = np.asarray(windows, np.int64).reshape(-1, 2)
    sizes = W[:, 1] - W[:, 0]
    out = [[] for _ in range(world)]
    for s in np.unique(sizes):
        idx = np.flatnonzero(sizes == s)
        for r in range(world):
            out[r].extend(idx[r::world].tolist())
    return [np.asarray(sorted(v), np.int64) for v in out]


def pair_cost(n: int, s_max: int, s_min: int) -> float:
    """w^2-weighted cost proxy of a pair's top-down search (first layers dominate)."""
    c, s = 0.0, s_max
    while s >= s_min:
        c += 4.0 * n / s * s * s
        s //= 2
    return c


def _all_gather_variable(t, group=None):
    """all_gather of a 2-D tensor whose first dimension differs per rank (pad + trim)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(v.item()) for v in ns]
    m = max(ns) if ns else 0
    pad = torch.zeros((m, t.shape[1]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    outs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return [o[:k] for o, k in zip(outs, ns)]


def _gpu_mi_batch(x, y, windows, k):
    from . import isycos_mi_batch_ex

    r = isycos_mi_batch_ex(x, y, windows, k, outputs=REC_FIELDS)
    return {f: np.asarray(r[f].cpu() if hasattr(r[f], "cpu") else r[f], np.float64) for f in REC_FIELDS}


def sweep_sharded(x, y, windows, k: int, *, mi_batch=None, device=None):
    """Evaluate `windows` of (x, y) sharded over the process group; every rank returns all records
    (dict of float64 arrays in the input order)."""
    import torch
    import torch.distributed as dist

    mi_batch = mi_batch or _gpu_mi_batch
    world, rank = dist.get_world_size(), dist.get_rank()
    W = np.asarray(windows, np.int64).reshape(-1, 2)
    mine = interleave_by_class(W, world)[rank]
    rec = mi_batch(x, y, W[mine], k) if len(mine) else {f: np.zeros(0) for f in REC_FIELDS}
    dev = device or ("cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu")
    payload = np.zeros((len(mine), 1 + len(REC_FIELDS)), np.float64)
    payload[:, 0] = mine
    for j, f in enumerate(REC_FIELDS):
        payload[:, 1 + j] = rec[f]
    parts = _all_gather_variable(torch.from_numpy(payload).to(dev))
    out = {f: np.empty(len(W)) for f in REC_FIELDS}
    for p in parts:
        p = p.cpu().numpy()
        idx = p[:, 0].astype(np.int64)
        for j, f in enumerate(REC_FIELDS):
            out[f][idx] = p[:, 1 + j]
    return out


def _gpu_search(series, pairs, **kw):
    from . import isycos_search

    return isycos_search(series, pairs, **kw)


def _gpu_merge(results):
    from . import isycos_merge_windows

    return isycos_merge_windows(results)


def chunk_plan(n: int, n_p: int, s_max: int):
    """Alg. 4 line 14, clipped: chunk c = [max(0, cL - s_max), min(n, (c+1)L)), L = ceil(n / n_p)."""
    L = -(-n // n_p)
    return [(max(0, c * L - s_max), min(n, (c + 1) * L)) for c in range(n_p) if c * L < n]


STAT_NAMES = ["td_windows", "td_noise_checks", "td_skips", "td_accepted", "bu_climbs", "bu_iterations",
              "bu_neighbors", "bu_noise_checks", "bu_prunes", "bu_accepted", "distinct_windows",
              "distinct_pairs", "eval_cost", "auto_td", "auto_bu"]
FSTAT_NAMES = ["auto_nscore_td", "auto_nscore_bu"]  # sums over pairs (rank order: not bitwise)


def shard_units(n: int, pairs, units: str, world: int, *, n_chunks: int = 1, s_min: int = 64,
                s_max: int = 512):
    """Work units and their LPT assignment.  units = "pair": one unit per pair, cost = the w^2-weighted
    first-layer proxy (equal for equal-length pairs -> round robin); "pair_chunk": one unit per (pair,
    chunk) of the Alg. 4 plan, cost proportional to the chunk length.  Returns per rank a list of calls
    (pair indices, chunk range or None)."""
    if units == "pair":
        cost = [pair_cost(n, s_max, s_min)] * len(pairs)
        return [[(idx, None)] if idx else [] for idx in lpt_assign(cost, world)]
    plan = chunk_plan(n, max(1, n_chunks), s_max)
    us = [(p, c) for p in range(len(pairs)) for c in range(len(plan))]
    cost = [pair_cost(plan[c][1] - plan[c][0], s_max, s_min) for (_, c) in us]
    out = []
    for idx in lpt_assign(cost, world):
        by_chunk = {}
        for i in idx:
            p, c = us[i]
            by_chunk.setdefault(c, []).append(p)
        out.append([(ps, (c, c + 1)) for c, ps in sorted(by_chunk.items())])  # one call per chunk index
    return out


def search_sharded(series, pairs, *, search=None, merge=None, device=None, units: str = "pair", **kw):
    """SYCOS search over `pairs` sharded over the process group by work unit (shard_units); one NCCL
    all_gather of the result windows (plus one of the counters); every rank returns the merged result list
    sorted by (pair, method, t0) and the summed algorithm counters (+ this rank's kernel stats under
    "kernel" when the compute reports them).  Results never depend on the number of ranks: pair ids key the
    LAHC streams and (pair, chunk) units are independent searches merged by isycos_merge_windows (Alg. 4).
    With (pair, chunk) units distinct_windows / distinct_pairs / eval_cost count per unit (a window in the
    overlap of two chunks counts once per chunk)."""
    import torch
    import torch.distributed as dist

    search = search or _gpu_search
    merge = merge or _gpu_merge
    world, rank = dist.get_world_size(), dist.get_rank()
    n = len(series[0])
    pairs = [tuple(p) if len(p) > 2 else (p[0], p[1], i) for i, p in enumerate(pairs)]
    calls = shard_units(n, pairs, units, world, n_chunks=kw.get("n_chunks", 1), s_min=kw.get("s_min", 64),
                        s_max=kw.get("s_max", 512))[rank]
    res, st, kern = [], {}, {}
    for idx, chunks in calls:
        ckw = dict(kw)
        if chunks is not None:
            ckw["chunks"] = chunks
        r, s = search(series, [pairs[i] for i in idx], **ckw)
        res += r
        for k_, v in s.items():
            if k_ == "kernel":
                for f, x in v.items():
                    kern[f] = kern.get(f, 0) + x
            else:
                st[k_] = st.get(k_, 0) + v
    dev = device or ("cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu")
    payload = np.array([[r[0], r[1], r[2], r[3], r[4], r[5], r[6]] for r in res], np.float64).reshape(-1, 7)
    parts = _all_gather_variable(torch.from_numpy(payload).to(dev))
    merged = []
    for p in parts:
        for row in p.cpu().numpy():
            merged.append((int(row[0]), int(row[1]), int(row[2]), int(row[3]), float(row[4]), float(row[5]),
                           float(row[6])))
    if units == "pair_chunk":
        merged = merge(merged)
    merged.sort(key=lambda r: (r[0], r[1], r[2]))
    vec = torch.tensor([int(st.get(k, 0)) for k in STAT_NAMES], dtype=torch.int64, device=dev)
    fvec = torch.tensor([float(st.get(k, 0.0)) for k in FSTAT_NAMES], dtype=torch.float64, device=dev)
    dist.all_reduce(vec)
    dist.all_reduce(fvec)
    out = {k: int(v) for k, v in zip(STAT_NAMES, vec.cpu().tolist())}
    out.update({k: float(v) for k, v in zip(FSTAT_NAMES, fvec.cpu().tolist())})
    if kern:
        out["kernel"] = kern
    return merged, out
