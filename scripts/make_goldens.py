"""Write the full-size parity goldens under tests/golden/ — calls ONLY oracle/ and datagen/.

The GPU parity tests (tests/test_gpu_fullsize.py) compare the CUDA path against these files; the oracle
itself would take hours at these sizes, so its results are computed once here (SURVEY §4.2 T3 sizes,
VERDICT r1 "Next round" item 1):

  sweep_cfg3_sampled.json  configs[2] estimator sweep (n = 1e6, w = 1,024 / 4,096 / 16,384, stride 512),
                           every 25th window of the 5,820-window list for each k in {3, 4, 8}: the full
                           records (mi, h, nmi as float.hex, s_psi, s_log, zero_eps)
  search_cfg4_16pairs.json configs[3] full-size search (n = 1e6, scales 64..16,384, TD+BU, noise on) on
                           the 10 planted pairs + 6 fixed others: result windows and algorithm counters
  search_cfg5_prefix.json  configs[4] on the 1e6-sample prefix: scales 128..65,536, n_p = 4 chunks, TD with
                           noise pruning, pairs (0,1) (planted) and (2,3): results and counters

  python scripts/make_goldens.py [sweep|cfg4|cfg5 ...] [--jobs 8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")

CFG4_EXTRA = [0, 401, 802, 1000, 1203, 1604, 2015]  # fixed pair indices (of the 2,016); planted ones skipped
CFG5_PAIRS = [(0, 1), (2, 3)]
CFG5_PREFIX = 1_000_000
CFG5_CHUNKS = 4


def cfg4_pair_ids():
    import datagen

    wl = datagen.cfg4()
    planted = sorted(wl.planted)
    extra = [p for p in CFG4_EXTRA if p not in planted]
    return sorted(planted + extra)[:16]


def _hex(v):
    return float(v).hex()


def _results_json(res):
    return [[int(r[0]), int(r[1]), int(r[2]), int(r[3]), _hex(r[4]), _hex(r[5]), _hex(r[6])] for r in res]


# ------------------------------------------------------------------ configs[2] sweep sample
def _sweep_k(k):
    import datagen
    import oracle

    wl = datagen.cfg3()
    x, y = wl.series
    W = datagen.sweep_windows(len(x), wl.sweep["sizes"], wl.sweep["stride"])
    sel = list(range(0, len(W), 25))
    r = oracle.mi_batch(x, y, W[sel], k)
    return k, sel, {f: [(_hex(v) if f in ("mi", "h", "nmi") else int(v)) for v in r[f]] for f in r}


def make_sweep(jobs):
    os.environ.setdefault("ORACLE_THREADS", str(max(1, jobs // 3)))
    out = {"what": "configs[2] sweep, every 25th window of the (w = 1024/4096/16384, stride 512) list",
           "source": "oracle.mi_batch (scripts/make_goldens.py)", "per_k": {}}
    with ProcessPoolExecutor(3) as ex:
        for k, sel, rec in ex.map(_sweep_k, [3, 4, 8]):
            out["per_k"][str(k)] = {"index": sel, **rec}
    return out


# ------------------------------------------------------------------ configs[3] 16 pairs
_WL4 = None


def _cfg4_one(pid):
    global _WL4
    import datagen
    import oracle

    if _WL4 is None:
        _WL4 = datagen.cfg4()
    wl = _WL4
    xs, ys = wl.pairs[pid]
    t = time.time()
    res, st = oracle.search(wl.series, [(xs, ys, pid)], oracle.make_params(wl.search))
    return pid, res, st, time.time() - t


def make_cfg4(jobs):
    pids = cfg4_pair_ids()
    out = {"what": "configs[3] full-size search (n = 1e6, 64 series, scales 64..16384, TD+BU, noise on) "
                   "on 16 of the 2,016 pairs (10 planted + 6 fixed)",
           "source": "oracle.search per pair (scripts/make_goldens.py)", "pairs": pids, "per_pair": {}}
    with ProcessPoolExecutor(jobs) as ex:
        for pid, res, st, dt in ex.map(_cfg4_one, pids):
            out["per_pair"][str(pid)] = {"results": _results_json(res), "stats": st, "oracle_s": dt}
            print(f"cfg4 pair {pid}: {len(res)} windows, {dt:.0f} s", flush=True)
    return out


# ------------------------------------------------------------------ configs[4] prefix
_WL5 = None


def _cfg5_one(pair):
    global _WL5
    import datagen
    import oracle

    if _WL5 is None:
        _WL5 = datagen.cfg5()
    wl = _WL5
    series = [s[:CFG5_PREFIX] for s in wl.series]
    pid = wl.pairs.index(pair)
    t = time.time()
    res, st = oracle.search(series, [(pair[0], pair[1], pid)],
                            oracle.make_params(wl.search, n_chunks=CFG5_CHUNKS))
    return pid, res, st, time.time() - t


def make_cfg5(jobs):
    os.environ.setdefault("ORACLE_THREADS", str(max(1, jobs // len(CFG5_PAIRS))))
    out = {"what": f"configs[4] on the [0, {CFG5_PREFIX}) prefix: scales 128..65536, n_p = {CFG5_CHUNKS}, TD with "
                   "noise pruning", "source": "oracle.search per pair (scripts/make_goldens.py)",
           "pairs": CFG5_PAIRS, "prefix": CFG5_PREFIX, "n_chunks": CFG5_CHUNKS, "per_pair": {}}
    with ProcessPoolExecutor(len(CFG5_PAIRS)) as ex:
        for pid, res, st, dt in ex.map(_cfg5_one, CFG5_PAIRS):
            out["per_pair"][str(pid)] = {"results": _results_json(res), "stats": st, "oracle_s": dt}
            print(f"cfg5 pair {pid}: {len(res)} windows, {dt:.0f} s", flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="*", default=["sweep", "cfg4", "cfg5"])
    ap.add_argument("--jobs", type=int, default=os.cpu_count() or 8)
    args = ap.parse_args()
    os.makedirs(GOLD, exist_ok=True)
    makers = {"sweep": ("sweep_cfg3_sampled.json", make_sweep), "cfg4": ("search_cfg4_16pairs.json", make_cfg4),
              "cfg5": ("search_cfg5_prefix.json", make_cfg5)}
    for w in args.which:
        name, fn = makers[w]
        t = time.time()
        out = fn(args.jobs)
        out["wall_s"] = time.time() - t
        with open(os.path.join(GOLD, name), "w") as f:
            json.dump(out, f, separators=(",", ":"))
        print(f"wrote tests/golden/{name} in {out['wall_s']:.0f} s", flush=True)


if __name__ == "__main__":
    main()
