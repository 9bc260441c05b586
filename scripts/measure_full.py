"""Full-size configs[3] / configs[4] searches on one GPU (exploration + the bench side lines).

  python scripts/measure_full.py cfg4 [--pairs N] [--noise 0|1] [--method M]
  python scripts/measure_full.py cfg5 [--pairs N] [--noise 0|1]

Prints one JSON line per run: device-timed ms, results, counters, kernel stats.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", choices=["cfg4", "cfg5"])
    ap.add_argument("--pairs", type=int, default=0)
    ap.add_argument("--noise", type=int, default=-1)
    ap.add_argument("--method", type=int, default=0)
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    import torch

    import datagen
    import paper_2204_09131_b200 as isy

    t = time.time()
    wl = datagen.cfg4() if args.cfg == "cfg4" else datagen.cfg5()
    gen_s = time.time() - t
    pairs = wl.pairs[: args.pairs] if args.pairs else wl.pairs
    dev = [torch.from_numpy(s).cuda() for s in wl.series]
    kw = {}
    if args.noise >= 0:
        kw["noise"] = bool(args.noise)
    if args.method:
        kw["method"] = args.method
    stream = torch.cuda.current_stream()
    for r in range(args.reps):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w0 = time.time()
        ev0.record(stream)
        res, st = isy.search_workload(wl, series=dev, pairs=pairs, stream=stream, **kw)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        k = st.pop("kernel")
        print(json.dumps({"cfg": args.cfg, "pairs": len(pairs), "rep": r, "gen_s": gen_s, "ms": ms,
                          "wall_s": time.time() - w0, "results": len(res), "stats": st, "kernel": k,
                          "brute_eq_compares_per_s": 2.0 * st["distinct_pairs"] / (ms / 1e3),
                          **kw}), flush=True)


if __name__ == "__main__":
    main()
