"""Host-time profile of the product search driver on CPU (test infrastructure: oracle-evaluated windows).

  python -m tests.native.prof_driver [--workload cfg2] [--reps 3]

The first run evaluates every requested window with the oracle (OpenMP over the batch) and caches the
records; the timed re-runs replay them, so wall - eval = the driver's own host time per search.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import datagen  # noqa: E402
from native import harness  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=0)
    a = ap.parse_args()
    wl = getattr(datagen, a.workload)(**({"n": a.n} if a.n else {}))
    L = harness.lib()
    L.harness_use_cache(1)
    L.harness_parallel(1)
    t = time.perf_counter()
    res0, st0, ems, ev = harness.search(wl.series, wl.pairs, wl.search)
    print(f"first run {time.perf_counter() - t:.1f} s, evaluated {ev}, results {len(res0)}", flush=True)
    for _ in range(a.reps):
        t = time.perf_counter()
        res, st, ems, ev = harness.search(wl.series, wl.pairs, wl.search)
        wall = (time.perf_counter() - t) * 1e3
        assert res == res0
        print(f"wall {wall:.1f} ms, eval (cache replay) {ems:.1f} ms, driver host {wall - ems:.1f} ms, "
              f"rounds {st['kernel']['rounds']}, windows requested {st['kernel']['windows']}", flush=True)


if __name__ == "__main__":
    main()
