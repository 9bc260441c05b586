"""Small workload that launches every kernel family once, for compute-sanitizer.

  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python scripts/sanitize_workload.py

Families: ksg_small (w <= 64), ksg_tile (brute, R = 2/4; latency mode R = 1), warp_sorted (dense 65..256),
fused_sorted (latency-mode sorted windows), sort_window + sorted_knn (throughput form, incl. the XL
rank merge and the NEXT-3 block sort), KSG-1 and KSG-2, and one TD+BU search (two batches in flight).
Exits non-zero if any result differs from the oracle.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import datagen
    import oracle
    import paper_2204_09131_b200 as isy

    wl = datagen.cfg3()
    x, y = (s[:40_000] for s in wl.series)
    bad = 0

    def check(W, label, **kw):
        nonlocal bad
        W = np.asarray(W, np.int64).reshape(-1, 2)
        for variant in (0, 1):
            got = isy.isycos_mi_batch_ex(x, y, W, 4, variant=variant, **kw)
            ref = oracle.mi_batch(x, y, W, 4, variant=variant)
            ok = all(np.array_equal(np.asarray(got[f]), ref[f]) for f in ("mi", "s_psi", "s_log", "zero_eps"))
            print(f"{label} v{variant}: {'ok' if ok else 'MISMATCH'} ({len(W)} windows)", flush=True)
            bad += not ok

    check(datagen.sweep_windows(4000, [20, 48, 64], 97), "small")
    check([(100, 1100), (3000, 3700)], "tile-brute", brute=True)
    check([(10, 210), (500, 640)], "tile-latency")
    check(datagen.sweep_windows(40_000, [100, 200, 256], 60), "warp_sorted")
    check([(0, 1000), (2000, 4100), (7000, 7300)], "fused")
    check([(0, 9000), (100, 2100)] + [(37 + 256 * i, 37 + 256 * i + 1024) for i in range(6)], "sorted+xl+block",
          unfused=True)
    s = datagen.cfg1()
    gres, gst = isy.search_workload(s)
    ores, ost = oracle.search(s.series, s.pairs, oracle.make_params(s.search))
    ok = gres == ores
    print(f"search: {'ok' if ok else 'MISMATCH'} ({len(gres)} windows, {gst['kernel']['rounds']} rounds)", flush=True)
    bad += not ok
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
