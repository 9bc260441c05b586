"""Small workload that launches every kernel family, for the T5 checks.

compute-sanitizer is closed on the GPU pool (profiles/r02_sanitizer_closed.log), so tests/test_gpu_t5.py
runs this script in subprocesses instead:
  * poisoning: ISYCOS_POISON=<byte> makes every kernel fill its shared memory with the byte first, and the
    engine fill the scan scratch and the record buffers: a read of anything not written in the batch
    (initcheck) or a read racing a write in another warp (racecheck) changes the outputs, so the outputs
    under different poison bytes must be bitwise identical (--dump writes them);
  * repetition: every batch runs --repeat times in-process; any difference is a race / nondeterminism;
  * every output is also compared with the oracle (exit code 1 on any mismatch).

Families: ksg_small (w <= 64), ksg_tile (brute, R = 2/4; latency mode R = 1 for KSG-2), ksg_lat (latency
mode, KSG-1), warp_sorted (dense 65..256), fused_sorted (latency-mode sorted windows), sort_window +
sorted_knn (throughput form, incl. the XL rank merge and the NEXT-3 block sort), KSG-1 and KSG-2, and one
TD+BU search (two batches in flight).
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dump", default="")
    ap.add_argument("--repeat", type=int, default=2)
    args = ap.parse_args()
    import datagen
    import oracle
    import paper_2204_09131_b200 as isy

    wl = datagen.cfg3()
    x, y = (s[:40_000] for s in wl.series)
    bad = 0
    dump = {}

    def check(W, label, **kw):
        nonlocal bad
        W = np.asarray(W, np.int64).reshape(-1, 2)
        for variant in (0, 1):
            ref = oracle.mi_batch(x, y, W, 4, variant=variant)
            first = None
            for rep in range(args.repeat):
                got = isy.isycos_mi_batch_ex(x, y, W, 4, variant=variant, debug=True, **kw)
                cur = {f: np.asarray(got[f]).copy() for f in ("mi", "h", "nmi", "s_psi", "s_log", "zero_eps", "eps",
                                                              "nx", "ny")}
                ok = all(np.array_equal(cur[f], ref[f]) for f in ("mi", "s_psi", "s_log", "zero_eps"))
                if first is None:
                    first = cur
                else:
                    ok = ok and all(np.array_equal(cur[f], first[f]) for f in cur)
                if not ok:
                    print(f"{label} v{variant} rep {rep}: MISMATCH", flush=True)
                    bad += 1
            for f, v in first.items():
                dump[f"{label}_v{variant}_{f}"] = v
            print(f"{label} v{variant}: checked ({len(W)} windows x {args.repeat})", flush=True)

    check(datagen.sweep_windows(4000, [20, 48, 64], 97), "small")
    check([(100, 1100), (3000, 3700)], "tile-brute", brute=True)
    check([(10, 210), (500, 640), (900, 930)], "latency")
    check(datagen.sweep_windows(40_000, [100, 200, 256], 60), "warp_sorted")
    check([(0, 1000), (2000, 4100), (7000, 7300)], "fused")
    check([(0, 9000), (100, 2100)] + [(37 + 256 * i, 37 + 256 * i + 1024) for i in range(6)], "sorted_xl_block",
          unfused=True)
    check([(512 * i, 512 * i + 4096) for i in range(10)], "incremental", unfused=True, incremental=True)
    s = datagen.cfg1()
    ores, ost = oracle.search(s.series, s.pairs, oracle.make_params(s.search))
    for rep in range(args.repeat):
        gres, gst = isy.search_workload(s)
        if gres != ores:
            print(f"search rep {rep}: MISMATCH", flush=True)
            bad += 1
    dump["search"] = np.array([r[2:4] for r in gres], np.int64)
    print(f"search: checked ({len(gres)} windows x {args.repeat})", flush=True)
    if args.dump:
        np.savez(args.dump, **dump)
    print("T5 workload:", "FAIL" if bad else "ok", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
