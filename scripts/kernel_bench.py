#!/usr/bin/env python
"""Per-size-class throughput of the KSG window kernels (isycos_mi_batch_ex, device-resident inputs).

Prints one JSON line per (w, k): windows, kernel time (CUDA events around every KSG launch,
ISYCOS_F_PROFILE), Tcompare/s (2 w (w-1) compares per window) and the fraction of the issue-bound
roofline.  Used for kernel tuning and ncu captures (--only W to run one class).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", type=int, default=0)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--target", type=float, default=4e11, help="compares per launch set")
    args = ap.parse_args()
    import torch

    import datagen
    import paper_2204_09131_b200 as isy
    from bench import peak_compares

    wl = datagen.cfg3()
    x = torch.from_numpy(wl.series[0]).cuda()
    y = torch.from_numpy(wl.series[1]).cuda()
    n = x.numel()
    sizes = [32, 64, 128, 256, 512, 1024, 4096, 16384]
    if args.only:
        sizes = [args.only]
    peak = peak_compares(1965.0)
    for w in sizes:
        per = 2.0 * w * (w - 1)
        nw = int(min(max(args.target / per, 148), 400_000))
        stride = max(1, (n - w) // nw)
        t0 = np.arange(nw, dtype=np.int64) * stride % (n - w)
        W = np.stack([t0, t0 + w], 1)
        isy.isycos_mi_batch_ex(x, y, W, args.k, outputs=("mi",))  # warm (tables, buffers)
        best = None
        for _ in range(args.reps):
            r = isy.isycos_mi_batch_ex(x, y, W, args.k, outputs=("mi",), profile=True)
            ms = r["stats"]["kernel_ms"]
            if best is None or ms < best:
                best, st = ms, r["stats"]
        rate = nw * per / (best / 1e3)
        out = {"w": w, "k": args.k, "windows": nw, "kernel_ms": best, "Tcompare_s": rate / 1e12,
               "frac_of_bruteforce_roofline": rate / peak, "sorted_windows": st["sorted_windows"]}
        if st["scan_steps"]:
            out["scan_steps_per_point"] = st["scan_steps"] / max(1, st["sorted_points"])
            out["Gsteps_s"] = st["scan_steps"] / (best / 1e3) / 1e9
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
