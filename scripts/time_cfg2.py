"""configs[1] (cfg2) single-pair search, device-resident series, CUDA-event timed (exploration / traces).

  ISYCOS_TRACE=/tmp/t python scripts/time_cfg2.py [--reps N]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import datagen
    import paper_2204_09131_b200 as isy

    wl = datagen.cfg2()
    dev = [torch.from_numpy(s).cuda() for s in wl.series]
    stream = torch.cuda.current_stream()
    for r in range(args.reps):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record(stream)
        res, st = isy.search_workload(wl, series=dev, stream=stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        k = st["kernel"]
        print(json.dumps({"rep": r, "ms": ev0.elapsed_time(ev1), "results": len(res), "rounds": k["rounds"],
                          "host_ms": k["host_ms"], "windows": k["windows"], "launches": k["launches"]}), flush=True)


if __name__ == "__main__":
    main()
