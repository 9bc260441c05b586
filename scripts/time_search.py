"""Device-timed search steps of one workload (tuning sweeps): python scripts/time_search.py cfg2 [reps]."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_2204_09131_b200 as isy

    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    wl, _ = bench.make_workload(name)
    dev = [torch.from_numpy(s).cuda() for s in wl.series]
    ms, res, st = bench.timed_search(isy, wl, dev, None, torch.cuda.current_stream(), reps)
    k = st["kernel"]
    print(json.dumps({"workload": name, "ms": ms, "rounds": k["rounds"], "host_ms": k["host_ms"],
                      "windows": k["windows"], "results": len(res),
                      "env": {e: os.environ[e] for e in os.environ if e.startswith("ISYCOS_")}}), flush=True)


if __name__ == "__main__":
    main()
