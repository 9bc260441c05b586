#!/usr/bin/env python
"""bench.py — throughput of the iSYCOS hot path on B200 (the driver's contract).

A step = one pass of the whole hot path over one batch of synthetic input.  The
default workload is BASELINE.json configs[3] ("cfg4", the largest single-GPU configuration): 64 sensor-like
series of n = 1,000,000 float32 samples, all 2,016 pairs through the full SYCOS_TD + SYCOS_BU search with
MI-based noise pruning, k = 4, scales 64..16,384.  A step searches one batch of `--pairs-per-gpu` pairs per
GPU (default 64); successive steps take successive batches of the 2,016-pair list (the whole job is
2,016 / (64 N) steps).  Series are resident in HBM; the batch runs through the C ABI (isycos_search), and at
N > 1 through dist.search_sharded (pairs sharded by LPT, one NCCL all_gather of the result windows inside
the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload cfg4|cfg2|cfg5|cfg3] [--pairs-per-gpu B] [--no-side] [--no-cpu-baseline]

Metric (BASELINE.json): KSG window compares/s, counting 2*w*(w-1) brute-force-equivalent compares
(w(w-1) joint-distance + w(w-1) marginal compares) for every distinct window the searches consumed;
windows/s beside it.  Weak scaling: every GPU searches B pairs per step; value = all ranks' compares / the
max over ranks of the device-timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# issue-bound compare roofline: 148 SM x 4 SMSP x 32 lanes x 1 warp-instr/clk at
# clocks.max.sm = 1965 MHz = 3.72e13 lane-instr/s; >= 5 lane instructions per compare.
SMS, SMSP, LANES = 148, 4, 32
INSTR_PER_COMPARE = 5.0
REF_PREFIX = 20_000  # oracle sample: prefix of every series of the sampled pairs (>= s_max = 16,384)


def peak_compares(sm_mhz: float) -> float:
    return SMS * SMSP * LANES * sm_mhz * 1e6 / INSTR_PER_COMPARE


# ----------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str | None):
        self.gpu_id = gpu_id
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")

    def start(self):
        cmd = ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200"]
        if self.gpu_id:
            cmd += ["-i", self.gpu_id]
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(cmd, stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------------------- workloads
def make_workload(name: str):
    import datagen

    if name == "cfg4":
        wl = datagen.cfg4()
        desc = {"workload": "configs[3] (cfg4): 64 series x 1,000,000 f32, 2,016 pairs, full TD+BU search",
                "n": 1_000_000, "series": 64, "pairs": 2016, "k": 4, "scales": "64..16384 (TD halving)",
                "method": "TD+BU", "noise_pruning": True, "sigma": 0.2, "tau_ratio": 0.25}
    elif name == "cfg2":
        wl = datagen.cfg2()
        desc = {"workload": "configs[1] (cfg2): one pair, n = 100,000, full TD+BU search", "n": 100_000,
                "pairs": 1, "k": 4, "scales": "32..4096 (TD halving)", "method": "TD+BU", "noise_pruning": True,
                "sigma": 0.2, "tau_ratio": 0.25}
    elif name == "cfg5":
        wl = datagen.cfg5()
        desc = {"workload": "configs[4] (cfg5): 16 series x 10,000,000 f32, 120 pairs, TD + noise pruning, "
                            "16 chunks per pair", "n": 10_000_000, "series": 16, "pairs": 120, "k": 4,
                "scales": "128..65536", "method": "TD", "noise_pruning": True, "n_chunks": 16}
    elif name == "cfg1":
        wl = datagen.cfg1()
        desc = {"workload": "configs[0] (cfg1)", "n": 2048, "pairs": 1, "k": 4, "scales": "64..512",
                "method": "TD+BU", "noise_pruning": True}
    else:
        raise SystemExit(f"unknown workload {name}")
    return wl, desc


def batch_pairs(wl, step: int, per_gpu: int, world: int):
    """Pairs (xs, ys, global pair index) of global step `step`: world * per_gpu consecutive pairs of the
    workload's pair list (cyclic), so successive steps cover the whole job."""
    P = len(wl.pairs)
    B = min(P, per_gpu * world)
    return [(*wl.pairs[(step * B + i) % P], (step * B + i) % P) for i in range(B)]


def traffic_for(path):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(path)
        return t["bytes_per_launch"] if isinstance(t, dict) else t
    except Exception:
        return None


def issue_for(key):
    try:
        with open(os.path.join(ROOT, "profiles", "issue.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def compares_of(stats):
    # 2 * sum w(w-1) over the distinct windows the search consumed (brute-force-equivalent compares)
    return 2.0 * stats["distinct_pairs"]


def search_kw(wl, **over):
    sc = wl.search
    kw = dict(s_min=sc.s_min, s_max=sc.s_max, k=sc.k, sizes=list(sc.sizes) or None, noise=sc.noise,
              tau_ratio=sc.tau_ratio, p=sc.p, sigma=sc.sigma, method=sc.method, delta_td=sc.delta_td,
              delta_bu=sc.delta_bu, t_max_idle=sc.t_max_idle, h=sc.h, n_chunks=sc.n_chunks, seed=sc.seed)
    kw.update(over)
    return kw


# ----------------------------------------------------------------------------------------- the oracle
def _oracle_pair(args):
    """One oracle search (subprocess worker): pair (xs, ys, id) on the series prefix [0, prefix)."""
    name, pair, prefix, over = args
    import oracle

    wl, _ = make_workload(name)
    series = [s[:prefix] for s in wl.series]
    t = time.perf_counter()
    res, st = oracle.search(series, [pair], oracle.make_params(wl.search, **over))
    return time.perf_counter() - t, compares_of(st), st["distinct_windows"], len(res)


def oracle_sample(name: str, pairs, prefix: int, cores: int, over=None):
    """The oracle as it stands (plain single-threaded C++), one process per host core, each running the full
    search of one pair on a series prefix; returns the aggregate throughput over the wall time."""
    from concurrent.futures import ProcessPoolExecutor

    t = time.perf_counter()
    with ProcessPoolExecutor(cores) as ex:
        outs = list(ex.map(_oracle_pair, [(name, p, prefix, over or {}) for p in pairs]))
    wall = time.perf_counter() - t
    comps = sum(o[1] for o in outs)
    wins = sum(o[2] for o in outs)
    return {"wall_s": wall, "compares": comps, "windows": wins, "cpu_s": sum(o[0] for o in outs),
            "value": comps / wall, "windows_per_s": wins / wall}


def cpu_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return os.cpu_count() or 1, model


def oracle_sample_desc(name, prefix, n_pairs, cores, model, wl_n):
    return (f"{n_pairs} pairs of the step's batch, one per host core ({cores} cores, {model}), each the full "
            f"search with the same parameters on the series prefix [0, {prefix}) ({prefix / wl_n:.1%} of n); "
            f"throughput = their brute-force-equivalent compares / wall time")


def run_reference(args, rank, world):
    """The base contract's reference arm for this tier: the oracle (no upstream code exists; BASELINE.json
    'published' is empty), timed on the host cores, on our arm's config/metric; each step a bounded sample
    (nproc pairs of the step's batch on a series prefix)."""
    if rank != 0:
        return 0
    wl, desc = make_workload(args.workload)
    cores, model = cpu_info()
    n = len(wl.series[0])
    prefix = min(n, REF_PREFIX) if args.workload in ("cfg4", "cfg5") else min(n, 25_000)
    over = {"n_chunks": 1} if args.workload == "cfg5" else {}
    if args.workload == "cfg5":
        prefix = min(n, 131_072)
    times, comps, wins = [], 0.0, 0
    for i in range(args.warmup + args.steps):
        pairs = batch_pairs(wl, i, cores, 1)[:cores]
        o = oracle_sample(args.workload, pairs, prefix, cores, over)
        if i >= args.warmup:
            times.append(o["wall_s"])
            comps += o["compares"]
            wins += o["windows"]
    tot = sum(times)
    value = comps / tot
    sample = oracle_sample_desc(args.workload, prefix, cores, cores, model, n)
    line = {
        "impl": "reference", "metric": "KSG window compares/s", "value": value, "unit": "compares/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_of(desc, args, world), "windows_per_s": wins / tot,
        "cpu_baseline": {"value": value, "unit": "compares/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "compares/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_of(desc, args, world):
    c = dict(desc)
    if args.workload in ("cfg4", "cfg5"):
        c["pairs_per_gpu_per_step"] = args.pairs_per_gpu
        c["global_batch_pairs"] = args.pairs_per_gpu * world
    c["l2"] = "flushed between steps (256 MiB write)"
    c["parallelism"] = (f"dp{world}: pairs sharded by LPT, one NCCL all_gather per step" if world > 1 and
                        args.workload != "cfg2" else (f"replicas x{world}" if world > 1 else "1 GPU"))
    return c


# ----------------------------------------------------------------------------------------- side lines
def sweep_cfg3(isy, stream, reps: int):
    """configs[2] estimator sweep (5,820 windows x k in {3,4,8} = 17,460 window evaluations, w = 1,024 /
    4,096 / 16,384, stride 512) through isycos_mi_batch_ex with device-resident series and windows: the
    throughput form of the kernels.  Timed with CUDA events after one warm-up pass."""
    import torch

    import datagen

    wl = datagen.cfg3()
    dx, dy = (torch.from_numpy(s).cuda() for s in wl.series)
    W = datagen.sweep_windows(len(wl.series[0]), wl.sweep["sizes"], wl.sweep["stride"])
    dW = torch.from_numpy(W).cuda()
    out = {"mi": torch.empty(len(W), dtype=torch.float64, device="cuda")}
    ks = wl.sweep["ks"]
    bf = 2.0 * float(((W[:, 1] - W[:, 0]) * (W[:, 1] - W[:, 0] - 1)).sum()) * len(ks)

    def one(profile):
        agg = {}
        for k in ks:
            r = isy.isycos_mi_batch_ex(dx, dy, dW, k, outputs=("mi",), out=out, stream=stream, profile=profile)
            for f, v in r["stats"].items():
                agg[f] = agg.get(f, 0) + v
        return agg

    one(False)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    st = {}
    for _ in range(reps):
        for f, v in one(True).items():
            st[f] = st.get(f, 0) + v
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    peak = peak_compares(1965.0)
    alg = (st["prof_scan_steps"] + st["prof_search_probes"]) / reps
    kms = st["sorted_kernel_ms"] / reps
    return {"workload": f"configs[2] sweep: {len(W)} windows x k in {{3,4,8}} = {len(W) * len(ks)} window "
                        "evaluations per step",
            "ms_per_step": ms, "windows_per_s": len(W) * len(ks) / (ms / 1e3),
            "bruteforce_equivalent_compares_per_s": bf / (ms / 1e3),
            "roofline": {"bound": "alu", "kernel": "sorted-marginal throughput path (sort + scan)",
                         "achieved": alg / (kms / 1e3) / 1e12 if kms else None, "peak": peak / 1e12,
                         "unit": "Tcompare/s", "frac": alg / (kms / 1e3) / peak if kms else None,
                         "kernel_share_of_step": kms / ms if ms else None,
                         "ncu_issue": issue_for("sorted_throughput"),
                         "algorithmic_compares_per_step": alg,
                         "scan_steps_per_point": st["scan_steps"] / max(1, st["sorted_points"])}}


def timed_search(isy, wl, series, pairs, stream, reps, **kw):
    import torch

    isy.search_workload(wl, series=series, pairs=pairs, stream=stream, **kw)  # warm
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(reps):
        res, st = isy.search_workload(wl, series=series, pairs=pairs, stream=stream, **kw)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    return ms, res, st


def noise_protocol(isy, wl, series, pairs, stream, reps):
    """The paper's Origin-vs-Noise protocol (Figs. 6-7): the same search with MI-based noise
    pruning on and off — device time, MI evaluations consumed, distinct windows, compares."""
    out = {}
    for name, noise in (("noise_on", True), ("noise_off", False)):
        ms, res, st = timed_search(isy, wl, series, pairs, stream, reps, noise=noise)
        out[name] = {"ms_per_step": ms, "results": len(res), "td_windows": st["td_windows"],
                     "td_skips": st["td_skips"], "bu_iterations": st["bu_iterations"], "bu_prunes": st["bu_prunes"],
                     "distinct_windows": st["distinct_windows"], "compares": compares_of(st),
                     "compares_per_s": compares_of(st) / (ms / 1e3)}
    out["speedup_noise_on"] = out["noise_off"]["ms_per_step"] / out["noise_on"]["ms_per_step"]
    return out


def side_configs1(isy, stream, reps):
    import torch

    wl, desc = make_workload("cfg2")
    dev = [torch.from_numpy(s).cuda() for s in wl.series]
    ms, res, st = timed_search(isy, wl, dev, None, stream, reps, profile=True)
    k = st["kernel"]
    return {"workload": desc, "ms_per_step": ms, "compares_per_s": compares_of(st) / (ms / 1e3),
            "windows_per_s": st["distinct_windows"] / (ms / 1e3), "results": len(res), "rounds": k["rounds"],
            "host_ms": k["host_ms"],
            "noise_protocol": noise_protocol(isy, wl, dev, None, stream, reps)}


def side_configs4(isy, stream, n_pairs):
    import torch

    wl, desc = make_workload("cfg5")
    dev = [torch.from_numpy(s).cuda() for s in wl.series]
    pairs = [(*wl.pairs[i], i) for i in range(n_pairs)]
    out = {"workload": dict(desc, pairs_timed=n_pairs)}
    out.update(noise_protocol(isy, wl, dev, pairs, stream, 1))
    return out


# ----------------------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=["cfg4", "cfg2", "cfg5", "cfg1"])
    ap.add_argument("--pairs-per-gpu", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-side", action="store_true", help="skip the configs[1]/[2]/[4] side lines")
    ap.add_argument("--cfg5-pairs", type=int, default=8)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)
    # kernel timing samples every 8th search round (CUDA event records are host time on every round)
    os.environ.setdefault("ISYCOS_PROFILE_EVERY", "8")
    if world > 1:  # the search driver's host pool: share the box's cores between the ranks on it
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        os.environ.setdefault("ISYCOS_HOST_THREADS", str(max(2, min(16, (os.cpu_count() or 16) // local_world))))

    import torch

    # ISYCOS_BENCH_DRYRUN=1: a code-path check of the N > 1 flow on a box with fewer GPUs than ranks (ranks share
    # a GPU, gloo on the host for the collectives; the ranks' kernels never wait on one another).  Its line is
    # marked "dry_run" and is never a scaling number.
    dry_run = world > 1 and os.environ.get("ISYCOS_BENCH_DRYRUN") == "1"
    if dry_run:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if dry_run:
            dist.init_process_group("gloo")
        else:
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks) in the log
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2204_09131_b200 import build

    if rank == 0:
        build.build()
    if dist:
        dist.barrier()
    import paper_2204_09131_b200 as isy
    from paper_2204_09131_b200 import dist as idist

    wl, desc = make_workload(args.workload)
    stream = torch.cuda.current_stream()
    dev_series = [torch.from_numpy(s).cuda() for s in wl.series]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    multi_pair = args.workload in ("cfg4", "cfg5")
    step_no = [0]

    def step(series, profile=True, only=None):
        kw = search_kw(wl, profile=profile, profile_only=only, stream=stream)
        if not multi_pair:  # single-pair search: replicas only
            return isy.isycos_search(series, wl.pairs, **kw)
        pairs = batch_pairs(wl, step_no[0], args.pairs_per_gpu, world)
        step_no[0] += 1
        if dist:
            return idist.search_sharded(series, pairs, units="pair", **kw)
        return isy.isycos_search(series, pairs, **kw)

    def sync_all():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        flush.zero_()
        _, wst = step(dev_series)
    torch.cuda.synchronize()
    # the dominant kernel path: larger kernel time in the last warm-up step (every launch group timed); the
    # timed steps record CUDA events around that path's launches only
    warm_k = wst["kernel"]
    dom_path = "sorted_marginal" if warm_k["sorted_kernel_ms"] >= warm_k["brute_kernel_ms"] else "brute_force"
    only = "sorted" if dom_path == "sorted_marginal" else "brute"

    props = torch.cuda.get_device_properties(local)
    try:
        gpu_id = str(props.uuid) if str(props.uuid).startswith("GPU-") else "GPU-" + str(props.uuid)
    except Exception:
        gpu_id = None
    sampler = ClockSampler(gpu_id)
    sampler.start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ms_total, comps, wins, kpairs, launches, ksg_launches, rounds = 0.0, 0.0, 0, 0, 0, 0, 0
    host_ms = wall_ms = 0.0
    kk = {}
    results = 0
    for i in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (256 MiB > 126 MB L2)
        sync_all()
        if i == 0:  # the first timed step is an NVTX range: `ncu --nvtx --nvtx-include timed_step/` lists its launches
            torch.cuda.nvtx.range_push("timed_step")
        ev0.record(stream)
        res, st = step(dev_series, only=only)
        ev1.record(stream)
        if i == 0:
            torch.cuda.nvtx.range_pop()
        sync_all()
        ms_total += ev0.elapsed_time(ev1)
        comps += compares_of(st)        # global (search_sharded all-reduces the counters)
        wins += st["distinct_windows"]
        results += len(res)
        k = st.get("kernel", {})        # this rank's kernel stats
        kpairs += k.get("point_pairs", 0)
        for f in ("sorted_kernel_ms", "brute_kernel_ms", "scan_steps", "search_probes", "brute_point_pairs",
                  "sorted_windows", "windows", "profiled_rounds", "prof_brute_point_pairs", "prof_scan_steps",
                  "prof_search_probes", "h2d_bytes", "d2h_bytes"):
            kk[f] = kk.get(f, 0) + k.get(f, 0)
        launches += k.get("launches", 0)
        ksg_launches += k.get("ksg_launches", 0)
        rounds += k.get("rounds", 0)
        host_ms += k.get("host_ms", 0.0)
        wall_ms += k.get("wall_ms", 0.0)
    clocks = sampler.stop()

    # end to end: pinned host series through the public API, H2D of the series inside the timed region,
    # the result windows read back to the host
    host_series = [torch.from_numpy(s).pin_memory() for s in wl.series]
    e2e_ms, e2e_comps, h2d, d2h = 0.0, 0.0, 0, 0
    for _ in range(args.steps):
        flush.zero_()
        sync_all()
        ev0.record(stream)
        res, st = step(host_series, profile=False)
        ev1.record(stream)
        sync_all()
        e2e_ms += ev0.elapsed_time(ev1)
        e2e_comps += compares_of(st)
        k = st.get("kernel", {})
        h2d += k.get("h2d_bytes", 0)
        d2h += k.get("d2h_bytes", 0) + len(res) * 48

    def agg(v, op):
        if not dist:
            return v
        t = torch.tensor([float(v)], dtype=torch.float64, device="cpu" if dry_run else "cuda")
        dist.all_reduce(t, op=op)
        return t.item()

    import torch.distributed as tdist

    ms_max = agg(ms_total, tdist.ReduceOp.MAX)
    e2e_max = agg(e2e_ms, tdist.ReduceOp.MAX)
    if not multi_pair and dist:  # replicas: every rank's own counters
        comps = agg(comps, tdist.ReduceOp.SUM)
        wins = agg(wins, tdist.ReduceOp.SUM)
        e2e_comps = agg(e2e_comps, tdist.ReduceOp.SUM)
    launches_all = agg(launches, tdist.ReduceOp.SUM)
    h2d_all = agg(h2d, tdist.ReduceOp.SUM)
    d2h_all = agg(d2h, tdist.ReduceOp.SUM)

    if rank == 0:
        value = comps / (ms_max / 1e3)
        peak = peak_compares(1965.0)
        # per path: the sorted-marginal kernels' algorithmic work = scan candidate checks + binary-search
        # probes; the brute-force kernels' = 2 w (w-1) compares per window.  Dominant = larger kernel time.
        paths = {
            "sorted_marginal": {"kernel_ms": kk.get("sorted_kernel_ms", 0.0),
                                "compares": kk.get("prof_scan_steps", 0) + kk.get("prof_search_probes", 0),
                                "kernel": "fused_sorted_kernel / warp_sorted_kernel / sort_window_kernel + "
                                          "sorted_knn_kernel (+ rank_merge_kernel)"},
            "brute_force": {"kernel_ms": kk.get("brute_kernel_ms", 0.0),
                            "compares": 2.0 * kk.get("prof_brute_point_pairs", 0),
                            "kernel": "ksg_small_kernel + ksg_tile_kernel"},
        }
        other = "brute_force" if dom_path == "sorted_marginal" else "sorted_marginal"
        paths[other]["kernel_ms"] = warm_k["brute_kernel_ms" if other == "brute_force" else "sorted_kernel_ms"]
        paths[other]["compares"] = (2.0 * warm_k["prof_brute_point_pairs"] if other == "brute_force"
                                    else warm_k["prof_scan_steps"] + warm_k["prof_search_probes"])
        paths[other]["timed_in"] = "last warm-up step (rank 0)"
        paths[dom_path]["timed_in"] = ("timed steps (rank 0): CUDA events around this path's launches in every "
                                       f"{os.environ['ISYCOS_PROFILE_EVERY']}th round "
                                       f"({kk.get('profiled_rounds', 0)} rounds)")
        for p in paths.values():
            p["achieved_Tcompare_s"] = p["compares"] / (p["kernel_ms"] / 1e3) / 1e12 if p["kernel_ms"] else None
            p["frac"] = (p["achieved_Tcompare_s"] * 1e12 / peak) if p["achieved_Tcompare_s"] else None
        dom = dom_path
        achieved = paths[dom]["achieved_Tcompare_s"] * 1e12 if paths[dom]["achieved_Tcompare_s"] else None
        line = {
            "metric": "KSG window compares/s", "value": value, "unit": "compares/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generators shaped like the paper's workloads; DESIGN.md §4)",
            "config": config_of(desc, args, world),
            "windows_per_s": wins / (ms_max / 1e3),
            "results_per_step": results / args.steps,
            "roofline": {"bound": "alu", "achieved": achieved / 1e12 if achieved else None,
                         "peak": peak / 1e12, "unit": "Tcompare/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic_for(dom),
                         "kernel": paths[dom]["kernel"], "path": dom,
                         "peak_basis": "issue-bound: 148 SM x 4 SMSP x 32 lanes x 1965 MHz / 5 lane-instr "
                                       "per compare (DESIGN.md §6)",
                         "kernel_share_of_step": (paths[dom]["kernel_ms"] * rounds / max(1, kk.get("profiled_rounds", 0))
                                                  / ms_total) if ms_total else None,
                         "paths": paths,
                         "ncu_issue": issue_for(dom),
                         "bruteforce_equivalent_compares_per_step_rank0": 2.0 * kpairs / args.steps},
            "e2e": {"value": e2e_comps / (e2e_max / 1e3), "unit": "compares/s",
                    "h2d_bytes_per_step": int(h2d_all // args.steps), "d2h_bytes_per_step": int(d2h_all // args.steps)},
            "gpu_launches": int(launches_all),
            "ksg_launches_rank0": ksg_launches,
            "rounds_per_step_rank0": rounds / args.steps,
            "host_ms_per_step_rank0": host_ms / args.steps,
            "clocks": clocks,
        }
        if dry_run:
            line["dry_run"] = "ranks share one GPU, gloo collectives: a code-path check, not a measurement"
        if world == 1 and not args.no_cpu_baseline and multi_pair:
            cores, model = cpu_info()
            pairs = batch_pairs(wl, 0, cores, 1)[:cores]
            prefix = REF_PREFIX if args.workload == "cfg4" else 131_072
            o = oracle_sample(args.workload, pairs, prefix, cores, {"n_chunks": 1} if args.workload == "cfg5" else {})
            line["cpu_baseline"] = {"value": o["value"], "unit": "compares/s", "cores": cores, "kind": "oracle",
                                    "sample": oracle_sample_desc(args.workload, prefix, len(pairs), cores, model,
                                                                 len(wl.series[0])),
                                    "windows_per_s": o["windows_per_s"], "wall_s": o["wall_s"]}
        if world == 1 and not args.no_side:
            line["side_configs1_search"] = side_configs1(isy, stream, max(3, args.steps))
            line["side_configs2_sweep"] = sweep_cfg3(isy, stream, max(1, args.steps // 2))
            line["side_configs4_search"] = side_configs4(isy, stream, args.cfg5_pairs)
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
