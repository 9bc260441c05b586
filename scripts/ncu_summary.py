#!/usr/bin/env python
"""Summarise ncu captures into small committed text files under profiles/.

  python scripts/ncu_summary.py rep  gpurun_out/prof.ncu-rep  profiles/r01_tile4096.md
  python scripts/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.md
"""
import collections
import csv
import io
import os
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Issued Warp Per Scheduler", "No Eligible", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Branch Efficiency", "Avg. Divergent Branches",
        "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput", "Memory Throughput"]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def rep(path, dst):
    rows = ncu_csv(["-i", path, "--page", "details"])
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full summary: `{path.split('/')[-1]}`", ""]
    by_id = collections.OrderedDict()
    for r in rows[1:]:
        by_id.setdefault(r[idx["ID"]], []).append(r)
    raw = ncu_csv(["-i", path, "--page", "raw"])
    rhdr = raw[0] if raw else []
    for kid, rs in by_id.items():
        lines.append(f"## launch {kid}: `{rs[0][idx['Kernel Name']][:120]}`")
        lines.append("")
        lines.append("| metric | unit | value |")
        lines.append("|---|---|---|")
        seen = set()
        for r in rs:
            m = r[idx["Metric Name"]]
            if m in KEYS and m not in seen:
                seen.add(m)
                lines.append(f"| {m} | {r[idx['Metric Unit']]} | {r[idx['Metric Value']]} |")
        # dram bytes from the raw page
        for want in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                     "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"):
            if want in rhdr:
                j = rhdr.index(want)
                row = raw[2 + int(kid)] if len(raw) > 2 + int(kid) else None
                if row:
                    lines.append(f"| {want} | {raw[1][j]} | {row[j]} |")
        lines.append("")
    # instruction mix from the source page
    src = ncu_csv(["-i", path, "--page", "source", "--print-source", "sass"])
    # one section per kernel: ["Kernel Name", name], header row, data rows
    sections = []
    for r in src:
        if r and r[0] == "Kernel Name":
            sections.append([r[1] if len(r) > 1 else "?", None, []])
        elif sections and sections[-1][1] is None:
            sections[-1][1] = r
        elif sections:
            sections[-1][2].append(r)
    for name, h, rows in sections:
        if not h:
            continue
        ix = {k: i for i, k in enumerate(h)}
        if "Source" not in ix or "Instructions Executed" not in ix:
            continue
        mix = collections.Counter()
        stall = collections.Counter()
        tot = stot = 0
        for r in rows:
            if len(r) != len(h):
                continue
            s = r[ix["Source"]].strip()
            if not s or not r[ix["Instructions Executed"]].isdigit():
                continue
            toks = s.split()
            op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
            n = int(r[ix["Instructions Executed"]] or 0)
            sm = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            mix[op] += n
            stall[op] += sm
            tot += n
            stot += sm
        lines += [f"## instruction mix of `{name[:90]}` (warp-level executed) and stall-sample share", "",
                  "| opcode | % instr | % stall samples |", "|---|---|---|"]
        for op, n in mix.most_common(16):
            lines.append(f"| {op} | {100 * n / max(tot, 1):.1f} | {100 * stall[op] / max(stot, 1):.1f} |")
        lines.append("")
    open(dst, "w").write("\n".join(lines) + "\n")


def launches(path, dst):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in rows if r[0] == "ID")
    idx = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0, 0.0])  # launches, us, grid sum, small grids, small us
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    per = collections.defaultdict(dict)
    for r in rows:
        if r[0] == "ID" or len(r) != len(hdr):
            continue
        m = r[idx["Metric Name"]]
        v = float(r[idx["Metric Value"]].replace(",", ""))
        if m == "gpu__time_duration.sum":
            v *= scale.get(r[idx["Metric Unit"]], 1.0)
        per[r[idx["ID"]]][m] = v
        per[r[idx["ID"]]]["name"] = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")
    for d in per.values():
        if "gpu__time_duration.sum" not in d:
            continue
        a = agg[d["name"]]
        a[0] += 1
        a[1] += d["gpu__time_duration.sum"]
        g = d.get("launch__grid_size", 0.0)
        a[2] += g
        if g and g < 148:
            a[3] += 1
            a[4] += d["gpu__time_duration.sum"]
    tot = sum(v[1] for v in agg.values())
    lines = [f"# launch list summary: `{path.split('/')[-1]}` (ncu --metrics gpu__time_duration.sum, "
             "cold-cache, serialised: compare shares, not absolutes)", "",
             "| kernel | launches | total us | share | avg us | avg grid | launches with grid < 148 (their us) |",
             "|---|---|---|---|---|---|---|"]
    for k, (n, us, gs, ns, nus) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f}% | {us / n:.2f} | {gs / n:.0f} | "
                     f"{ns} ({nus:.0f}) |")
    open(dst, "w").write("\n".join(lines) + "\n")


def traffic(path, key, name_re=".*", dst="profiles/traffic.json"):
    """Average dram__bytes_read.sum + dram__bytes_write.sum per captured launch of a --set full report;
    stored under `key` (a bench.py path name) for bench.py's roofline "traffic" field."""
    import json
    import os

    import re

    raw = ncu_csv(["-i", path, "--page", "raw"])
    hdr, units = raw[0], raw[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    kn = hdr.index("Kernel Name")
    tot, n = 0.0, 0
    for row in raw[2:]:
        if len(row) != len(hdr) or not re.search(name_re, row[kn]):
            continue
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            j = hdr.index(m)
            b += float(row[j].replace(",", "")) * scale.get(units[j], 1.0)
        tot += b
        n += 1
    d = json.load(open(dst)) if os.path.exists(dst) else {}
    d[key] = {"bytes_per_launch": tot / max(n, 1), "launches": n, "source": os.path.basename(path),
              "kernels": name_re}
    json.dump(d, open(dst, "w"), indent=1)
    print(key, d[key])


def issue(path, key, name_re=".*", dst="profiles/issue.json"):
    """Issue efficiency of the matching launches of a --set full report (launch-duration weighted):
    warp-issue utilisation (smsp__issue_active / cycles) x lane utilisation (avg active threads / 32) =
    the fraction of the SMs' FP32/INT32 lane-issue peak actually used (the north star's "% of issue
    peak").  Stored under `key` for bench.py's roofline object."""
    import json
    import os
    import re

    rows = ncu_csv(["-i", path, "--page", "details"])
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in rows[1:]:
        if len(r) <= ix["Metric Value"] or not re.search(name_re, r[ix["Kernel Name"]]):
            continue
        d = per.setdefault(r[ix["ID"]], {})
        val = r[ix["Metric Value"]].replace(",", "")
        if r[ix["Metric Name"]] == "Duration":  # normalise to us
            sc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
            val = str(float(val) * sc.get(r[ix["Metric Unit"]], 1.0))
        d[r[ix["Metric Name"]]] = val
    tw = busy = lanes = 0.0
    n = 0
    for d in per.values():
        try:
            dur = float(d["Duration"])
            b = float(d["Issue Slots Busy"]) / 100.0
            a = float(d["Avg. Active Threads Per Warp"]) / 32.0
        except (KeyError, ValueError):
            continue
        tw += dur
        busy += dur * b
        lanes += dur * b * a
        n += 1
    if not n:
        print(key, "no launches matched")
        return
    out = {"issue_slots_busy": busy / tw, "lane_issue_frac": lanes / tw, "launches": n,
           "source": os.path.basename(path), "kernels": name_re}
    dd = json.load(open(dst)) if os.path.exists(dst) else {}
    dd[key] = out
    json.dump(dd, open(dst, "w"), indent=1)
    print(key, out)


def opcodes(path, name_re, dst):
    """Executed warp instructions per SASS opcode (summed over the matching launches of a --set full capture),
    with the average active lanes and the share of warp-stall samples, from ncu's source page."""
    rows = ncu_csv(["-i", path, "--page", "source", "--kernel-name", f"regex:{name_re}", "--print-source", "sass"])
    ops, thr, st = collections.Counter(), collections.Counter(), collections.Counter()
    hdr = None
    for r in rows:
        if "Source" in r and "Instructions Executed" in r:
            hdr = r
            i_src, i_ie = r.index("Source"), r.index("Instructions Executed")
            i_te, i_s = r.index("Thread Instructions Executed"), r.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) <= max(i_src, i_ie, i_te, i_s):
            continue
        try:
            ie, te, sm = int(r[i_ie]), int(r[i_te]), int(r[i_s])
        except ValueError:
            continue
        t = r[i_src].split()
        op = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "?")).split(".")[0]
        ops[op] += ie
        thr[op] += te
        st[op] += sm
    tot, tt, ts = sum(ops.values()), sum(thr.values()), max(1, sum(st.values()))
    with open(dst, "w") as f:
        f.write(f"# {name_re} in {os.path.basename(path)}: executed warp instructions by SASS opcode\n")
        if not tot:
            f.write("no launches matched\n")
            return
        f.write(f"warp instructions {tot}  thread instructions {tt}  average lanes {tt / tot:.1f}\n")
        for op, c in ops.most_common(30):
            f.write(f"{op:10s} {c / tot * 100:5.1f}%  lanes {thr[op] / c:5.1f}  stall share {st[op] / ts * 100:5.1f}%\n")


if __name__ == "__main__":
    {"rep": rep, "launches": launches, "traffic": traffic, "issue": issue, "opcodes": opcodes}[sys.argv[1]](*sys.argv[2:])
