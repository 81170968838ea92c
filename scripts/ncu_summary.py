"""Summarise an ncu report (.ncu-rep) or a launch-list CSV into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_r01_cfg2.md [--traffic-json profiles/ncu_traffic_cfg2.json]
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv profiles/launches_r01_cfg2.md
"""
import argparse
import collections
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    "Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
    "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
    "Theoretical Occupancy", "Waves Per SM", "L1/TEX Hit Rate", "L2 Hit Rate",
    "Warp Cycles Per Issued Instruction", "No Eligible", "Dynamic Shared Memory Per Block",
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed.sum", "smsp__inst_executed.sum", "lts__t_bytes.sum",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def short(name):
    m = re.search(r"(k_\w+)", name)
    return m.group(1) if m else name[:40]


def summarise_rep(rep, out_md, traffic_json):
    rows = ncu_csv(rep, "details")
    h = rows[0]
    ki, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    det = collections.OrderedDict()
    for r in rows[1:]:
        k = short(r[ki])
        det.setdefault(k, collections.OrderedDict())
        if r[mi] in KEYS and r[mi] not in det[k]:
            det[k][r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = ncu_csv(rep, "raw")
    rh = raw[0]
    units = dict(zip(rh, raw[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    rawd = collections.OrderedDict()
    stalls = collections.OrderedDict()
    for r in raw[2:]:
        d = dict(zip(rh, r))
        k = short(d["Kernel Name"])
        rawd[k] = {m: f"{d.get(m)} {units.get(m, '')}".strip() for m in RAW if m in d}
        st = {}
        for key, v in d.items():
            if key.startswith("smsp__pcsamp_warps_issue_stalled") and not key.endswith("not_issued"):
                try:
                    fv = float(v.replace(",", ""))
                except ValueError:
                    continue
                if fv > 0:
                    st[key.replace("smsp__pcsamp_warps_issue_stalled_", "")] = fv
        tot = sum(st.values()) or 1.0
        stalls[k] = sorted(((n, v / tot) for n, v in st.items()), key=lambda t: -t[1])[:6]
    lines = [f"# ncu summary: `{rep}`", ""]
    for k in det:
        lines.append(f"## {k}")
        for m, v in det[k].items():
            lines.append(f"- {m}: {v}")
        if k in rawd:
            for m, v in rawd[k].items():
                lines.append(f"- {m}: {v}")
        if k in stalls:
            lines.append("- top stall reasons (share of samples): " +
                         ", ".join(f"{n} {100 * v:.0f}%" for n, v in stalls[k]))
        lines.append("")
    with open(out_md, "w") as fh:
        fh.write("\n".join(lines))
    if traffic_json:
        traffic = {}
        for k, d in rawd.items():
            try:
                def nbytes(v):
                    num, unit = v.split(" ", 1)
                    return float(num.replace(",", "")) * scale.get(unit.strip(), 1.0)
                rd = nbytes(d["dram__bytes_read.sum"])
                wr = nbytes(d["dram__bytes_write.sum"])
                # profiler kinds: every pass-2 variant is "pass2"
                kind = k.replace("k_", "").replace("_gauss", "")
                kind = "pass2" if kind.startswith("pass2") else kind
                traffic[kind] = rd + wr
                if "smsp__inst_executed.sum" in d:  # warp instructions per launch
                    inst = float(d["smsp__inst_executed.sum"].split(" ", 1)[0].replace(",", ""))
                    traffic.setdefault("_inst", {})[kind] = inst
            except Exception:
                pass
        with open(traffic_json, "w") as fh:
            json.dump(traffic, fh, indent=1)
    print(open(out_md).read())


def summarise_launches(path, out_md):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(d["Kernel Name"])
        data.setdefault(k, []).append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in data.values()) or 1.0
    lines = [f"# launch list: `{path}` (ncu gpu__time_duration.sum, cold-cache, serialised)", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(data.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
    with open(out_md, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("out")
    ap.add_argument("--launches", action="store_true")
    ap.add_argument("--traffic-json")
    a = ap.parse_args()
    if a.launches:
        summarise_launches(a.src, a.out)
    else:
        summarise_rep(a.src, a.out, a.traffic_json)
