"""Summarise ncu outputs into the tracked files under profiles/.

    python profiles/summarize.py launches <launches.csv> <out.md>
    python profiles/summarize.py report <prof.ncu-rep> <out.md> [<traffic.json> <pixels_per_launch>]

`launches` aggregates a `--metrics gpu__time_duration.sum` launch list into
per-kernel totals and shares (cold-cache, serialised: compare shares).
`report` extracts the key metrics of a `--set full` capture per launch and,
optionally, writes dram bytes per pixel of the association kernel for
bench.py's `roofline.traffic`.
"""

import collections
import csv
import io
import json
import subprocess
import sys


def _rows(text):
    return list(csv.reader(io.StringIO(text)))


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
             "second": 1e6}
    for r in data:
        if len(r) > mi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0].replace("void ", "")
            tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
            cnt[name] += 1
    total = sum(tot.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / total:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "L2 Hit Rate", "Executed Instructions", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]


def report(rep, out, traffic_json=None, pixels=None):
    det = _rows(subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                               text=True).stdout)
    raw = _rows(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                               text=True).stdout)
    h = det[0]
    ii, ki, mi, vi, ui = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value",
                                                  "Metric Unit"))
    per = collections.OrderedDict()
    for r in det[1:]:
        if r[mi] in WANT:
            per.setdefault((r[ii], r[ki].split("(")[0]), {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    rh, ru = raw[0], raw[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3,
             "usecond": 1.0, "msecond": 1e3}
    rawvals = {}
    for r in raw[2:]:
        key = r[rh.index("ID")]
        vals = {}
        for m in RAW:
            if m in rh:
                i = rh.index(m)
                unit = ru[i]
                try:
                    v = float(r[i].replace(",", "")) * scale.get(unit, 1.0)
                    unit = "byte" if unit.endswith("byte") else ("us" if unit.endswith("second") else unit)
                    vals[m] = f"{v:.6g} {unit}"
                except ValueError:
                    vals[m] = r[i]
        rawvals[key] = vals
    lines = []
    traffic = {}
    for (i, name), m in per.items():
        rv = rawvals.get(i, {})
        lines.append(f"### launch {i}: `{name}`")
        for k in WANT:
            if k in m:
                lines.append(f"- {k}: {m[k]}")
        for k, v in rv.items():
            lines.append(f"- {k}: {v}")
        try:
            b = float(rv["dram__bytes_read.sum"].split()[0]) + float(
                rv["dram__bytes_write.sum"].split()[0])
            traffic.setdefault(name, []).append(b)
        except (KeyError, ValueError):
            pass
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_json and pixels:
        assoc = [v for k, vs in traffic.items() if "k_cell<1" in k or "k_cell<true" in k for v in vs]
        if assoc:
            json.dump({"kernel": "k_cell<ACC> (association + centre-update pass)",
                       "dram_bytes_per_pixel": sum(assoc) / len(assoc) / float(pixels),
                       "pixels_per_launch": int(pixels), "source": rep, "launches": len(assoc)},
                      open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        report(sys.argv[2], sys.argv[3], *(sys.argv[4:6] if len(sys.argv) > 5 else []))
