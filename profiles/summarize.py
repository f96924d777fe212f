#!/usr/bin/env python
"""Summarise Nsight Compute output for profiles/ (run here, no GPU needed).

  python profiles/summarize.py full <report.ncu-rep> <records> <label>   key metrics of a --set full capture
  python profiles/summarize.py launches <launches.csv>                    per-kernel share of a launch list
  python profiles/summarize.py lines <report.ncu-rep> <records>          hottest source lines

The numbers feed DESIGN.md ("Measurements") and bench.py's roofline.traffic
(profiles/ncu_summary.json).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
    "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
]


def _num(s):
    return float(s.replace(",", ""))


def full(rep, records, label):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"label": label, "kernel": vals[hdr.index("Kernel Name")], "records": records}
    lines = ["# %s" % label, "", "kernel: %s" % out["kernel"], "", "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            lines.append("| %s | %s | %s |" % (k, vals[i], units[i]))
            try:
                out[k] = _num(vals[i])
            except ValueError:
                pass
    # per-record figures
    rd = out.get("dram__bytes_read.sum", 0)
    wr = out.get("dram__bytes_write.sum", 0)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
    wr *= scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
    out["dram_bytes_per_launch"] = rd + wr
    lines += ["", "dram bytes per launch: %.4g (read %.4g + write %.4g)" % (rd + wr, rd, wr)]
    if "smsp__inst_executed.sum" in out:
        lines.append("warp instructions per record: %.2f" % (out["smsp__inst_executed.sum"] / records))
    if "smsp__thread_inst_executed.sum" in out:
        lines.append("thread instructions per record: %.1f" % (out["smsp__thread_inst_executed.sum"] / records))
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                st.append((_num(vals[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    lines += ["", "stall reasons (pc sampling):", ""]
    for v, h in sorted(st, reverse=True)[:10]:
        lines.append("- %s: %.1f%%" % (h, 100 * v / tot))
    return out, "\n".join(lines) + "\n"


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    iK, iM, iV, iU = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if r[iM] == "gpu__time_duration.sum":
            agg[r[iK]].append(_num(r[iV]) * scale.get(r[iU], 1e-3))
    tot = sum(sum(v) for v in agg.values())
    lines = ["| kernel | launches | mean us | share of listed time |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append("| %s | %d | %.1f | %.1f%% |" % (k[:80].replace("|", "/"), len(v), sum(v) / len(v), 100 * sum(v) / tot))
    # one timed step launches the fast kernel (no-stats instance) and k_slow once
    # each; their mean durations give each kernel's share of the step
    def stats_instance(name):  # k_split<SEPS, STATS, ...> / k_batch<STATS, ...>
        if "<" not in name:
            return False
        args = [x.strip() for x in name[name.index("<") + 1:name.index(">")].split(",")]
        i = 1 if "k_split" in name else 0
        return len(args) > i and args[i] in ("1", "true")
    step = {k: sum(v) / len(v) for k, v in agg.items()
            if "fpp::" in k and ("k_slow" in k or not stats_instance(k))}
    st = sum(step.values()) or 1.0
    lines += ["", "one step (product kernels, mean per launch; cold-cache, serialised under ncu):", "",
              "| kernel | mean us | share of step |", "|---|---|---|"]
    for k, v in sorted(step.items(), key=lambda kv: -kv[1]):
        lines.append("| %s | %.1f | %.1f%% |" % (k[:80], v, 100 * v / st))
    return "\n".join(lines) + "\n"


def hot_lines(rep, records, top=25):
    """Per CUDA source line: warp instructions per record and share of warp-state samples."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, agg = None, collections.OrderedDict()
    for r in csv.reader(io.StringIO(raw)):
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) < 8 or r[0] in ("", "Line No"):
            continue
        try:
            agg[(cur, r[0])] = (int(r[7]), int(r[4]), r[1].strip()[:70])
        except ValueError:
            pass
    tot_s = sum(v[1] for v in agg.values()) or 1
    lines = ["| file:line | warp inst / record | share of samples | source |", "|---|---|---|---|"]
    for (f, ln), (ie, ss, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        lines.append("| %s:%s | %.2f | %.1f%% | `%s` |" % (f, ln, ie / records, 100 * ss / tot_s, src.replace("|", "/")))
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    if sys.argv[1] == "full":
        d, text = full(sys.argv[2], float(sys.argv[3]), sys.argv[4])
        print(text)
        js = os.path.join(HERE, "ncu_summary.json")
        allj = json.load(open(js)) if os.path.exists(js) else {}
        allj[sys.argv[4]] = d
        json.dump(allj, open(js, "w"), indent=1)
    elif sys.argv[1] == "lines":
        print(hot_lines(sys.argv[2], float(sys.argv[3])))
    else:
        print(launches(sys.argv[2]))
