"""Summaries of ncu outputs for profiles/ (tracked), from gpurun_out/ (scratch).

    python tools/ncu_summarize.py launches <launch-list.csv> <out.md>
    python tools/ncu_summarize.py full <report.ncu-rep> <out-prefix> [algorithmic_bytes]

`launches`: per-kernel count / total / mean / share of a `--metrics
gpu__time_duration.sum` launch list (cold-cache, serialised: the SHARE is what
compares with the live timing, not the absolute).
`full`: key counters, warp-stall breakdown and the hottest SASS lines of one
`--set full` capture; writes <prefix>.md and <prefix>.json (dram bytes per
launch -> bench.py's roofline.traffic).
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        agg.setdefault(name, []).append(v * scale)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# Launch list: `{path.split('/')[-1]}`", "",
             "ncu `--metrics gpu__time_duration.sum --clock-control none` (serialised, cold caches).", "",
             "| kernel | launches | total us | mean us | share |", "|---|---:|---:|---:|---:|"]
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{name}` | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")
    lines.append(f"| **all** | {sum(len(v) for v in agg.values())} | {tot:.1f} | | 100% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg.per_second", "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_tc.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def _ncu_csv(rep, *args):
    r = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def full(rep, prefix, algo_bytes=None):
    rows = _ncu_csv(rep, "--page", "raw")
    hdr, units = rows[0], rows[1]
    out = {"report": rep.split("/")[-1]}
    for k, r in enumerate(rows[2:]):
        name = r[hdr.index("Kernel Name")]
        m = OrderedDict()
        for key in KEYS:
            if key in hdr:
                m[key] = (r[hdr.index(key)], units[hdr.index(key)])
        stalls = []
        for i, h in enumerate(hdr):
            if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        rd = float(m["dram__bytes_read.sum"][0].replace(",", ""))
        wr = float(m["dram__bytes_write.sum"][0].replace(",", ""))
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
        rd *= mult.get(m["dram__bytes_read.sum"][1], 1)
        wr *= mult.get(m["dram__bytes_write.sum"][1], 1)
        dur = float(m["gpu__time_duration.sum"][0].replace(",", ""))
        # ncu prints the unit either spelled out ("msecond") or abbreviated ("ms")
        tunit = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
                 "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
        dur_s = dur * tunit[m["gpu__time_duration.sum"][1]]
        out.setdefault("kernels", []).append({
            "kernel": name, "gpu_time_s": dur_s, "dram_bytes_read": rd, "dram_bytes_write": wr,
            "dram_bytes_per_launch": rd + wr, "dram_gbs": (rd + wr) / dur_s / 1e9,
            "algorithmic_bytes_per_launch": algo_bytes,
            "metrics": {k: " ".join(v) for k, v in m.items()},
            "stalls_pct": {n: round(100 * v / tot, 1) for v, n in sorted(stalls, reverse=True)[:10]}})
    k0 = out["kernels"][0]
    out["dram_bytes_per_launch"] = k0["dram_bytes_per_launch"]
    # hottest SASS lines of the first kernel
    src = _ncu_csv(rep, "--page", "source", "--print-source", "sass")
    hot = []
    if len(src) > 2:
        h = src[1]
        ie, ws, sc = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
        ins = []
        for r in src[2:]:
            try:
                ins.append((float(r[ws] or 0), float(r[ie] or 0), r[sc].strip()[:70]))
            except ValueError:
                pass
        totw = sum(i[0] for i in ins) or 1.0
        toti = sum(i[1] for i in ins) or 1.0
        hot = [(round(100 * w / totw, 1), round(100 * e / toti, 2), s) for w, e, s in sorted(ins, reverse=True)[:12]]
        out["warp_instructions"] = toti
    json.dump(out, open(prefix + ".json", "w"), indent=1)
    lines = [f"# ncu --set full: `{out['report']}`", ""]
    for kk in out["kernels"]:
        lines += [f"## `{kk['kernel']}`", "", "| metric | value |", "|---|---|"]
        lines += [f"| {k} | {v} |" for k, v in kk["metrics"].items()]
        lines += [f"| dram bytes / launch (read+write) | {kk['dram_bytes_per_launch'] / 1e6:.1f} MB |",
                  f"| achieved dram GB/s under ncu | {kk['dram_gbs']:.0f} |"]
        if algo_bytes:
            lines.append(f"| algorithmic bytes / launch | {algo_bytes / 1e6:.1f} MB |")
        lines += ["", "Warp stalls (share of samples): " +
                  ", ".join(f"{n} {v}%" for n, v in kk["stalls_pct"].items()), ""]
    if hot:
        lines += ["Hottest SASS (stall share %, instruction share %, source):", "", "```"]
        lines += [f"{w:5.1f}% {e:6.2f}%  {s}" for w, e, s in hot] + ["```"]
    open(prefix + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
