"""Summarise ncu captures into profiles/ (run here, on the CPU box).

  python profiles/summarize_ncu.py <full.ncu-rep> <launches.csv> <tag> [--config c3_1080p]

Writes profiles/<tag>_kernels.md (key metrics per profiled kernel + the launch
list's per-kernel time shares) and updates profiles/ncu_traffic.json with the
march kernel's DRAM bytes per launch (read by bench.py for roofline.traffic).
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__t_sectors.sum", "L2 sectors (32 B)"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads / instruction"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6,
              "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def stalls(rep, kernel_regex):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "-k",
                          f"regex:{kernel_regex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    h, v = rows[0], rows[2]
    res = {}
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                x = float(v[i])
            except ValueError:
                continue
            if x > 0:
                res[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = x
    tot = sum(res.values()) or 1
    return {k: round(100 * x / tot, 1) for k, x in sorted(res.items(), key=lambda kv: -kv[1])[:8]}


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1e-6)
        name = r[ki].split("(")[0].replace("void ", "").replace("ngprt_dev::<unnamed>::", "")
        a = tot.setdefault(name, [0.0, 0])
        a[0] += v
        a[1] += 1
    return tot


def main():
    rep, launches, tag = Path(sys.argv[1]), Path(sys.argv[2]), sys.argv[3]
    config = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "c3_1080p"
    h, units, data = ncu_raw(rep)
    lines = [f"# ncu summary `{tag}`", "",
             f"Source: `{rep.name}` (`ncu --set full --clock-control none`, cold L2 per replay) and "
             f"`{launches.name}` (`--metrics gpu__time_duration.sum`, every launch).", ""]
    traffic = l2 = l2_read = l2_util = None
    for row in data:
        name = row[h.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").replace("ngprt_dev::<unnamed>::", "").replace("unnamed>::", "")
        lines.append(f"## {short}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m, label in METRICS:
            if m in h:
                i = h.index(m)
                lines.append(f"| {label} (`{m}`) | {row[i]} {units[i]} |")
        if "march_kernel" in short:
            i, j = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
            traffic = (float(row[i]) * UNIT_SCALE.get(units[i], 1) +
                       float(row[j]) * UNIT_SCALE.get(units[j], 1))
            l2 = None
            if "lts__t_bytes.sum" in h:
                k = h.index("lts__t_bytes.sum")
                l2 = float(row[k]) * UNIT_SCALE.get(units[k], 1)
            elif "lts__t_sectors.sum" in h:  # 32 B sectors
                l2 = float(row[h.index("lts__t_sectors.sum")]) * 32.0
            # the gather traffic proper: sectors the SMs' L1s request from L2, and
            # how busy the L2 slices are with them
            l2_read = l2_util = None
            if "lts__t_sectors_srcunit_tex.sum" in h:
                l2_read = float(row[h.index("lts__t_sectors_srcunit_tex.sum")]) * 32.0
            m = "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed"
            if m in h:
                l2_util = float(row[h.index(m)])
        st = stalls(rep, short.split("<")[0].split("::")[-1])
        if st:
            lines.append("")
            lines.append("Warp-stall sampling (% of stalled samples): " +
                         ", ".join(f"{k} {v}" for k, v in st.items()))
        lines.append("")
    shares = launch_shares(launches)
    total = sum(v[0] for v in shares.values())
    lines += ["## Launch list (all kernels of the run, serialised, cold per launch)", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (ms, n) in sorted(shares.items(), key=lambda kv: -kv[1][0]):
        lines.append(f"| {k[:70]} | {n} | {ms:.3f} | {100 * ms / total:.1f}% |")
    (HERE / f"{tag}_kernels.md").write_text("\n".join(lines) + "\n")
    if traffic is not None:
        tp = HERE / "ncu_traffic.json"
        d = json.loads(tp.read_text()) if tp.exists() else {}
        d[config] = {"dram_bytes_per_launch": traffic, "l2_bytes_per_launch": l2,
                     "l2_read_bytes_per_launch": l2_read, "l2_slice_util_pct": l2_util,
                     "source": f"{rep.name} ({tag})", "kernel": "march_kernel (K1)"}
        tp.write_text(json.dumps(d, indent=1) + "\n")
    print((HERE / f"{tag}_kernels.md").read_text())


if __name__ == "__main__":
    main()
