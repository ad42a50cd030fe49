"""Turn one gpurun session's artefacts into the committed profile summaries.

  python tools/profile_report.py <tag> <lib.so used on the box>

Reads gpurun_out/{bench_<tag>.json, configs_<tag>.jsonl, prof_<tag>.ncu-rep,
launches_<tag>.csv (optional)} and writes profiles/<tag>_bench.json,
<tag>_configs.jsonl / .md, <tag>_kernels.md (profiles/summarize_ncu.py) and
<tag>_k1_regions.md (ncu source counters joined with nvdisasm line info by
tools/ncu_source_lines.py).
"""
from __future__ import annotations

import collections
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
CONFIG_NAMES = ["c1_256 (256x256, L=4, 2^19, bench, 256^3/128^3 DT)",
                "c2_blob800 (800x800, L=2, 2^22, blob), one frame per call",
                "c2_blob800, 100-camera orbit as 2 calls of 50 cameras",
                "c3_1080p (1920x1080, L=2, 2^21, mip360c calibrated)", "c3_1080p, exact CUDA-core MLP",
                "c3_1080p_f32 (f32 storage)", "c3_mip360 (round-1 preset)",
                "c3_1080p, --shard tiles (N=1: one tile-major launch + assemble)",
                "c4_1080p_x64 (per-frame, camera ring)",
                "c4_1080p_x64, 64 cameras per call"] + \
               [f"c5_2160p boxes={n} (3840x2160, L=2, 2^22)" for n in (10, 35, 140, 560, 2240)] + \
               ["c5_2160p boxes=140, --shard tiles"]


def regions(tsv: Path, src: Path):
    """Classify SASS lines by the function the kernel loop called (inline chains)."""
    text = src.read_text().split("\n")

    def find(key, start=1):
        return next(i for i, l in enumerate(text, 1) if i >= start and key in l)
    dec_lo = find("void fine_level(")
    lane_lo = find("struct Lane {")
    march_lo = find("bool march_point(")
    kern_lo = find("march_kernel(const DevScene sc")
    end = find("// K0: ray generation")
    exit_lo = find("voxel_exit_step (occupancy.hpp:238-255): t_exit")
    exit_hi = find("float sz = t_exit - s.t;", exit_lo)

    def label(lab):
        inner, _, chain = lab.partition("|")
        frames = [inner] + (chain.split(">") if chain else [])
        frames = [(f.split(":")[0], int(f.split(":")[1])) for f in frames]
        mc = [(f, n) for f, n in frames if f == "march.cu"]
        # frames inside march_point's body decide march vs exit block
        for f, n in mc:
            if march_lo <= n < kern_lo:
                return ("voxel_exit_step (inside march_point)" if exit_lo <= n <= exit_hi
                        else "marching point (march_point)")
        for f, n in mc:
            if dec_lo <= n < lane_lo:
                return "decode (gathers, interpolation, fuse)"
        if any(kern_lo <= n < end for f, n in mc) or any(lane_lo <= n < march_lo for f, n in mc):
            return "warp loop, refill, composite"
        return "other"

    reg = collections.defaultdict(lambda: [0, 0, 0])
    lines = []
    for l in tsv.read_text().splitlines():
        lab, w, t, s = l.split("\t")
        w, t, s = int(w), int(t), int(s)
        lines.append((lab.split("|")[0] + (" <- " + lab.split("|")[1].split(">")[0] if "|" in lab else ""), w, t, s))
        r = reg[label(lab)]
        r[0] += w
        r[1] += t
        r[2] += s
    return reg, lines


def main():
    tag, lib = sys.argv[1], sys.argv[2]
    bench = json.loads((OUT / f"bench_{tag}.json").read_text())
    shutil.copy(OUT / f"bench_{tag}.json", PROF / f"{tag}_bench.json")
    rows = [json.loads(l) for l in (OUT / f"configs_{tag}.jsonl").read_text().splitlines() if l.strip()]
    shutil.copy(OUT / f"configs_{tag}.jsonl", PROF / f"{tag}_configs.jsonl")
    launches = OUT / f"launches_{tag}.csv"
    rep = OUT / f"prof_{tag}.ncu-rep"
    if launches.exists():
        shutil.copy(launches, PROF / f"{tag}_launches.csv")
    subprocess.run([sys.executable, str(PROF / "summarize_ncu.py"), str(rep),
                    str(launches if launches.exists() else PROF / "r01c_launches.csv"), tag],
                   check=True, capture_output=True)
    # configs table
    out = [f"# Throughput over the BASELINE configs (one B200), `{tag}`", "",
           f"`STEPS=8 bash tools/bench_configs.sh {tag}` under gpurun. Each step renders one frame; "
           "L2 is flushed before every timed step; times are CUDA events on the render stream.", "",
           "| config | fps | Mrays/s | K1 ms | K2 ms | roofline frac (K1 alg. bytes / HBM peak) | marching / occupied per ray |",
           "|---|---|---|---|---|---|---|"]
    for n, d in zip(CONFIG_NAMES, rows):
        st = d["config"]["mean_ray_stats"]
        out.append(f'| {n} | {d["value"]:.1f} | {d["mrays_per_s"]:.1f} | {d["kernel_ms"]["march_K1"]:.3f} '
                   f'| {d["kernel_ms"]["shade_K2"]:.3f} | {d["roofline"]["frac"]:.3f} | '
                   f'{st["marching"]:.1f} / {st["occupied"]:.2f} |')
    b = bench
    oc = b["roofline"].get("other_ceilings") or {}
    out += ["", f"Default `python bench.py` line of the same session (`{tag}_bench.json`): "
                f"**{b['value']:.1f} fps** device ({b['ms_per_step']:.2f} ms/frame), e2e {b['e2e']['value']:.1f} fps "
                f"(pipelined host API), e2e_sync {b['e2e_sync']['value']:.1f} fps, K1 {b['kernel_ms']['march_K1']:.3f} ms, "
                f"K2 {b['kernel_ms']['shade_K2']:.3f} ms, CPU reference {b.get('cpu_baseline', {}).get('value', float('nan')):.3f} fps.",
            f"K1 roofline: {b['roofline']['achieved']:.0f} GB/s algorithmic = {b['roofline']['frac']:.3f} of the HBM copy peak"
            + (f"; {oc['l2_gather32_gbs']['frac']:.2f} of the L2 32 B-gather ceiling, "
               f"{oc['l2_gather16_gbs']['frac']:.2f} of the 16 B one" if "l2_gather32_gbs" in oc else "") + "."]
    (PROF / f"{tag}_configs.md").write_text("\n".join(out) + "\n")
    # K1 source regions
    tsv = Path(f"/tmp/{tag}_k1.tsv")
    subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_source_lines.py"), lib, str(rep),
                    "march_kernelILi2ELb1ELb0ELb1E", str(tsv)], check=True, capture_output=True)
    reg, lines = regions(tsv, ROOT / "paper_2407_10482_b200" / "csrc" / "march.cu")
    tw = sum(v[0] for v in reg.values())
    ts = sum(v[2] for v in reg.values()) or 1
    md = [f"# K1 issue-slot breakdown by source region (`{tag}`)", "",
          "ncu source counters of one 1080p `march_kernel<2,1,0,1,...>` launch (config 3, tensor mode), "
          "joined per SASS instruction with `nvdisasm -gi` line info (`tools/ncu_source_lines.py`). "
          f"Total {tw / 1e9:.3f} G warp instructions.", "",
          "| region | warp instructions | share | threads / inst | stall samples |", "|---|---|---|---|---|"]
    for r, (w, t, s) in sorted(reg.items(), key=lambda kv: -kv[1][0]):
        md.append(f"| {r} | {w / 1e9:.3f} G | {w / tw * 100:.1f} % | {t / max(w, 1):.1f} | {s / ts * 100:.1f} % |")
    md += ["", "| top lines | warp instructions | threads / inst | stall samples |", "|---|---|---|---|"]
    for lab, w, t, s in sorted(lines, key=lambda x: -x[1])[:20]:
        md.append(f"| {lab} | {w / 1e6:.1f} M | {t / max(w, 1):.1f} | {s} |")
    (PROF / f"{tag}_k1_regions.md").write_text("\n".join(md) + "\n")
    print("\n".join(md[:12]))


if __name__ == "__main__":
    main()
