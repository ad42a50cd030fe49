#!/usr/bin/env python
"""bench.py — throughput of the B200 NGP-RT render path (BASELINE.json metric).

A step = one 1920x1080 frame rendered by every rank (weak scaling): raygen ->
march -> gather -> fuse -> composite (K1) -> deferred MLP (K2), on the
synthetic config-3 scene (SynthScene "c3_1080p"). Rank r
renders camera (r + N*step) mod 64 of sphere_views(64, 2.9) (config 4's camera
set); for N > 1 the finished frames are gathered to rank 0 over NCCL inside the
step (the only collective).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Timing: W untimed warm-up steps; L2 flushed (256 MiB write) before every timed
step; each step bracketed by CUDA events on the render stream after a barrier +
synchronize; total = sum over steps, max over ranks. `e2e` re-times the same
steps through the host-buffer C ABI (camera H2D and the RGB D2H inside the
timed region): ngprt_render_host_async with two frames in flight (the serving
call; `e2e`) and the synchronous ngprt_render_host (`e2e_sync`). `roofline` is K1's algorithmic bytes
(SURVEY.md §8(d) formula over the bit-exact per-ray counters) / K1's event time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "1080p fps & Mrays/s at 1/2/4/8 B200 vs host-CPU ref; achieved L2/HBM GB/s"
UNIT = "fps (1920x1080 frames/s, all GPUs)"
N_CAMS = 64
PAPER_FPS = 108.0  # 1080p, L=2, RTX 3090
L2_NOTE = ("flushed (256 MiB write) before every timed step; fine hash tables of <= 41 MB "
           "(config 1) are pinned by the renderer's persisting access-policy window, whose lines "
           "survive the flush by design (north_star); larger ones (config 3: 64 MB) are not "
           "pinned and are flushed like everything else")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c3_1080p")
    ap.add_argument("--mlp", choices=["tensor", "exact"], default=os.environ.get("NGPRT_MLP", "tensor"))
    ap.add_argument("--no-l2-flush", action="store_true")
    ap.add_argument("--batch", type=int, default=1,
                    help="cameras per ngprt_render call (one step renders a batch of frames)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target wall time of the bounded CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", choices=["cameras", "tiles"], default="cameras",
                    help="cameras: each rank renders whole frames (weak scaling, the default); "
                         "tiles: every frame split into interleaved tiles over the ranks")
    ap.add_argument("--tile", type=int, default=32, help="--shard tiles: tile edge in pixels")
    ap.add_argument("--scene", action="append", default=[],
                    help="override a synthetic-scene parameter, e.g. --scene n_boxes=560")
    return ap.parse_args()


def scene_config(ng, args):
    cfg = dict(ng.CONFIGS[args.config])
    for kv in args.scene:
        k, v = kv.split("=", 1)
        cfg[k] = type(cfg.get(k, 0.0))(v) if k in cfg else (float(v) if "." in v else int(v))
    return cfg


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_tensor_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text()).get("bf16_tflops", 0.0)) or None
    return None


def algorithmic_bytes(stats, L, b_c=2, b_f=2):
    """sum over rays of occupied*8*((8+2L)*b_c + 8L*b_f)
    + 4*occ_acc + 1*dist_acc + 12 (RGB out)."""
    import numpy as np
    s = stats.reshape(-1, 4).astype(np.float64)
    per_sample = 8 * ((8 + 2 * L) * b_c + 8 * L * b_f)
    return float((s[:, 1] * per_sample + 4 * s[:, 2] + 1 * s[:, 3]).sum() + 12 * s.shape[0])


def binding_ceiling(tj, k1_ms, ceilings):
    """Name what binds K1, from the ncu capture of the same build (tj, one K1
    launch) and this run's K1 time: the gather traffic its L1s request from L2
    (lts__t_sectors_srcunit_tex) against the L2-resident random 32 B-gather rate
    measured on this B200 and against the L2 slices' own sector throughput, and
    its DRAM traffic against the HBM copy peak."""
    if not tj or not tj.get("l2_read_bytes_per_launch"):
        return None
    l2 = tj["l2_read_bytes_per_launch"] / (k1_ms / 1e3) / 1e9
    out = {"l2_read_gbs": l2, "l2_slice_util_pct_ncu": tj.get("l2_slice_util_pct")}
    if ceilings and "l2_gather32_gbs" in ceilings:
        g = ceilings["l2_gather32_gbs"]["peak_gbs"]
        out.update(gather32_peak_gbs=g, gather32_frac=l2 / g)
    if tj.get("dram_bytes_per_launch"):
        peak, _ = load_peaks()
        out["dram_frac_of_hbm_peak"] = tj["dram_bytes_per_launch"] / (k1_ms / 1e3) / 1e9 / peak
    out["verdict"] = ("gather-latency bound: neither the L2 slices nor DRAM are near their "
                      "throughput (see DESIGN.md §4)")
    return out


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(self.device)],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            out, _ = self.p.communicate()
            self.lines = [l.split(", ") for l in out.strip().splitlines() if l.strip()]

    def summary(self):
        if not self.lines:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(l[1]) for l in self.lines if len(l) > 2 and l[1].replace(".", "").isdigit()]
        mx = [float(l[2]) for l in self.lines if len(l) > 2 and l[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for l in self.lines:
            for i, n in enumerate(names):
                if len(l) > 5 + i and l[5 + i].strip() == "Active":
                    reasons.add(n)
        load = [v for v in sm if v > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.lines)}


def cpu_sample(scene_synth, cams, W, H, seconds, kind_pref="reference"):
    """Bounded CPU-baseline sample: FULL frames of the timed cameras (the same
    frames the GPU renders) by oracle/_ref (the reference itself) when present,
    else the C restatement, with every host thread, until `seconds` of work; plus
    the one-thread rate on a 4-row band (1 thread and nproc)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from checkers import REF_SO, CpuScene
    import paper_2407_10482_b200 as ng
    kind = "reference" if (kind_pref == "reference" and REF_SO.exists()) else "port"
    cs = CpuScene(scene_synth.desc_ptr, "ref" if kind == "reference" else "oracle")
    threads = os.cpu_count() or 1
    r1 = 4
    t = time.perf_counter()
    cs.render(cams[0], ng.Opts(window=(0, H // 2 - r1 // 2, W, r1)).to_c(), nthreads=1)
    one_thread_mrays = W * r1 / (time.perf_counter() - t) / 1e6
    dt, frames = 0.0, 0
    while frames < len(cams) and (frames == 0 or dt < seconds):
        t = time.perf_counter()
        cs.render(cams[frames], ng.Opts().to_c(), nthreads=threads)
        dt += time.perf_counter() - t
        frames += 1
    cs.close()
    rays = W * H * frames
    model = ""
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                model = l.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"kind": kind, "cores": threads, "rays": rays, "seconds": dt,
            "mrays_per_s": rays / dt / 1e6, "fps": frames / dt,
            "one_thread_mrays_per_s": one_thread_mrays, "cpu_model": model,
            "sample": f"{frames} full {W}x{H} frame(s) of the timed cameras, {threads} threads "
                      f"(one-thread rate from a {W}x{r1} band)"}


def run_reference(args):
    """The reference arm: the unmodified reference's CPU render path (oracle/_ref,
    the reference headers compiled in place; the C restatement when that is
    absent), on every host thread, one FULL frame of the same config and camera
    sequence per step (same_config). It loads no product library: the scene and
    cameras come from the synthetic-scene generator linked into the checker."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import paper_2407_10482_b200 as ng  # host structs only; the product .so stays unloaded
    sys.path.insert(0, str(ROOT / "tests"))
    import checkers
    from checkers import REF_SO, CpuScene
    kind = "reference" if REF_SO.exists() else "port"
    gen = checkers.ref() if kind == "reference" else checkers.oracle_synth()
    cfg = scene_config(ng, args)
    W, H = cfg["width"], cfg["height"]
    scene = ng.SynthScene(_lib=gen, **cfg)
    UNIT = f"fps ({W}x{H} frames/s, all GPUs)"
    n_cams = max(N_CAMS, int(cfg.get("n_cams", 1)))
    cams = ng.cameras(n_cams, W, H, _lib=gen)
    cs = CpuScene(scene.desc_ptr, "ref" if kind == "reference" else "oracle")
    threads = os.cpu_count() or 1
    # warm-up steps: one 8-row band each (page-in of the scene, OpenMP pool start)
    for s in range(args.warmup):
        cs.render(cams[s % n_cams], ng.Opts(window=(0, H // 2, W, 8)).to_c(), nthreads=threads)
    tot, rays = 0.0, 0
    stats_sum = None
    for i in range(args.steps):
        cam = cams[(args.warmup + i) % n_cams]  # the camera run_ours renders at this step (rank 0)
        t = time.perf_counter()
        _, st = cs.render(cam, ng.Opts().to_c(), nthreads=threads)
        tot += time.perf_counter() - t
        rays += W * H
        m = st.reshape(-1, 4).astype("float64").mean(0)
        stats_sum = m if stats_sum is None else stats_sum + m
    fps = rays / tot / (W * H)
    ms = stats_sum / max(1, args.steps)
    line = {"metric": METRIC, "value": fps, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "mrays_per_s": rays / tot / 1e6,
            "config": {"workload": f"{args.config}: {W}x{H}, host CPU reference render path "
                                   f"(canonical render_ray composition, SURVEY.md §8(c))",
                       "step": "one full frame per step, camera (warmup + i) % "
                               f"{n_cams} of sphere_views({n_cams}, 2.9), as rank 0 of the "
                               "GPU arm renders",
                       "same_config": True,
                       "mean_ray_stats": {"marching": round(float(ms[0]), 2),
                                          "occupied": round(float(ms[1]), 2),
                                          "occ_acc": round(float(ms[2]), 2),
                                          "dist_acc": round(float(ms[3]), 2)},
                       "libraries": f"{REF_SO.relative_to(ROOT) if kind == 'reference' else 'oracle/_build'}"
                                    " only (scene generator linked in; no product library)"},
            "cpu_baseline": {"value": fps, "unit": UNIT, "cores": threads, "kind": kind,
                             "sample": f"{args.steps} full {W}x{H} frames, {threads} OpenMP threads "
                                       "(rows scheduled dynamically)"},
            "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line))
    return 0


def run_tiles(args):
    """--shard tiles: single-frame latency mode (BASELINE configs 4 and 5). Every
    rank renders its interleaved tile x tile tiles of the SAME frame in one
    K0/K1/K2 launch (ngprt_render_opts.shard_*), the compact shards are gathered
    to rank 0 over NCCL and de-interleaved there (ngprt_shard_assemble). A step
    is one frame of the whole job (strong scaling)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2407_10482_b200 as ng
    from paper_2407_10482_b200 import multigpu as mg

    rank, world, local = dist_env()
    backend = os.environ.get("NGPRT_BENCH_BACKEND", "nccl")
    if os.environ.get("NGPRT_BENCH_SHARE_GPU"):
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group(backend, **({"device_id": dev} if backend == "nccl" else {}))
    cfg = scene_config(ng, args)
    W, H, T = cfg["width"], cfg["height"], args.tile
    synth = ng.SynthScene(**cfg)
    scene = ng.Scene(synth, device=local)
    info = scene.info()
    n_cams = max(N_CAMS, int(cfg.get("n_cams", 1)))
    B = max(1, args.batch)
    cams = ng.cameras(n_cams, W, H)
    opts = ng.Opts(mlp=args.mlp, profile=True)
    UNIT = f"fps ({W}x{H} frames/s, all GPUs)"
    stream = torch.cuda.current_stream(dev)
    P = ng.shard_pixels(W, H, world, T)
    gb = torch.empty((world, B, P, 3), dtype=torch.float32, device=dev) if rank == 0 else None
    sh = torch.empty((B, P, 3), dtype=torch.float32, device=dev) if world > 1 else gb[0]
    frame = torch.empty((B, H, W, 3), dtype=torch.float32, device=dev) if rank == 0 else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def cams_of(step):
        return [cams[(step * B + j) % n_cams] for j in range(B)]

    def step_fn(step):
        mg.render_tile_shard(scene, cams_of(step), opts, rank, world, T, out=sh, stream=stream)
        if world > 1:
            dist.gather(sh, gather_list=list(gb.unbind(0)) if rank == 0 else None, dst=0)
        if rank == 0:
            ng.shard_assemble(gb, world, B, W, H, T, 3, out=frame, stream=stream)

    b_store = 2 if info.storage == 2 else 4
    alg, stats_mean = {}, {}
    for s in range(args.warmup + args.steps):
        for j, c in enumerate(cams_of(s)):
            idx = (s * B + j) % n_cams
            if idx not in alg:
                _, st = ng.render(scene, [c], ng.Opts(mlp=args.mlp), stats=True)
                st = st.cpu().numpy()
                alg[idx] = algorithmic_bytes(st, scene.L, b_store, b_store)
                stats_mean[idx] = st.reshape(-1, 4).mean(0)
    for s in range(args.warmup):
        step_fn(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    k0, k1, k2, launches = [], [], [], 0
    with Clocks(local) as clk:
        for i in range(args.steps):
            if not args.no_l2_flush:
                flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            ev[i][0].record(stream)
            step_fn(args.warmup + i)
            ev[i][1].record(stream)
            torch.cuda.synchronize()
            z, a, b, n = ng.render_timing3(scene)
            k0.append(z), k1.append(a), k2.append(b)
            launches += n + (1 if rank == 0 else 0)
    total_ms = sum(e0.elapsed_time(e1) for e0, e1 in ev)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    frames = args.steps * B
    fps = frames / (total_ms / 1e3)
    # e2e: the same steps plus the D2H read of each assembled frame into pinned
    # host memory on rank 0, by wall clock (max over ranks)
    host = torch.empty((B, H, W, 3), dtype=torch.float32).pin_memory() if rank == 0 else None
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        step_fn(args.warmup + i)
        if rank == 0:
            host.copy_(frame, non_blocking=True)
    torch.cuda.synchronize()
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_fps = frames / float(t.item())
    if rank == 0:
        peak, peak_src = load_peaks()
        k1_avg = sum(k1) / len(k1)
        bytes_rank = np.mean([sum(alg[(s * B + j) % n_cams] for j in range(B))
                              for s in range(args.warmup, args.warmup + args.steps)]) / world
        achieved = bytes_rank / (k1_avg / 1e3) / 1e9
        ms = np.mean([stats_mean[(s * B + j) % n_cams] for s in range(args.warmup, args.warmup + args.steps)
                      for j in range(B)], axis=0)
        line = {
            "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": fps / PAPER_FPS,
            "dtype": "f32 (fp16 feature storage, lossless)", "data": "synthetic",
            "mrays_per_s": fps * W * H / 1e6,
            "config": {"workload": f"{args.config}: {W}x{H} '{cfg['occupancy']}' synthetic scene, "
                                   f"L={scene.L}, one frame per step split over {world} rank(s)",
                       "l2": L2_NOTE if not args.no_l2_flush
                             else "not flushed",
                       "mean_ray_stats": {k: round(float(v), 2) for k, v in
                                          zip(["marching", "occupied", "occ_acc", "dist_acc"], ms)},
                       "parallelism": f"tile sharding: interleaved {T}x{T} tiles, tile t on rank "
                                      f"t % {world}, one K0/K1/K2 launch per rank per frame, NCCL "
                                      "gather of the equal-size compact shards to rank 0, then the "
                                      "ngprt_shard_assemble de-interleave kernel"},
            "kernel_ms": {"raygen_K0": sum(k0) / len(k0), "march_K1": k1_avg,
                          "shade_K2": sum(k2) / len(k2)},
            "roofline": {"bound": "l2", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "kernel": "march_kernel (K1), rank 0",
                         "peak_source": peak_src,
                         "note": "algorithmic bytes of the frame / world per rank"},
            "e2e": {"value": e2e_fps, "unit": UNIT, "h2d_bytes_per_step": 168 * B,
                    "d2h_bytes_per_step": B * W * H * 12,
                    "timer": "wall clock: render + gather + assemble + D2H of the frame into pinned "
                             "host memory on rank 0, max over ranks"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2407_10482_b200 as ng
    from paper_2407_10482_b200 import multigpu as mg

    rank, world, local = dist_env()
    # Test hooks for the multi-rank flow on a 1-GPU box (functional only, the
    # numbers mean nothing): NGPRT_BENCH_BACKEND=gloo, NGPRT_BENCH_SHARE_GPU=1.
    backend = os.environ.get("NGPRT_BENCH_BACKEND", "nccl")
    if os.environ.get("NGPRT_BENCH_SHARE_GPU"):
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cfg = scene_config(ng, args)
    W, H = cfg["width"], cfg["height"]
    synth = ng.SynthScene(**cfg)
    scene = ng.Scene(synth, device=local)
    info = scene.info()
    # the config's camera ring (c2: the 100-camera orbit), at least 64 distinct views
    n_cams = max(N_CAMS, int(cfg.get("n_cams", 1)))
    B = max(1, args.batch)
    cams = ng.cameras(n_cams, W, H)
    opts = ng.Opts(mlp=args.mlp, profile=True)
    UNIT = f"fps ({W}x{H} frames/s, all GPUs)"
    stream = torch.cuda.current_stream(dev)
    # two frame buffers: step s renders frame s while frame s-1 is gathered to rank 0
    outs = [torch.empty((B, H, W, 3), dtype=torch.float32, device=dev) for _ in range(2)]
    gbufs = [torch.empty_like(outs[0]) for _ in range(world)] if rank == 0 else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def cam_ids(step):
        """This rank's cameras of step `step` (B consecutive frames of its share)."""
        return [mg.camera_of(rank, world, step * B + j, n_cams) for j in range(B)]

    def cams_of(step):
        return [cams[c] for c in cam_ids(step)]

    def step_fn(step, last=False):
        out = outs[step & 1]
        work = None
        if world > 1 and step > 0:
            # NCCL gather of the previous frame, overlapping this frame's render
            # (the NCCL stream waits for the work already on `stream`: frame step-1)
            _, work = mg.gather_frames(outs[(step - 1) & 1], world, bufs=gbufs, async_op=True)
        ng.render(scene, cams_of(step), opts, out=out, stream=stream)
        if work is not None:
            work.wait()  # the step ends after the transfer
        if world > 1 and last:
            mg.gather_frames(out, world, bufs=gbufs)  # the last frame's own gather, unoverlapped

    # per-camera algorithmic bytes from the bit-exact counters (untimed)
    b_store = 2 if info.storage == 2 else 4
    alg = {}
    for c in sorted({c for s in range(args.warmup + args.steps) for c in cam_ids(s)}):
        if c not in alg:
            rgb_c, st = ng.render(scene, [cams[c]], ng.Opts(mlp=args.mlp), stats=True)
            st = st.cpu().numpy()
            shaded = int((rgb_c != 0).any(-1).sum().item())  # final_t < 1 rays (the rest are black)
            alg[c] = (algorithmic_bytes(st, scene.L, b_store, b_store), st.reshape(-1, 4).mean(0),
                      shaded)
    for s in range(args.warmup):
        step_fn(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    k0_ms, k1_ms, k2_ms, launches, bytes_k1 = [], [], [], 0, 0.0
    with Clocks(local) as clk:
        for i in range(args.steps):
            s = args.warmup + i
            if not args.no_l2_flush:
                flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            ev[i][0].record(stream)
            step_fn(s, last=i == args.steps - 1)
            ev[i][1].record(stream)
            torch.cuda.synchronize()
            z, a, b, n = ng.render_timing3(scene)
            k0_ms.append(z)
            k1_ms.append(a)
            k2_ms.append(b)
            launches += n
            bytes_k1 += sum(alg[c][0] for c in cam_ids(s))
    total_ms = sum(e0.elapsed_time(e1) for e0, e1 in ev)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    frames = args.steps * world * B
    fps = frames / (total_ms / 1e3)

    # ---- e2e through the host-buffer C ABI (H2D camera, D2H RGB inside) ----
    # (a) the serving call: ngprt_render_host_async per frame, two frames in
    #     flight, so frame i's 24.9 MB device->host copy (copy engine) overlaps
    #     frame i+1's march; ngprt_render_host_wait at the end. Timed by wall
    #     clock from the first enqueue to the wait. No L2 flush can sit between
    #     pipelined frames: the scene (4.46 GB) and each frame's DRAM reads
    #     (~1.5 GB) exceed the 126 MB L2.
    # (b) the synchronous call ngprt_render_host per frame (L2 flushed before
    #     each), reported as e2e_sync.
    opts_e2e = ng.Opts(mlp=args.mlp)
    host_bufs = [torch.empty((B, H, W, 3), dtype=torch.float32).pin_memory().numpy()
                 for _ in range(2)]
    for s in range(min(2, args.warmup)):
        ng.render_host(scene, cams_of(s), opts_e2e, out=host_bufs[0])
        ng.render_host_async(scene, cams_of(s), host_bufs[s & 1], opts_e2e)
    ng.render_host_wait(scene)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        ng.render_host_async(scene, cams_of(args.warmup + i), host_bufs[i & 1], opts_e2e)
    ng.render_host_wait(scene)
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_fps = frames / float(t.item())

    e2e_sync_s = 0.0
    for i in range(args.steps):
        if not args.no_l2_flush:
            flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        ng.render_host(scene, cams_of(args.warmup + i), opts_e2e, out=host_bufs[0])
        e2e_sync_s += time.perf_counter() - t0
    t = torch.tensor([e2e_sync_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_sync_fps = frames / float(t.item())

    if rank == 0:
        peak, peak_src = load_peaks()
        k1_avg = sum(k1_ms) / len(k1_ms)
        achieved = (bytes_k1 / args.steps) / (k1_avg / 1e3) / 1e9
        traffic = l2_traffic = None
        tj = {}
        tp = ROOT / "profiles" / "ncu_traffic.json"
        if tp.exists():
            tj = json.loads(tp.read_text()).get(args.config, {})
            traffic = tj.get("dram_bytes_per_launch")
            l2_traffic = tj.get("l2_bytes_per_launch")
        # also report K1 against the L2 and random-gather ceilings
        # measured on this B200 (tools/measure_peaks.cu -> profiles/*_peaks.json)
        ceilings = None
        pk = sorted((ROOT / "profiles").glob("*_peaks.json"))
        if pk:
            pj = json.loads(pk[-1].read_text())
            ceilings = {k: {"peak_gbs": pj[k], "frac": achieved / pj[k]}
                        for k in ("l2_read_gbs", "l2_gather32_gbs", "l2_gather16_gbs",
                                  "hbm_gather32_gbs") if k in pj}
            ceilings["source"] = f"profiles/{pk[-1].name} ({pj.get('method', '')})"
        shaded = np.mean([sum(alg[c][2] for c in cam_ids(args.warmup + i))
                          for i in range(args.steps)])
        k2_avg = sum(k2_ms) / len(k2_ms)
        k2_flop = 11520.0 * shaded  # 11,520 FLOP per shaded ray
        mean_stats = np.mean([alg[c][1] for i in range(args.steps)
                              for c in cam_ids(args.warmup + i)], axis=0)
        line = {
            "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": fps / PAPER_FPS,
            "dtype": "f32 (fp16 feature storage, lossless)", "data": "synthetic",
            "mrays_per_s": fps * W * H / 1e6,
            "config": {"workload": (
                f"{args.config}: {W}x{H} '{cfg['occupancy']}' synthetic scene"
                + (f" ({cfg['n_boxes']} boxes)" if cfg['occupancy'] == 'boxes' else "")
                + f", L={scene.L}, 2^{int(cfg['fine_table_len']).bit_length() - 1} entries/level, "
                f"L_C={cfg['L_C']}, {cfg['occ_base_res']}^3 pyramid, "
                f"{int(synth.desc.dist_res)}^3 distance grid, occupancy "
                f"{100 * synth.occupancy_fraction():.2f}%, mlp={args.mlp}"),
                       "cameras": f"sphere_views({n_cams}, 2.9); rank r renders cameras "
                                  f"(r + N*(step*{B} + j)) % {n_cams}, j < {B} per step"
                                  + (f" (one ngprt_render call of {B} cameras)" if B > 1 else ""),
                       "l2": L2_NOTE if not args.no_l2_flush
                             else "not flushed; scene (4.4 GB) larger than L2",
                       "mean_ray_stats": {"marching": round(float(mean_stats[0]), 2),
                                          "occupied": round(float(mean_stats[1]), 2),
                                          "occ_acc": round(float(mean_stats[2]), 2),
                                          "dist_acc": round(float(mean_stats[3]), 2)},
                       "scene_device_bytes": int(info.device_bytes),
                       "counters": "timed renders request no per-ray MarchCounters (stats = NULL, "
                                   "so K1 compiles the counter updates out); mean_ray_stats and the "
                                   "algorithmic bytes come from an untimed render of the same "
                                   "frames with counters (bit-identical images)",
                       "parallelism": f"dp{world} (camera sharding; NCCL gather of frame s-1 to "
                                      "rank 0 overlaps the render of frame s; the last step also "
                                      "gathers its own frame)"},
            "kernel_ms": {"raygen_K0": sum(k0_ms) / len(k0_ms), "march_K1": k1_avg,
                          "shade_K2": k2_avg},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": "march_kernel (K1)",
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": bytes_k1 / args.steps,
                         "l2_traffic": l2_traffic, "other_ceilings": ceilings,
                         # measured bytes (ncu, same build, profiles/ncu_traffic.json) over
                         # this run's K1 event time, and the ceiling that binds
                         "l2_gbs": (l2_traffic / (k1_avg / 1e3) / 1e9) if l2_traffic else None,
                         "dram_gbs": (traffic / (k1_avg / 1e3) / 1e9) if traffic else None,
                         "binding_ceiling": binding_ceiling(tj, k1_avg, ceilings)},
            "k2_tensor": {"kernel": "shade_tc_pipe_kernel (K2)" if args.mlp == "tensor" else "shade_exact_kernel",
                          "shaded_rays": int(shaded), "flop_per_launch": k2_flop,
                          "achieved_tflops": k2_flop / (k2_avg * 1e-3) / 1e12,
                          "peak_tflops": load_tensor_peak(),
                          "note": "psi FLOP (23-64-64-3); the tensor path issues 3 bf16 products "
                                  "per FLOP (hi/lo split) and runs layer 3 on CUDA cores"},
            "e2e_sync": {"value": e2e_sync_fps, "unit": UNIT,
                         "api": "ngprt_render_host per frame (pinned host RGB, L2 flushed before each)"},
            "e2e": {"value": e2e_fps, "unit": UNIT, "h2d_bytes_per_step": 168 * B,
                    "d2h_bytes_per_step": B * W * H * 12,
                    "ms_per_step": 1e3 * frames / e2e_fps / args.steps,
                    "timer": "host wall clock from the first enqueue to ngprt_render_host_wait "
                             "returning (every frame's RGB is in pinned host memory); close to the "
                             "device value because each 24.9 MB copy runs on the copy engine while "
                             "the next frame marches (e2e_sync shows the unpipelined call)",
                    "api": "ngprt_render_host_async per frame, 2 frames in flight, "
                           "ngprt_render_host_wait at the end (pinned host RGB buffers)",
                    "l2": "not flushed between pipelined frames: scene 4.46 GB and ~1.5 GB of "
                          "DRAM reads per frame exceed the 126 MB L2"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_sample(synth, [cams_of(args.warmup + i)[0] for i in range(args.steps)], W, H,
                            args.cpu_seconds)
            line["cpu_baseline"] = {"value": cb["fps"], "unit": UNIT, "cores": cb["cores"],
                                    "kind": cb["kind"], "sample": cb["sample"],
                                    "mrays_per_s": cb["mrays_per_s"],
                                    "one_thread_mrays_per_s": cb["one_thread_mrays_per_s"],
                                    "cpu_model": cb["cpu_model"]}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def launch_ranks(args) -> int:
    """`--gpus N` without a torch.distributed launcher: re-launch this script as N
    ranks (torch.distributed.run, one process per GPU, NCCL, rendezvous on
    127.0.0.1). Fails loudly when fewer than N GPUs are visible, unless
    NGPRT_BENCH_SHARE_GPU=1 (a functional test of the multi-rank flow on one GPU)."""
    import socket
    import torch
    n_vis = torch.cuda.device_count()
    if n_vis < args.gpus and not os.environ.get("NGPRT_BENCH_SHARE_GPU"):
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found "
                         f"{n_vis} (set NGPRT_BENCH_SHARE_GPU=1 to run the ranks on one GPU "
                         "for a functional test)\n")
        return 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)  # rank 0 only; other ranks exit at once
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args)
    _, world, _ = dist_env()
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        return 2
    return run_tiles(args) if args.shard == "tiles" else run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
