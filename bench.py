#!/usr/bin/env python
"""Benchmark: path samples/s and Mrays/s at 1080p, depth 8, on 1/2/4/8 GPUs,
vs the CPU reference path (BASELINE.json `metric`).

Workload (BASELINE.json configs[3]): the ~1.06 M-triangle
procedural pushbutton assembly with mixed OpenPBR materials (coat, glass,
metal, dielectric, emissive) under a synthetic HDR sky, 1920x1080, 256 spp,
max_depth 8, rr_start 3.  One step = one full frame (W*H*spp paths) tiled
across the ranks (interleaved 16x16 tiles) plus the NCCL merge onto rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

`--impl reference` times the reference's algorithm on the host cores: the
float64 C restatement in oracle/ (the reference is Python/numba and is not
installed on the GPU box), all threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "path samples/s and Mrays/s at 1080p depth 8 (1/2/4/8 GPU) vs CPU ref"
UNIT = "samples/s"
HBM_FALLBACK_GBS = 6650.0


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", default="pushbutton")
    p.add_argument("--width", type=int, default=1920)
    p.add_argument("--height", type=int, default=1080)
    p.add_argument("--spp", type=int, default=256)
    p.add_argument("--depth", type=int, default=8)
    p.add_argument("--rr-start", type=int, default=3)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--tile", type=int, default=16)
    p.add_argument("--mode", choices=["tiles", "spp"], default="tiles",
                   help="multi-GPU split: interleaved tiles or contiguous sample ranges")
    p.add_argument("--config", choices=["c4", "c5"], default="c4",
                   help="c5 = BASELINE configs[4]: 3840x2160, 1024 spp, spp split")
    p.add_argument("--flags", type=int, default=0)
    p.add_argument("--bvh-bins", type=int, default=12,
                   help="SAH bins of the scene BVH (12 = the reference's build_bvh)")
    p.add_argument("--bvh-leaf", type=int, default=4,
                   help="leaf size of the scene BVH (4 = the reference's build_bvh)")
    p.add_argument("--batch-paths", type=int, default=0,
                   help="paths per wavefront batch (0 = library default)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-variant", action="store_true",
                   help="skip the reference-lobe variant measurement")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--ref-step-seconds", type=float, default=6.0)
    a = p.parse_args()
    if a.config == "c5":
        a.width, a.height, a.spp, a.mode = 3840, 2160, 1024, "spp"
    return a


def workload_config(args, n_tris: int, world: int) -> dict:
    desc = {
        "pushbutton": "C4: procedural CAD pushbutton assembly, mixed OpenPBR materials "
                      "(metal, dielectric, coat, glass, emissive) + synthetic HDR sky",
        "pushbutton_ref": "C4 (reference lobes only, gradient sky)",
        "sphere70k": "C3: bumpy_sphere(70k) on a metal plane, gradient sky",
        "cornell_c2": "C2: Cornell box, metal + glossy dielectric boxes",
        "cornell_c2x": "C2: Cornell box, metal + coat + glass boxes",
    }.get(args.workload, args.workload)
    return {
        "workload": f"{desc}, {n_tris} triangles, {args.width}x{args.height}, {args.spp} spp, "
                    f"max_depth {args.depth}",
        "scene": args.workload, "triangles": n_tris, "width": args.width,
        "height": args.height, "spp": args.spp, "max_depth": args.depth,
        "rr_start_depth": args.rr_start, "seed": args.seed,
        "parallelism": ((f"tiles{args.tile}x{world}" if args.mode == "tiles" else f"spp/{world}")
                        if world > 1 else "single"),
        "l2": "no explicit flush: every step streams ~8 GB of wavefront queues and path "
              "state through L2 (126 MB); the hot part of the traversal set stays L2-resident "
              "through ordinary caching, as in any steady-state render",
    }


def build_workload(args, device="auto"):
    """The scene and its BVH (the reference's tree; device=None builds it
    with the host restatement -- the reference arm never touches the GPU)."""
    from workloads import scene_by_name
    from paper_2407_19977_b200 import build_bvh
    scene = scene_by_name(args.workload, width=args.width, height=args.height)
    bvh = build_bvh(scene.triangles, leaf_size=args.bvh_leaf, bins=args.bvh_bins, device=device)
    return scene, bvh


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region."""
    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw",
              "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "200", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in self.rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in self.rows if num(r[2]) is not None]
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for name, val in zip(names, r[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ------------------------------------------------------------------ helpers

def measured_peak():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            return float(json.loads(f.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def cpu_baseline(args, seconds: float) -> dict:
    """The float64 oracle (the reference's algorithm restated in C) on a
    bounded pixel sample of the workload's reference-lobe variant (what the
    reference can render), all host threads."""
    from oracle.oracle import default_threads
    name, _, oc, cam = reference_setup(args)
    w, h = args.width, args.height
    threads = default_threads()
    n = min(w * h, max(threads * 256, 8192))
    paths = 0
    segs = 0
    t_total = 0.0
    sample = 0
    rng = np.random.default_rng(1)
    while t_total < seconds:
        pix = np.sort(rng.choice(w * h, size=min(n, w * h), replace=False))
        t0 = time.perf_counter()
        _, seg = oc.sample_values(pix, sample, cam, w, h, args.seed, args.depth, args.rr_start,
                                  1e-4, threads)
        dt = time.perf_counter() - t0
        t_total += dt
        paths += pix.size
        segs += int(seg.sum())
        sample += 1
        if dt < seconds / 8:
            n = min(w * h, n * 2)
    return {"value": paths / t_total, "unit": UNIT, "cores": threads, "kind": "port",
            "mrays_per_s": segs / t_total / 1e6,
            "sample": f"{paths} random (pixel, sample) paths of the {name!r} frame (same settings) "
                      f"over {sample} sample indices, {t_total:.1f} s on {threads} threads "
                      f"(oracle/lt_oracle.c, float64 restatement of the reference)"}


# ------------------------------------------------------------------ arms

# The reference (luxtrace) has no coat / transmission lobe and no HDR
# environment: it renders a workload's reference-lobe
# variant -- same geometry and camera, coat -> base, glass -> dielectric
# specular, HDR sky -> the bench gradient.
REFERENCE_VARIANT = {"pushbutton": "pushbutton_ref", "cornell_c2x": "cornell_c2"}


def reference_setup(args):
    """The CPU reference's inputs: the workload's reference-lobe variant from
    workloads.py, its tree from oc_build_bvh (= build_bvh, bvh.py:286-298),
    the oracle scene and the packed camera; the product is not involved."""
    import workloads
    from oracle.oracle import OracleScene, camera_pack
    from oracle.oracle import build_bvh as oracle_build_bvh
    name = REFERENCE_VARIANT.get(args.workload, args.workload)
    scene = workloads.scene_by_name(name, width=args.width, height=args.height)
    bvh = oracle_build_bvh(scene.triangles, leaf_size=args.bvh_leaf, bins=args.bvh_bins)
    return name, scene, OracleScene.from_scene(scene, bvh), camera_pack(scene.camera)


def run_reference(args, rank: int, world: int) -> None:
    """The reference's algorithm on the host cores: the float64 C
    restatement in oracle/, all threads; the product package is never
    imported."""
    if rank != 0:
        return
    from oracle.oracle import default_threads
    name, scene, oc, cam = reference_setup(args)
    w, h = args.width, args.height
    threads = default_threads()
    rng = np.random.default_rng(2)
    # calibrate the per-step pixel sample to about --ref-step-seconds
    n = min(4096, w * h)
    while True:
        pix = np.sort(rng.choice(w * h, size=n, replace=False))
        t0 = time.perf_counter()
        oc.sample_values(pix, 0, cam, w, h, args.seed, args.depth, args.rr_start, 1e-4, threads)
        dt = time.perf_counter() - t0
        if dt > 0.5 or n >= w * h:
            n = int(min(w * h, max(min(1024, w * h), n * args.ref_step_seconds / max(dt, 1e-3))))
            break
        n = min(w * h, n * 4)
    times, segs = [], []
    for step in range(args.warmup + args.steps):
        pix = np.sort(rng.choice(w * h, size=n, replace=False))
        t0 = time.perf_counter()
        _, seg = oc.sample_values(pix, step % args.spp, cam, w, h, args.seed, args.depth,
                                  args.rr_start, 1e-4, threads)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
            segs.append(int(seg.sum()))
    total = sum(times)
    value = n * args.steps / total
    cfg = workload_config(args, len(scene.triangles), world)
    if name != args.workload:
        cfg["scene"] = name
        cfg["workload"] = (f"{cfg['workload']} -- rendered as its reference-lobe variant "
                           f"{name!r} (same geometry and camera; the reference has no coat, "
                           f"glass or HDR environment)")
    sample = (f"each step: {n} random pixels x 1 sample of the {w}x{h} frame "
              f"({n / (w * h) / args.spp:.2e} of the full {args.spp}-spp workload)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg, "mrays_per_s": sum(segs) / total / 1e6,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def trace_source_sha() -> str:
    """Hash of the trace kernel's sources with comments and blank space
    removed: ties committed ncu figures to the kernel code that is timed
    (a comment edit does not make them stale, a code edit does)."""
    import hashlib
    import re
    h = hashlib.sha256()
    for f in ("lt_traverse.cuh", "lt_device.cuh", "lt_kernels.cu", "lt_kernels.h"):
        src = (ROOT / "paper_2407_19977_b200" / "csrc" / f).read_text()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        src = re.sub(r"//[^\n]*", "", src)
        h.update("\n".join(ln.strip() for ln in src.splitlines() if ln.strip()).encode())
    return h.hexdigest()[:16]


def ncu_trace_figures(workload: str):
    """Per-ray traffic per memory level and unit utilisations of k_trace
    from the committed ncu capture (profiles/trace_ncu.json, written by
    tools/trace_ncu.py), if it was taken on the kernel sources timed here."""
    f = ROOT / "profiles" / "trace_ncu.json"
    if not f.exists():
        return None, "no profiles/trace_ncu.json"
    d = json.loads(f.read_text()).get(workload)
    if not d:
        return None, f"no ncu capture for {workload!r}"
    if d.get("source_sha") != trace_source_sha():
        return None, (f"stale: ncu capture of kernel sources {d.get('source_sha')}, timed "
                      f"{trace_source_sha()}")
    return d, d.get("source")


def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2407_19977_b200 import RenderSettings, build_bvh, render_progressive
    from paper_2407_19977_b200._lib import LT_FLAG_COUNT, LT_FLAG_PROFILE, read_bandwidth
    from paper_2407_19977_b200.device import DeviceScene
    from paper_2407_19977_b200.distributed import (merge_spp_ordered, merge_tiles,
                                                   render_distributed, spp_range)
    from paper_2407_19977_b200.integrator import Accumulator, render_pass_device

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    scene, bvh = build_workload(args)
    settings = RenderSettings(samples_per_pixel=args.spp, max_depth=args.depth,
                              rr_start_depth=args.rr_start, seed=args.seed)
    l2_gbs = read_bandwidth(local_rank, 32 << 20, 10)      # 32 MB: L2-resident
    hbm_probe = read_bandwidth(local_rank, 4 << 30, 5)      # 4 GB: HBM
    shard = (rank, world, args.tile) if world > 1 and args.mode == "tiles" else None
    stream = torch.cuda.current_stream(dev)
    samples_per_step = args.width * args.height * args.spp

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def stepper(ds_, acc_):
        def step(flags, spp=None):
            acc_.sum.zero_()
            acc_.valid.zero_()
            acc_.invalid.zero_()
            n = spp or args.spp
            if args.mode == "spp":
                lo, hi = spp_range(n, rank, world)
                render_pass_device(ds_, ds_.camera, settings, acc_, lo, hi - lo,
                                   flags=flags | args.flags, max_batch_paths=args.batch_paths,
                                   stream=stream)
                if world > 1:
                    merge_spp_ordered(acc_, dst=0)
                return
            render_pass_device(ds_, ds_.camera, settings, acc_, 0, n, flags=flags | args.flags,
                               shard=shard, max_batch_paths=args.batch_paths, stream=stream)
            if world > 1:
                merge_tiles(acc_, dst=0)
        return step

    def timed(step, n, flags, sampler=None):
        """n steps between CUDA events on the launching stream, barrier +
        synchronize on both sides; returns the max over ranks in ms."""
        torch.cuda.synchronize(dev)
        barrier()
        if sampler:
            sampler.start()
            time.sleep(0.3)
        torch.cuda.synchronize(dev)
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(n):
            step(flags)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        clocks = sampler.stop() if sampler else None
        return max_over_ranks(ev0.elapsed_time(ev1)), clocks

    def e2e_of(scene_, bvh_, n):
        """The metric through the public API, as a luxtrace caller makes it:
        the scene's plain (pageable) numpy arrays uploaded by every call,
        the image back as float64 means; wall clock, max over ranks."""
        def call():
            if world > 1:
                return render_distributed(scene_, settings, bvh_, tile_size=args.tile,
                                          mode=args.mode, device=local_rank)
            return render_progressive(scene_, settings, bvh=bvh_, device=local_rank)
        call()
        torch.cuda.synchronize(dev)
        barrier()
        t0 = time.perf_counter()
        phases = []
        for _ in range(n):
            res = call()
            if res is not None and hasattr(res, "timings"):
                phases.append(res.timings)
        torch.cuda.synchronize(dev)
        el = max_over_ranks(time.perf_counter() - t0)
        env = scene_.environment
        h2d = env.texels.nbytes if getattr(env, "texels", None) is not None else 0
        h2d += sum(getattr(scene_.triangles, nm).nbytes for nm in
                   ["v0", "v1", "v2", "n0", "n1", "n2", "material_index"])
        h2d += sum(getattr(bvh_, nm).nbytes for nm in
                   ["bounds_min", "bounds_max", "left_child", "right_child", "first_triangle",
                    "triangle_count", "triangle_order"])
        return {"value": samples_per_step * n / el, "unit": UNIT,
                "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(args.width * args.height * (3 * 8 + 8))
                if rank == 0 else 0,
                "steps": n, "ms_per_step": 1e3 * el / n,
                "phases_ms": {k: statistics.mean(p[k] for p in phases) for k in phases[0]}
                if phases else None,
                "api": "render_progressive(scene, settings, bvh) (render_distributed for N>1): "
                       "scene upload from the caller's pageable numpy arrays + BVH flatten + "
                       "render + image D2H, wall clock"}

    ds = DeviceScene(scene, bvh, device=local_rank)
    acc = Accumulator(scene.camera.width, scene.camera.height, local_rank)
    step = stepper(ds, acc)

    # untimed: work counters (same paths, reduced spp)
    step(LT_FLAG_COUNT, min(args.spp, 16))
    torch.cuda.synchronize(dev)
    cst = ds.stats()
    slab_per_ray = cst["slab_tests"] / max(1, cst["rays"])
    tri_per_ray = cst["tri_tests"] / max(1, cst["rays"])
    # 32 B per child-box test, 48 B per triangle test, 32 B ray
    # in + 16 B hit out
    bytes_per_ray = 32.0 * slab_per_ray + 48.0 * tri_per_ray + 48.0

    for _ in range(args.warmup):
        step(0)
    ms_max, clocks = timed(step, args.steps, LT_FLAG_PROFILE,
                           ClockSampler(local_rank) if rank == 0 else None)
    st = ds.stats()    # the last timed step on this rank
    rays_per_step = sum_over_ranks(st["rays"])
    value = samples_per_step * args.steps / (ms_max / 1e3)
    mrays = rays_per_step * args.steps / (ms_max / 1e3) / 1e6

    # roofline of the dominant kernel (closest-hit traversal), this rank:
    # measured bytes per memory level (ncu, same kernel sources) over the
    # live trace time, against the measured HBM and L2 rates
    peak, peak_src = measured_peak()
    trace_ms = st["trace_ms"]
    launches = max(1, st["trace_launches"])
    rays_s = st["rays"] / (trace_ms / 1e3) if trace_ms > 0 else None
    ncu, ncu_src = ncu_trace_figures(args.workload)
    level = {}
    if ncu and rays_s:
        level = {
            "hbm": {"achieved": ncu["dram_bytes_per_ray"] * rays_s / 1e9, "peak": peak,
                    "unit": "GB/s", "peak_source": peak_src},
            "l2": {"achieved": ncu["l2_bytes_per_ray"] * rays_s / 1e9, "peak": l2_gbs,
                   "unit": "GB/s", "peak_source": "measured in this run (32 MB streaming "
                                                 "read, lt_read_bandwidth)"},
        }
        for v in level.values():
            v["frac"] = v["achieved"] / v["peak"]
    roofline = {
        "bound": "l2", "kernel": "k_trace (closest-hit BVH traversal)",
        "achieved": level["l2"]["achieved"] if level else None,
        "peak": l2_gbs, "unit": "GB/s",
        "frac": level["l2"]["frac"] if level else None,
        "traffic": (ncu["dram_bytes_per_ray"] * st["rays"] / launches) if ncu else None,
        "levels": level or None,
        "binding_unit": ({"unit": "L1 data pipe (LSU wavefronts)",
                          "l1_wavefront_pct": ncu.get("l1_wavefront_pct"),
                          "fma_pipe_pct": ncu.get("fma_pipe_pct"),
                          "alu_pipe_pct": ncu.get("alu_pipe_pct"),
                          "issue_active_pct": ncu.get("issue_active_pct"),
                          "simt_threads_per_warp_instruction": ncu.get("simt_threads")}
                         if ncu else None),
        "ncu_source": ncu_src, "kernel_source_sha": trace_source_sha(),
        "algorithmic_bytes_per_ray": bytes_per_ray, "slab_tests_per_ray": slab_per_ray,
        "tri_tests_per_ray": tri_per_ray, "trace_launches_per_step": launches,
        "trace_ms_per_step": trace_ms, "trace_share_of_step": trace_ms / (ms_max / args.steps),
        "hbm_read_gbs_probe": hbm_probe,
        "note": "frac = measured L2 bytes (ncu lts__t_bytes per ray x live ray rate) over the "
                "measured L2 streaming-read rate; the traversal set is served from L2/L1, so HBM "
                "carries little of it (levels.hbm); the unit that bounds k_trace is the L1 data "
                "pipe: one wavefront per lane per divergent node load (binding_unit)",
    }

    e2e = e2e_of(scene, bvh, max(1, min(args.steps, 5))) if not args.no_e2e else None

    # the same frame on the scene the CPU reference renders (the workload's
    # reference-lobe variant), device-timed and end to end: the like-for-like
    # comparison with `--impl reference`
    variant = None
    vname = REFERENCE_VARIANT.get(args.workload)
    if vname and not args.no_variant:
        import workloads
        vscene = workloads.scene_by_name(vname, width=args.width, height=args.height)
        vbvh = build_bvh(vscene.triangles, leaf_size=args.bvh_leaf, bins=args.bvh_bins)
        vds = DeviceScene(vscene, vbvh, device=local_rank)
        vstep = stepper(vds, acc)
        for _ in range(2):
            vstep(0)
        n_v = max(1, min(args.steps, 10))
        vms, _ = timed(vstep, n_v, 0)
        variant = {"workload": vname, "value": samples_per_step * n_v / (vms / 1e3),
                   "unit": UNIT, "steps": n_v, "ms_per_step": vms / n_v,
                   "e2e": e2e_of(vscene, vbvh, max(1, min(args.steps, 3)))
                   if not args.no_e2e else None}
        vds.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "fp32", "data": "synthetic",
            "config": workload_config(args, len(scene.triangles), world),
            "mrays_per_s": mrays, "rays_per_step": rays_per_step,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "reference_variant": variant, "parity": parity_summary(), "clocks": clocks,
            "gpu_launches": int(st["kernel_launches"] * args.steps),
        }
        print(json.dumps(line), flush=True)


def parity_summary():
    """The committed parity record (profiles/parity_r02.json, written by the
    -m gpu parity tests on the B200): agreement fractions and id-mismatch
    counts per fixture."""
    f = ROOT / "profiles" / "parity_r02.json"
    if not f.exists():
        return None
    d = json.loads(f.read_text())
    return {"source": "profiles/parity_r02.json", "entries": len(d.get("entries", {})),
            "headline": d.get("headline")}


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # LT_BENCH_BACKEND=gloo with LT_BENCH_SHARE_GPU=1 runs the multi-rank
        # code path with every rank on the available GPU(s) and the merge
        # staged through host memory (functional check on a 1-GPU box: the
        # ranks' kernels never wait on each other).  Timing runs use NCCL,
        # one GPU per rank.
        backend = os.environ.get("LT_BENCH_BACKEND", "nccl")
        if os.environ.get("LT_BENCH_SHARE_GPU") == "1":
            local_rank = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
