#!/usr/bin/env python
"""bench.py — ETD2RK-DS spectral time stepping on B200 (driver contract).

Default workload: BASELINE config 4 — 3D coupled FitzHugh–Nagumo, n=1023
interior points per axis (1.07e9 points per species), tau=0.05, P02, seeded
inputs.  A "step" is one ETD2RK-DS time step of both species (13 eigenbasis
transforms each).  Metric: grid-point updates per second
(one species value advanced one step), FP64.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config C] [--n N] [--no-cpu] [--dry-run]

--gpus N > 1 without torchrun's WORLD_SIZE in the environment re-launches this
script as N ranks (torch.distributed.run, one process per GPU, 127.0.0.1
rendezvous); under torchrun each rank shards config 4's z-slabs over NCCL.
--dry-run does no device work: the ranks rendezvous over gloo, check the
per-rank device-memory budget of the sharded plan (etd_plan_device_bytes) and
rank 0 prints the line it would measure with (n_gpus, parallelism, ranks seen).

--impl reference times the reference's own CPU implementation (oracle/_ref,
the unmodified etdrd core + OpenBLAS) on this host's cores, as a bounded
sample of the same workload (see oracle/ref_driver.cpp ref_sample_step).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.19  # measured DMMA.8x8x4 peak, profiles/r01_fp64_peak.jsonl (MEASURED_PEAKS has no FP64)
FP64_PEAK_NOTE = "measured: tools/fp64_peak.cu DMMA m8n8k4 sustained on this pool's B200 (profiles/r01_fp64_peak.jsonl)"


def hbm_peak():
    """HBM roofline denominator: MEASURED_PEAKS.json's hbm_gbs (driver-measured copy
    bandwidth on this pool), else B200_PROFILING.md's stated fallback."""
    try:
        v = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
    except (OSError, ValueError, KeyError, TypeError):
        return 6650.0, "of fallback: B200_PROFILING.md 6.65 TB/s (MEASURED_PEAKS.json absent)"


HBM_PEAK_GBS, HBM_PEAK_NOTE = hbm_peak()


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        load = [s for s in sm if s > 300] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


# ------------------------------------------------------------------ CPU reference (bounded sample)
def cpu_reference_sample(cfg, n, reps: int, warmup: int = 1):
    """Reference etdrd step (oracle/_ref + OpenBLAS, all host cores) on a bounded
    sample at full pencil length; returns (pt_upd_per_s list, cores, sample text)."""
    from oracle import Ref
    cores = os.cpu_count() or 1
    Ref.set_threads(cores)
    nsub = 16 if n >= 512 else max(4, n // 16)
    src_kind, params = (1, None) if cfg.nspecies == 1 else (10, (0.1, 0.01, 0.5))
    rates = []
    for i in range(warmup + reps):
        sec, pts, parts = Ref.sample_step(n, nsub, cfg.nspecies, cfg.tau, cfg.kappa, cfg.q, src_kind, params)
        if i >= warmup:
            rates.append(pts / sec)
    sample = (f"reference etdrd step ({'make_plan+advance' if cfg.nspecies == 1 else 'composed 3D system step'}, "
              f"OpenBLAS {cores} threads) on a {n}x{n}x{nsub} z-sub-box, z-applies re-timed on full-length "
              f"(n={n}) z-pencils; rate = sample points / estimated step time")
    return rates, cores, sample


def reference_arm(args, cfg, n, rank, world):
    if rank != 0:
        return 0
    steps, warmup = args.steps, args.warmup
    from oracle import Ref
    if not Ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libetdrd_ref.so not built"}))
        return 0
    if cfg.dim == 2:
        # full reference steps fit: time make_plan+advance directly
        from paper_2601_06849_b200 import configs
        cores = os.cpu_count() or 1
        Ref.set_threads(cores)
        u0 = configs.initial_state(cfg, n)[0]
        Ref.scalar_run(cfg.dim, n, cfg.tau, cfg.kappa[0], cfg.q, u0, warmup, src_kind=1)
        _, _, _, sec = Ref.scalar_run(cfg.dim, n, cfg.tau, cfg.kappa[0], cfg.q, u0, steps, src_kind=1)
        rate = n ** 2 * steps / sec
        ms = sec / steps * 1e3
        sample = f"reference make_plan+advance, full {n}x{n} grid, {steps} steps, OpenBLAS {cores} threads"
    else:
        rates, cores, sample = cpu_reference_sample(cfg, n, steps, warmup)
        rate = statistics.median(rates)
        ms = cfg.points(n) * cfg.nspecies / rate * 1e3
    unit = "grid-point updates/s"
    line = {"metric": "grid-point updates/sec (FP64)", "value": rate, "unit": unit, "impl": "reference",
            "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "config": workload_config(cfg, n, world),
            "cpu_baseline": {"value": rate, "unit": unit, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": rate, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(cfg, n, world):
    return {"workload": f"BASELINE config {cfg.id}: " + cfg.describe().split(": ", 1)[1].replace(f"n={cfg.n}", f"n={n}"),
            "grid": [n] * cfg.dim, "species": cfg.nspecies, "points_per_species": n ** cfg.dim,
            "tau": cfg.tau, "pade": "P02", "parallelism": f"zslab{world}" if world > 1 else "single",
            "l2": "inputs larger than L2" if n ** cfg.dim * 8 > 126e6 else "L2-resident working set (no flush)"}


# ------------------------------------------------------------------ B200 arm
def b200_arm(args, cfg, n, rank, world, local_rank):
    import numpy as np
    import torch
    from paper_2601_06849_b200 import configs

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    kw = {}
    if world > 1:
        if cfg.dim != 3:
            raise SystemExit("2D configs are not sharded (replicas only); use a 3D config for N>1")
        from paper_2601_06849_b200 import nccl_unique_id
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        kw = {"world_size": world, "rank": rank, "nccl_id": obj[0]}
    plan = configs.make_plan(cfg, n, device=local_rank, **kw)
    comm_ranks = plan.comm_ranks()  # ncclCommCount of the plan's communicator when sharded
    from paper_2601_06849_b200 import etd as E
    dev_bytes = E.plan_device_bytes(plan.grid, cfg.nspecies, world, rank)
    t0 = time.time()
    ics = configs.initial_state(cfg, n, z0=plan.slab[0], z1=plan.slab[1] if cfg.dim == 3 else None)
    t_ic = time.time() - t0
    for s, a in enumerate(ics):
        plan.upload(s, a)
    stream = torch.cuda.ExternalStream(plan.stream, device=torch.device("cuda", local_rank))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (also builds the CUDA graphs)
    plan.step(args.warmup)
    barrier()

    # ---- timed region: device-resident inputs, events on the launching stream ----
    plan.set_profiling(True)  # per-launch events (eager launches; each launch >> launch latency at this size)
    clocks = ClockSampler(local_rank)
    clocks.start()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    plan.step(args.steps)
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    stats = plan.stage_stats()
    parity = list(plan.parity_split())
    fold_level = list(plan.fold_level())
    plan.set_profiling(False)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_pts = cfg.points(n) * cfg.nspecies
    value = total_pts / (ms * 1e-3)

    # roofline of the dominant kernel (largest share of the step)
    per = []
    for s in stats:
        avg = s["ms_total"] / max(1, s["launches"])
        per.append((avg, s))
    if dist is not None:  # slowest rank's per-stage times
        t = torch.tensor([p[0] for p in per], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        per = [(float(a), s) for a, (_, s) in zip(t.tolist(), per)]
    # The dominant kernel is the transform family with the largest share of the step:
    # the forward contractions (etd_contract, FOLD 5 / 4 launches of equal FLOPs) or the
    # fused backward launches (etd_back6); achieved = its executed FLOPs per launch over
    # its average launch time.  The slowest single launch is reported next to it.
    fams = {}
    for a, st in per:
        if st["flops_per_launch"] <= 0:
            continue
        fam = "forward contractions (etd_contract)" if "_fwd" in st["name"] else "backward contractions (etd_back6)"
        f = fams.setdefault(fam, {"ms": 0.0, "flops": 0.0, "dense": 0.0, "launches": 0, "names": []})
        f["ms"] += a
        f["flops"] += st["flops_per_launch"]
        f["dense"] += st.get("dense_flops_per_launch", st["flops_per_launch"])
        f["launches"] += 1
        f["names"].append(st["name"])
    dom_fam, domf = max(fams.items(), key=lambda kv: kv[1]["ms"])
    dom_ms = domf["ms"] / domf["launches"]
    achieved = domf["flops"] / (domf["ms"] * 1e-3) * 1e-12
    slow_ms, slow = max((x for x in per if x[1]["flops_per_launch"] > 0), key=lambda x: x[0])
    traffic, traffic_stage = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tr = json.load(open(tpath)).get(f"cfg{cfg.id}_n{n}", {})
            # per-launch DRAM bytes of one ncu-captured launch of the family
            for name in domf["names"] + [k for k in tr if ("_fwd" in k) == ("forward" in dom_fam)]:
                if name in tr:
                    traffic, traffic_stage = tr[name], name
                    break
        except (OSError, ValueError):
            traffic = None
    transform_ms = sum(a for a, st in per if st["flops_per_launch"] > 0)
    transform_flops = sum(st["flops_per_launch"] for _, st in per)
    comm_ms = ms - sum(a for a, _ in per)  # exchange + pack/unpack + commit (sharded), launch gaps

    dense_flops = sum(st.get("dense_flops_per_launch", st["flops_per_launch"]) for _, st in per)

    def stage_line(a, st):
        if st["flops_per_launch"] > 0:
            return {"name": st["name"], "ms": round(a, 3), "bound": "tensor",
                    "tflops": round(st["flops_per_launch"] / (a * 1e-3) * 1e-12, 2),
                    "frac": round(st["flops_per_launch"] / (a * 1e-3) * 1e-12 / FP64_PEAK_TFLOPS, 4),
                    "dense_equiv_tflops": round(st.get("dense_flops_per_launch", 0) / (a * 1e-3) * 1e-12, 2)}
        gbs = st["bytes_per_launch"] / (a * 1e-3) * 1e-9
        return {"name": st["name"], "ms": round(a, 3), "bound": "hbm", "gbs": round(gbs, 1),
                "frac": round(gbs / HBM_PEAK_GBS, 4)}

    dense_ach = domf["dense"] / (domf["ms"] * 1e-3) * 1e-12
    roofline = {"bound": "tensor", "achieved": round(achieved, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": round(achieved / FP64_PEAK_TFLOPS, 4), "traffic": traffic, "traffic_stage": traffic_stage,
                "kernel_share_of_step": round(domf["ms"] / ms, 4), "launches_per_step": domf["launches"],
                "avg_launch_ms": round(dom_ms, 3),
                "slowest_launch": {"name": slow["name"], "ms": round(slow_ms, 3),
                                   "tflops": round(slow["flops_per_launch"] / (slow_ms * 1e-3) * 1e-12, 3),
                                   "frac": round(slow["flops_per_launch"] / (slow_ms * 1e-3) * 1e-12
                                                 / FP64_PEAK_TFLOPS, 4)},
                "basis": "executed",
                "basis_note": ("achieved = the FLOPs the launch executes (the DST-I parity split runs a quarter of "
                               "the dense 2n per point per transform) / its event-timed duration; "
                               "dense_equiv_achieved = SURVEY 8(d)'s dense count over the same time (exceeds the "
                               "peak by construction); executed FLOP = 512 x DMMA.8x8x4 instructions "
                               "(sm__inst_executed_pipe_tensor_subpipe_dmma.sum, profiles/r02_ncu_full_cfg3_contract.md)"),
                "dense_equiv_achieved": round(dense_ach, 3),
                "kernel": dom_fam,
                "peak_source": FP64_PEAK_NOTE,
                "algorithmic_flops_per_launch": domf["flops"] / domf["launches"],
                "dense_flops_per_launch": domf["dense"] / domf["launches"],
                "all_transforms": {"tflops": round(transform_flops / (transform_ms * 1e-3) * 1e-12, 3),
                                   "frac": round(transform_flops / (transform_ms * 1e-3) * 1e-12 / FP64_PEAK_TFLOPS, 4),
                                   "ms_per_step": round(transform_ms, 3),
                                   "dense_equiv_tflops": round(dense_flops / (transform_ms * 1e-3) * 1e-12, 3)},
                "parity_split": parity,
                "fold_level": fold_level,
                "flops_note": ("achieved/frac count the FLOPs the transforms execute: on parity-split axes "
                               "(DST-I even/odd modes, DESIGN.md §4a) 2(2h)h/n per point and transform, h=(n+1)/2, "
                               "half of the dense 2n (SURVEY §8(d)); with the second-level split (fold_level 2, "
                               "DESIGN.md §4b) a forward transform runs two launches of 2(2H)H/n, H=h/2, a quarter "
                               "of the dense FLOPs; dense_equiv_tflops = 26 n N per species-step over the same time; "
                               "fold_* stages are the HBM-bound stack passes of the second-level split"),
                "stages": [stage_line(a, st) for a, st in per],
                "non_kernel_ms_per_step": round(comm_ms, 3),
                "hbm_peak_gbs": HBM_PEAK_GBS, "hbm_peak_source": HBM_PEAK_NOTE}

    # ---- e2e through the public API: pinned host in -> step -> pinned host out ----
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    hin = [torch.from_numpy(a).pin_memory() for a in ics]
    hout = [torch.empty_like(h).pin_memory() for h in hin]
    cnt = plan.local_count

    ptr = lambda lst, i: lst[i].data_ptr() if i < len(lst) else 0

    def e2e_step():
        # public API call: etd_advance(host in -> 1 step -> host out), copies
        # pipelined against the first/last kernels inside the library
        plan.advance_ptr(ptr(hin, 0), ptr(hin, 1), ptr(hout, 0), ptr(hout, 1), 0, 0.0, 1)

    e2e_step()  # warm
    barrier()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    f0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    f1.record(stream)
    barrier()
    e2e_wall = (time.perf_counter() - w0) / e2e_steps
    e2e_ms = max(f0.elapsed_time(f1) / e2e_steps, e2e_wall * 1e3)
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    bytes_io = cnt * 8 * cfg.nspecies * world
    e2e = {"value": total_pts / (e2e_ms * 1e-3), "unit": "grid-point updates/s", "h2d_bytes_per_step": bytes_io,
           "d2h_bytes_per_step": bytes_io, "ms_per_step": e2e_ms,
           "api": "etd_advance(pinned host U,V in -> 1 step -> pinned host U,V out)"}
    finite = bool(np.all(np.isfinite(hout[0].numpy())))
    del hin, hout

    # ---- e2e through the reference-shaped value API on plain (pageable) numpy
    # arrays: etd2rkds_step_system / advance allocate the output state per call,
    # as the reference's advance returns a new Field (stepper.hpp:85-86) ----
    e2e_pageable = None
    if world == 1 and args.e2e_pageable:
        from paper_2601_06849_b200 import etd as E
        src = cfg.source

        def pageable_step():
            if cfg.nspecies == 1:
                return E.advance(plan, E.StepperState(0, 0.0, ics[0]), src)
            return E.etd2rkds_step_system(plan, E.SystemState(0, 0.0, ics[0], ics[1]), src)

        r = pageable_step()  # warm: allocates the plan's pinned mirror once
        del r
        barrier()
        w0 = time.perf_counter()
        for _ in range(e2e_steps):
            r = pageable_step()
            del r
        barrier()
        pg_ms = (time.perf_counter() - w0) / e2e_steps * 1e3
        e2e_pageable = {"value": total_pts / (pg_ms * 1e-3), "unit": "grid-point updates/s", "ms_per_step": pg_ms,
                        "h2d_bytes_per_step": bytes_io, "d2h_bytes_per_step": bytes_io,
                        "api": ("etd2rkds_step_system(plan, SystemState(numpy U, V), f): pageable host arrays in, "
                                "new pageable arrays out, 1 step per call; staged through the plan's pinned "
                                "mirror by host copy threads (wall clock)")}

    line = {"metric": "grid-point updates/sec (FP64)", "value": value, "unit": "grid-point updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded counter-based RNG, DESIGN.md Inputs)",
            "config": dict(workload_config(cfg, n, world), comm_ranks=comm_ranks, device_bytes_per_rank=dev_bytes),
            "roofline": roofline, "e2e": e2e, "e2e_pageable": e2e_pageable,
            "gpu_launches": plan.launches_per_step * args.steps, "clocks": clk, "finite": finite,
            "ic_seconds": round(t_ic, 2)}

    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            rates, cores, sample = cpu_reference_sample(cfg, n, reps=2, warmup=1) if cfg.dim == 3 else (None, None, None)
            if cfg.dim == 2:
                from oracle import Ref
                cores = os.cpu_count() or 1
                Ref.set_threads(cores)
                _, _, _, sec = Ref.scalar_run(cfg.dim, n, cfg.tau, cfg.kappa[0], cfg.q, ics[0], 3, src_kind=1)
                rates = [n ** 2 * 3 / sec]
                sample = f"reference make_plan+advance, full {n}x{n} grid, 3 steps"
            line["cpu_baseline"] = {"value": statistics.median(rates), "unit": "grid-point updates/s",
                                    "cores": cores, "kind": "reference", "sample": sample}
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "unit": "grid-point updates/s", "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    plan.close()
    if world == 1 and not args.no_alt:
        line["alt_backends"] = {"dense_transforms": alt_plan(args, cfg, n, ics, local_rank, "dense"),
                                "thomas": alt_plan(args, cfg, n, ics, local_rank, "thomas")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def alt_plan(args, cfg, n, ics, local_rank, kind):
    """The same step on the same inputs with
      kind "dense":  the dense n x n eigenbasis contractions (ETD_DENSE=1, no parity
                     split) — the roofline of the plain DMMA contraction kernel;
      kind "thomas": BackendKind::Thomas (per-pole complex tridiagonal sweeps,
                     thomas.cpp).
    Device-resident, CUDA events on the plan's stream.  Reported next to the
    headline, which stays the eigenbasis-transform path the north star names."""
    import torch
    from paper_2601_06849_b200 import configs, etd
    try:
        if kind == "dense":
            os.environ["ETD_DENSE"] = "1"
            try:
                tp = configs.make_plan(cfg, n, device=local_rank)
            finally:
                os.environ.pop("ETD_DENSE", None)
        else:
            tp = configs.make_plan(cfg, n, device=local_rank, backend=etd.BackendKind.Thomas)
    except Exception as e:  # e.g. out of memory on a smaller device
        return {"value": None, "note": f"unavailable: {e}"}
    try:
        for s_, a in enumerate(ics):
            tp.upload(s_, a)
        tp.step(max(1, args.warmup))
        stream = torch.cuda.ExternalStream(tp.stream, device=torch.device("cuda", local_rank))
        tp.set_profiling(True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tp.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        stages = []
        tr_ms = tr_fl = 0.0
        for st in tp.stage_stats():
            a = st["ms_total"] / max(1, st["launches"])
            if kind == "dense" and st["flops_per_launch"] > 0:
                tf = st["flops_per_launch"] / (a * 1e-3) * 1e-12
                tr_ms, tr_fl = tr_ms + a, tr_fl + st["flops_per_launch"]
                stages.append({"name": st["name"], "ms": round(a, 3), "bound": "tensor", "tflops": round(tf, 2),
                               "frac": round(tf / FP64_PEAK_TFLOPS, 4)})
                continue
            gbs = st["bytes_per_launch"] / (a * 1e-3) * 1e-9
            stages.append({"name": st["name"], "ms": round(a, 3), "bound": "hbm", "gbs": round(gbs, 1),
                           "frac": round(gbs / HBM_PEAK_GBS, 4)})
        out = {"value": cfg.points(n) * cfg.nspecies / (ms * 1e-3), "unit": "grid-point updates/s",
               "ms_per_step": ms, "stages": stages}
        if kind == "dense":
            tf = tr_fl / (tr_ms * 1e-3) * 1e-12
            out["all_transforms"] = {"tflops": round(tf, 3), "frac": round(tf / FP64_PEAK_TFLOPS, 4),
                                     "ms_per_step": round(tr_ms, 3)}
            out["note"] = "dense n x n DMMA contractions (ETD_DENSE=1): 26 n N FLOPs per species-step"
        else:
            out["note"] = "BackendKind::Thomas on the device; algorithmic bytes = stage inputs + outputs"
        return out
    finally:
        tp.close()


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(n):
    """One process per GPU: re-run this script under torch.distributed.run with N
    ranks (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* set by the launcher).  Rank 0
    prints the JSON line; the launcher's exit code is returned."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    env = dict(os.environ, ETD_BENCH_LAUNCHED="1", OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def dry_run(args, cfg, n, rank, world):
    """Rendezvous + per-rank budget, no device work (CPU-testable N>1 path)."""
    import torch.distributed as dist
    from paper_2601_06849_b200 import etd as E
    launched = "WORLD_SIZE" in os.environ
    if launched:
        dist.init_process_group("gloo")
    grid = E.unit_box_grid(cfg.dim, n + 1)
    mine = E.plan_device_bytes(grid, cfg.nspecies, world, rank) if cfg.dim == 3 or world == 1 else None
    lo, hi = E.zslab_partition(n, world, rank) if cfg.dim == 3 else (0, 1)
    me = {"rank": rank, "world_size": dist.get_world_size() if launched else 1, "slab": [lo, hi],
          "device_bytes": mine}
    got = [None] * world
    if launched:
        dist.all_gather_object(got, me)
    else:
        got = [me]
    if rank == 0:
        line = {"metric": "grid-point updates/sec (FP64)", "value": None, "unit": "grid-point updates/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "dry_run": True,
                "ranks_seen": len(got), "world_sizes_seen": sorted({g["world_size"] for g in got}),
                "slabs": [g["slab"] for g in got],
                "per_rank_device_bytes": [g["device_bytes"] for g in got],
                "config": workload_config(cfg, n, world)}
        print(json.dumps(line), flush=True)
    if launched:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int, default=None, help="override the grid size (testing only)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e-pageable", dest="e2e_pageable", action="store_false",
                    help="skip the pageable-numpy e2e line")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the Thomas-backend line")
    ap.add_argument("--dry-run", action="store_true", help="rendezvous and budget check only (no device work)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus is not None and args.gpus > 1:
        return launch_ranks(args.gpus)
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.gpus is not None and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    from paper_2601_06849_b200 import configs
    cfg = configs.CONFIGS[args.config]
    n = args.n or cfg.n
    if args.dry_run:
        return dry_run(args, cfg, n, rank, world)
    if args.impl == "reference":
        return reference_arm(args, cfg, n, rank, world)
    return b200_arm(args, cfg, n, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
