#!/usr/bin/env python
"""Benchmark of the hot path: pods placed/s and servers ranked/s (BASELINE.json metric).

One step = one pass of the whole hot path (snapshot, request
decode, flows, filter, statistics, scoring, argmax, commit, top-up) over one batch:
nacs_schedule_batch on config C4 — fat-tree k=32 (8192 servers), 100k requests per GPU
(weak scaling: every rank schedules its own 100k-request shard), TOPSIS with the Flat
schema.  A second line of numbers ("ahp") runs AHP Flat on C3 (k=16, 10k requests), the
largest config whose O(n_f^2) AHP pass fits a bench step.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU: launched by torchrun; one process per GPU, no data-path collective (requests
are independent, R21); the timed region is bracketed by barriers and the max over ranks
is taken.  --impl reference times the CPU oracle (the deliberately slow double-precision
program written from the paper) on a bounded sample of the same workload.
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

import numpy as np  # noqa: E402

from inputs import gen  # noqa: E402

# Algorithmic operation counts.
TOPSIS_OPS_ALL = 3       # per server ranked: the CPU/RAM/access-bandwidth compares of the filter
TOPSIS_OPS_FEAS = 45     # per feasible server: stats (14) + closeness (30) + argmax (1)
# kernels launched per nacs_schedule_batch call: TOPSIS = k_pod_max + k_layout_order (the chunk
# layout and the largest-first order, one CTA each) + k_batch_warp + k_batch (deferred requests;
# exits at once when none); AHP = k_batch
LAUNCHES = {"topsis": 4, "ahp": 1}
# DRAM bytes per launch of k_batch_warp from the committed `ncu --set full` capture
TRAFFIC = os.path.join(ROOT, "profiles", "ncu_traffic.json")
AHP_RCP_PER_PAIR = 1     # per unordered pair per non-constant criterion per pass: one reciprocal


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-ahp", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-once", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-paths", action="store_true")
    ap.add_argument("--sim", action="store_true", help="also run the E2 simulator campaign (context only)")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-matrix", action="store_true")
    ap.add_argument("--no-cold", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region through NVML (the
    library behind nvidia-smi), in-process every 20 ms: spawning nvidia-smi inside the
    timed region takes the driver lock and stalls the launch queue.  Falls back to
    nvidia-smi when NVML is unavailable."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._first = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(device))
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        return [str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits]

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    self.samples.append(self._sample_nvml())
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._first.set()
            self._stop.wait(0.02 if self._nvml is not None else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        # let the first query finish before the timed region
        self._first.wait(timeout=10)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


CFG_K = {"C2": 8, "C3": 16, "C4": 32}


def workload(rank: int, cfg: str, n_req: int | None = None):
    """Snapshot and this rank's request shard of a batch config (weak scaling: the config's
    request count per rank, or its first n_req requests)."""
    k = CFG_K[cfg]
    snap = gen.snapshot(k, gen.CONFIG_SEEDS[cfg])
    R = gen.CONFIG_REQUESTS[cfg] if n_req is None else n_req
    reqs = gen.requests(R, gen.CONFIG_SEEDS[cfg] + 1000 + 7919 * rank)
    name = f"{cfg}: fat-tree k={k} ({k ** 3 // 4} servers), {R} requests/GPU of 4-20 containers, batch"
    return snap, reqs, name


def quality(reqs: dict, out: dict) -> dict:
    """SURVEY 8(d) reporting: acceptance rate, accepted pods, mean U(i) (Eq. 1) over the
    accepted containers and mean U(ij) (Eq. 2, R23: bw^a / bw^max) over their vlinks."""
    o = {k: (v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v)) for k, v in out.items()}
    R = int(reqs["n_requests"])
    co, vo = reqs["container_off"].astype(np.int64), reqs["vlink_off"].astype(np.int64)
    st = o["status"][:R]
    acc_r = st == 1
    req_of_c = np.repeat(np.arange(R), np.diff(co))
    req_of_v = np.repeat(np.arange(R), np.diff(vo))
    acc_c = acc_r[req_of_c]
    acc_v = acc_r[req_of_v]
    Cn, Vn = int(co[-1]), int(vo[-1])
    ui = 0.5 * (o["cpu_alloc"][:Cn][acc_c] / reqs["cpu_max"][acc_c] + o["ram_alloc"][:Cn][acc_c] / reqs["ram_max"][acc_c])
    uij = o["bw_alloc"][:Vn][acc_v] / reqs["bw_max"][acc_v]
    pods = np.zeros(R, np.int64)
    np.maximum.at(pods, req_of_c, reqs["pod_of"].astype(np.int64) + 1)
    return {"acceptance": float(acc_r.mean()) if R else None, "accepted_pods": int(pods[acc_r].sum()),
            "U_i": float(ui.mean()) if ui.size else None, "U_ij": float(uij.mean()) if uij.size else None}


def alu_peak_tops(mhz: float) -> float:
    """FP32/INT issue roof: 148 SMs x 4 schedulers x 32 lanes per clock (T thread-instr/s)."""
    return 148 * 128 * mhz * 1e6 / 1e12


# ncu issue-slot utilisation of the TOPSIS batch kernel in the bench launch configuration
# (profiles/r01_summary.md: k_batch_warp, C4, 100k requests)
TOPSIS_NCU_ISSUE = 0.411


def topsis_roofline(st: dict, kernel_ms: float, mhz: float, pk_kind: str) -> dict:
    """Method-equivalent ALU throughput of the TOPSIS batch kernels: SURVEY 8(d)'s algorithmic op
    count (3 per server ranked + 45 per feasible server) per second against the issue roof.  The
    kernel reads only `slots_read_frac` of the slots a two-pass scan reads (whole-tile statistics,
    pruned scoring), so this is a method-equivalent rate; `ncu_issue_slots` is how busy the
    SMs actually were (ncu, profiles/r01_summary.md)."""
    ops = TOPSIS_OPS_ALL * st["servers_ranked"] + TOPSIS_OPS_FEAS * st["feasible"]
    achieved = ops / (kernel_ms / 1e3) / 1e12
    peak = alu_peak_tops(mhz)
    traffic = None
    if os.path.exists(TRAFFIC):
        traffic = json.load(open(TRAFFIC)).get("k_batch_warp", {}).get("dram_bytes_per_launch")
    read_frac = (st["scanned_a"] + st["scanned_b"]) / max(1, 2 * st["servers_ranked"])
    return {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Top/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": "k_batch_warp<TOPSIS> (whole call)",
            "ops": "method-algorithmic: 3 per server ranked + 45 per feasible server (SURVEY 8(d))",
            "slots_read_frac": read_frac, "ncu_issue_slots": TOPSIS_NCU_ISSUE,
            "peak_source": f"148 SMs x 128 lanes x {mhz:.0f} MHz (sm_max_mhz, {pk_kind})"}


# Thread-instructions per EXECUTED AHP term: the sorted-level passes evaluate each unordered pair
# of distinct levels once per pass, 4 terms sharing one MUFU.RCP in ~15 instructions
AHP_INSTR_PER_TERM = 15 / 4


def ahp_roofline(st: dict, kernel_ms: float, mhz: float) -> dict:
    """AHP against the issue-slot bound of what the kernel executes: 2 passes x the unordered
    pairs of distinct levels per non-constant criterion (nacs_stats.ahp_pairs) x ~15/4
    instructions per term, over the 148 x 128 lane-issue roof."""
    terms = 2 * st["ahp_pairs"]
    achieved = terms * AHP_INSTR_PER_TERM / (kernel_ms / 1e3) / 1e12
    peak = alu_peak_tops(mhz)
    return {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "T instr/s", "frac": achieved / peak,
            "terms_per_step": terms, "kernel": "k_batch<AHP> (sorted-level passes)",
            "ops": "2 passes x level pairs x 15/4 instructions per term (4-term groups, one MUFU.RCP each)",
            "peak_source": f"148 SMs x 128 lanes x {mhz:.0f} MHz"}


def run_ours(args, rank, world, local):
    import torch
    from paper_1909_07673_b200 import nacs

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(dev)  # a dedicated stream: events and kernels on the same handle
    torch.cuda.set_stream(stream)
    ctx = nacs.Context(local, stream)
    pk, pk_kind = peaks()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def measure(method, schema="flat", cfg="C4", n_req=None, **kw):
        snap, reqs, name = workload(rank, cfg, n_req)
        name = name.replace("batch", f"{method.upper()} {schema.capitalize()}, batch")
        ctx.load_topology(snap)
        d = {k: (torch.from_numpy(v).to(dev) if isinstance(v, np.ndarray) else v) for k, v in reqs.items()}
        out = ctx._alloc_out(reqs, True)[0]
        for _ in range(args.warmup):  # warm-up includes the flush (its first launch loads torch's module)
            flush.zero_()
            ctx.schedule_batch(d, method, schema, out=out, flags=nacs.NACS_ASYNC, **kw)
        torch.cuda.synchronize(dev)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        sampler = ClockSampler(local)
        barrier()
        with sampler:
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            for i in range(args.steps):
                flush.zero_()
                ev[i][0].record(stream)
                ctx.schedule_batch(d, method, schema, out=out, flags=nacs.NACS_ASYNC, **kw)
                ev[i][1].record(stream)
            t1.record(stream)
            torch.cuda.synchronize(dev)
        barrier()
        total_ms = max_over_ranks(t0.elapsed_time(t1))
        kern_ms = [a.elapsed_time(b) for a, b in ev]
        kern_avg = max_over_ranks(sum(kern_ms) / len(kern_ms))
        st = ctx.last_stats()  # stats of the last step (deterministic: identical every step)
        pod_steps = sum_over_ranks(st["pod_steps"])
        value = pod_steps * args.steps / (total_ms / 1e3)
        n = snap["k"] ** 3 // 4
        q = quality(reqs, out)
        q["accepted_pods_per_s"] = sum_over_ranks(q["accepted_pods"]) * args.steps / (total_ms / 1e3)
        res = dict(name=name, value=value, ms_per_step=total_ms / args.steps, kernel_ms=kern_avg, quality=q,
                   pod_steps_per_step=pod_steps, servers_ranked_per_s=value * n, n=n, stats=st,
                   clocks=sampler.summary(), snap=snap, reqs=reqs, out=out, d=d)
        return res

    topsis = measure("topsis", "flat", "C4")
    ahp = None if args.no_ahp else measure("ahp", "flat", "C3")
    # AHP and TOPSIS x {Flat, Clustering, Network} (T4 P:315-331) at C3 and C4
    matrix = None if args.no_matrix else measure_matrix(args, measure, topsis, ahp, pk)
    # rank once per request, pods walk the first pod step's order
    once = None if args.no_once else measure("topsis", rank_once=True)
    # the paper-literal variant flags as benchmarked modes
    variants = None
    if not args.no_variants:
        variants = {}
        for name, meth, kw in (("topsis_path_filter_0 (select then route, R6 flag)", "topsis", {"path_filter": 0}),
                               ("ahp_shifted_rule (R8 flag)", "ahp", {"ahp_rule": 1}),
                               ("ahp_l1_weights (R10 flag)", "ahp", {"l1_mode": 1})):
            if meth == "ahp" and args.no_ahp:
                continue
            v = measure(meth, "flat", "C4" if meth == "topsis" else "C3", **kw)
            variants[name] = {"workload": v["name"], "value": v["value"], "unit": "pods/s",
                              "ms_per_step": v["ms_per_step"]}
        # R2's alternative (bw_criterion = logical): one pod step through nacs_rank_topsis on the
        # C4 snapshot; the table of 8192 logical-bandwidth sums is rebuilt inside every call
        snap_c4 = gen.snapshot(32, gen.CONFIG_SEEDS["C4"])
        ctx.load_topology(snap_c4)
        for name, bwc in (("topsis_rank_access_bw (R2 default, one pod step per call)", 0),
                          ("topsis_rank_logical_bw (R2 flag, one pod step per call)", 1)):
            for _ in range(args.warmup):
                ctx.rank("topsis", "flat", 1500, 3000, bw_criterion=bwc)
            barrier()
            t = time.perf_counter()
            for _ in range(args.steps):
                ctx.rank("topsis", "flat", 1500, 3000, bw_criterion=bwc)
            el = max_over_ranks((time.perf_counter() - t) / args.steps)
            variants[name] = {"workload": "C4 snapshot (k=32, 8192 servers), host-pointer nacs_rank_topsis call",
                              "value": 8192 / el, "unit": "servers ranked/s (per GPU)", "ms_per_call": el * 1e3}

    # general-topology widest-shortest paths (modified Dijkstra)
    paths = None if args.no_paths else measure_paths(args, ctx, dev, stream, flush, barrier, max_over_ranks,
                                                     sum_over_ranks, rank, local)

    # C5 (BASELINE configs[4]): k=64, sequential scheduling with the servers sharded over the ranks
    c5 = None if args.no_c5 else measure_c5(args, rank, world, local, stream, max_over_ranks)

    # C2 sequential (live state, commits) for both methods
    c2 = None if args.no_matrix else measure_c2(args, ctx, stream, max_over_ranks)
    # standalone nacs_rank_topsis on cold snapshots against HBM
    cold = None if args.no_cold else measure_cold(args, ctx, dev, stream, flush, barrier, max_over_ranks,
                                                  sum_over_ranks, pk, pk_kind)
    # the E2 campaign through the discrete-event simulator (T5-shaped rows):
    # context only (the paper's T5 numbers are not a target), so only with --sim
    sim = measure_sim(ctx) if (args.sim and rank == 0) else None

    # roofline of the dominant kernel (k_batch_warp<TOPSIS>): issue-bound ALU
    clocks = topsis["clocks"]
    mhz = float(pk.get("sm_max_mhz", 1965.0))
    roofline = topsis_roofline(topsis["stats"], topsis["kernel_ms"], mhz, pk_kind)

    ahp_obj = None
    if ahp is not None:
        sa = ahp["stats"]
        ahp_obj = {"workload": ahp["name"], "value": ahp["value"], "unit": "pods/s",
                   "servers_ranked_per_s": ahp["servers_ranked_per_s"], "ms_per_step": ahp["ms_per_step"],
                   "pod_steps_per_step": ahp["pod_steps_per_step"], "fp64_decisions": sa["fp64_decisions"],
                   "quality": ahp["quality"], "roofline": ahp_roofline(sa, ahp["kernel_ms"], mhz)}

    # e2e: the public API with host buffers (staging copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        snap, reqs = topsis["snap"], topsis["reqs"]
        ctx.load_topology(snap)
        hout = ctx._alloc_out(reqs, False)[0]  # caller-allocated host outputs, reused per step
        ctx.schedule_batch(reqs, "topsis", "flat", out=hout)
        barrier()
        t = time.perf_counter()
        for _ in range(args.steps):
            ctx.schedule_batch(reqs, "topsis", "flat", out=hout)
        torch.cuda.synchronize(dev)
        el = max_over_ranks(time.perf_counter() - t)
        R = reqs["n_requests"]
        Cn, Vn = int(reqs["container_off"][-1]), int(reqs["vlink_off"][-1])
        e2e = {"value": topsis["pod_steps_per_step"] * args.steps / el, "unit": "pods/s",
               "h2d_bytes_per_step": 4 * (2 * (R + 1) + 5 * Cn + 4 * Vn),
               "d2h_bytes_per_step": 4 * (R + 3 * Cn + 2 * Vn)}

    cpu = None
    if paths is not None and rank == 0 and world == 1 and not args.no_cpu:
        paths["cpu_baseline"] = cpu_baseline_paths()
    if sim is not None and world == 1 and not args.no_cpu:
        sim["cpu_baseline"] = cpu_baseline_sim()
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(topsis["snap"], topsis["reqs"], budget_s=15.0)

    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        line = {"metric": "pods placed/sec (and servers ranked/sec)", "value": topsis["value"], "unit": "pods/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": topsis["ms_per_step"], "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": topsis["name"], "k": 32, "servers": topsis["n"],
                           "requests_per_gpu": gen.CONFIG_REQUESTS["C4"], "method": "topsis", "schema": "flat",
                           "parallelism": f"dp{world}: each rank schedules its own seeded 100k-request shard "
                                          "(requests independent, R21; no data-path collective)",
                           "l2": "flushed between steps (256 MB write)"},
                "servers_ranked_per_s": topsis["servers_ranked_per_s"],
                "pod_steps_per_step": topsis["pod_steps_per_step"],
                "kernel_ms": topsis["kernel_ms"], "fp64_decisions": topsis["stats"]["fp64_decisions"],
                "retries": topsis["stats"]["retries"], "quality": topsis["quality"],
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": args.steps * LAUNCHES["topsis"],
                "clocks": clocks, "ahp": ahp_obj, "matrix": matrix, "c2_sequential": c2, "rank_cold": cold,
                "variants": variants, "paths": paths, "simulator": sim, "c5": c5,
                "rank_once": None if once is None else {
                    "workload": once["name"].replace("batch", "batch, rank once per request (R25)"),
                    "value": once["value"], "unit": "pods/s", "ms_per_step": once["ms_per_step"],
                    "kernel_ms": once["kernel_ms"], "pod_steps_per_step": once["pod_steps_per_step"],
                    "quality": once["quality"],
                    "slots_read_frac": (once["stats"]["scanned_a"] + once["stats"]["scanned_b"])
                    / max(1, 2 * once["stats"]["servers_ranked"])},
                "paper_context": "T5 (P:416-426): TOPSIS 3.48-3.84 s, AHP 6.90-9.45 s per 6000-request k=20 campaign "
                                 "on an unnamed CUDA 10.1 GPU (~10-14 M / 4-7 M servers ranked/s derived)"}
        print(json.dumps(line))


AHP_C4_REQUESTS = 1000   # C4 AHP cell: the first 1000 requests per GPU (O(K^2) levels per pod step)


def measure_matrix(args, measure, topsis, ahp, pk):
    """AHP and TOPSIS x the three schemas of T4 at C3 and C4, batch mode,
    each cell device-timed like the headline (L2 flushed between steps)."""
    from paper_1909_07673_b200 import nacs
    mhz = float(pk.get("sm_max_mhz", 1965.0))
    cells = {}
    for cfg in ("C3", "C4"):
        for method in ("topsis", "ahp"):
            for schema in ("flat", "clustering", "network"):
                key = f"{cfg} {method} {schema}"
                if (cfg, method, schema) == ("C4", "topsis", "flat"):
                    r = topsis
                elif (cfg, method, schema) == ("C3", "ahp", "flat") and ahp is not None:
                    r = ahp
                else:
                    try:
                        r = measure(method, schema, cfg, AHP_C4_REQUESTS if (cfg, method) == ("C4", "ahp") else None)
                    except nacs.NacsError as e:
                        cells[key] = {"unavailable": str(e)}
                        continue
                st = r["stats"]
                rl = topsis_roofline(st, r["kernel_ms"], mhz, "") if method == "topsis" else \
                    ahp_roofline(st, r["kernel_ms"], mhz)
                cells[key] = {"workload": r["name"], "value": r["value"], "unit": "pods/s",
                              "servers_ranked_per_s": r["servers_ranked_per_s"], "ms_per_step": r["ms_per_step"],
                              "pod_steps_per_step": r["pod_steps_per_step"], "fp64_decisions": st["fp64_decisions"],
                              "quality": r["quality"],
                              "roofline": {k: rl[k] for k in ("bound", "achieved", "peak", "unit", "frac")}}
    return cells


def measure_c2(args, ctx, stream, max_over_ranks):
    """fat-tree k=8, 100 requests scheduled sequentially on the live state
    (commits), TOPSIS and AHP Flat; device arrays, the state reloaded before each rep."""
    import torch
    from paper_1909_07673_b200 import nacs
    snap, reqs = gen.config("C2")
    dev = torch.device("cuda", ctx.device)
    d = {k: (torch.from_numpy(v).to(dev) if isinstance(v, np.ndarray) else v) for k, v in reqs.items()}
    res = {}
    for method in ("topsis", "ahp"):
        out = ctx._alloc_out(reqs, True)[0]
        times = []
        for rep in range(args.warmup + args.steps):
            ctx.load_topology(snap)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.schedule_request(d, method, "flat", out=out, flags=nacs.NACS_ASYNC)
            e1.record(stream)
            torch.cuda.synchronize()
            if rep >= args.warmup:
                times.append(e0.elapsed_time(e1))
        ms = max_over_ranks(statistics.median(times))
        st = ctx.last_stats()
        res[method] = {"value": st["pod_steps"] / (ms / 1e3), "unit": "pods/s", "ms_per_step": ms,
                       "pod_steps_per_step": st["pod_steps"], "servers_ranked_per_s": st["servers_ranked"] / (ms / 1e3),
                       "quality": quality(reqs, out)}
    return {"workload": "C2: fat-tree k=8 (128 servers), 100 requests, sequential Flat scheduling (live state)",
            "modes": res}


def cold_states(snap: dict, B: int, seed: int = 1):
    """B distinct DC states (device-generated, seeded): the snapshot's links, residual CPU / RAM /
    access link and f_u drawn uniformly over their ranges (inputs/gen.py's magnitudes)."""
    import torch
    k = snap["k"]
    n = k ** 3 // 4
    row = np.concatenate([snap["cpu_res"], snap["ram_res"], snap["active"].astype(np.int32), snap["link_res"]])
    st = torch.from_numpy(np.tile(row.astype(np.int32), (B, 1))).cuda()
    g = torch.Generator(device="cuda").manual_seed(seed)
    st[:, :n] = torch.randint(0, snap["cpu_cap"] + 1, (B, n), device="cuda", generator=g, dtype=torch.int32)
    st[:, n:2 * n] = torch.randint(0, snap["ram_cap"] + 1, (B, n), device="cuda", generator=g, dtype=torch.int32)
    st[:, 2 * n:3 * n] = torch.randint(0, 2, (B, n), device="cuda", generator=g, dtype=torch.int32)
    st[:, 3 * n:4 * n] = torch.randint(50, snap["link_cap"] + 1, (B, n), device="cuda", generator=g, dtype=torch.int32)
    return st


COLD = (("C4 geometry", 32, 4096), ("C5 geometry", 64, 512))


def cold_traffic(k: int, B: int):
    """DRAM bytes per launch of k_rank_occ from the committed ncu capture (k = 32, B = 4096)."""
    if (k, B) != (32, 4096) or not os.path.exists(TRAFFIC):
        return None
    return json.load(open(TRAFFIC)).get("k_rank_occ", {}).get("dram_bytes_per_launch")


def measure_cold(args, ctx, dev, stream, flush, barrier, max_over_ranks, sum_over_ranks, pk, pk_kind):
    """standalone TOPSIS ranking on COLD snapshots against HBM: one
    nacs_rank_topsis_many call ranks one pod step (the request's first: demand, no flows) on each
    of B distinct device-resident DC states (B x 16 n bytes >> the 126 MB L2, so every step
    streams from HBM; no flush needed).  Algorithmic bytes per server: 16 read (cpu, ram, f_u,
    access link) + 4 written (the FP32 score)."""
    import torch
    from paper_1909_07673_b200 import nacs
    res = {}
    for name, k, B in COLD:
        snap = gen.snapshot(k, gen.CONFIG_SEEDS["C4" if k == 32 else "C5"])
        ctx.load_topology(snap)
        n = k ** 3 // 4
        st = cold_states(snap, B, seed=11 + ctx.device)
        out = dict(mask=None, scores=torch.empty((B, n), dtype=torch.float32, device=dev),
                   best=torch.empty(B, dtype=torch.int32, device=dev))
        for _ in range(args.warmup):
            ctx.rank_many(st, 1500, 3000, out=out, mask=False, flags=nacs.NACS_ASYNC)
        torch.cuda.synchronize(dev)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        for i in range(args.steps):
            ev[i][0].record(stream)
            ctx.rank_many(st, 1500, 3000, out=out, mask=False, flags=nacs.NACS_ASYNC)
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev) / args.steps)
        stats = ctx.last_stats()
        byts = B * n * (16 + 4)
        ach = byts / (ms / 1e3) / 1e9
        peak = float(pk.get("hbm_gbs", 6650.0))
        res[name] = {"workload": f"fat-tree k={k} ({n} servers): {B} distinct states per GPU, one pod step each "
                                 f"(demand 1500 mc / 3000 MiB, no flows), TOPSIS Flat",
                     "value": sum_over_ranks(B * n) / (ms / 1e3), "unit": "servers ranked/s",
                     "states_per_s": sum_over_ranks(B) / (ms / 1e3), "ms_per_step": ms,
                     "fp64_decisions": stats["fp64_decisions"], "gpu_launches": 1,
                     "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                                  "traffic": cold_traffic(k, B), "kernel": "k_rank_occ (nacs_rank.cu)",
                                  "bytes": "16 B read + 4 B score written per server",
                                  "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_kind})"}}
    return res


C5_REQUESTS = {"topsis": 40, "ahp": 12}


def measure_c5(args, rank, world, local, stream, max_over_ranks):
    """C5: fat-tree k=64 (65536 servers), sequential scheduling (live state) of the same requests
    on every rank, the servers sharded over the `world` ranks (nacs_create_sharded: replicated
    filter and commit, each rank scores its block, ncclAllGather of (score, index) keys per pod
    step; AHP sum-allreduces per-level weights and L2).  Strong scaling: the work is fixed, the
    ranks split it.  At N=1: the unsharded context, plus 8 loopback shards on the one GPU that
    must give identical placements.  Timed on the device (CUDA events), max over ranks."""
    import hashlib
    import torch
    from paper_1909_07673_b200 import nacs
    snap = gen.snapshot(64, gen.CONFIG_SEEDS["C5"])
    res = {}
    if world > 1:
        import torch.distributed as dist
        obj = [nacs.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        # the unsharded run on every rank is the reference the NCCL shards must reproduce
        modes = [("unsharded", None), (f"nccl_x{world}", (rank, world, obj[0]))]
    else:
        modes = [("unsharded", None), ("loopback_x8", (0, 8, None))]
    for method, nreq in C5_REQUESTS.items():
        reqs = gen.requests(nreq, gen.CONFIG_SEEDS["C5"] + 1000)
        warm = gen.subset(reqs, np.arange(2))
        for name, shard in modes:
            ctx = nacs.Context(local, stream, shard=shard)
            ctx.load_topology(snap)
            ctx.schedule_request(warm, method, "flat")
            ctx.load_topology(snap)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out = ctx.schedule_request(reqs, method, "flat")
            e1.record(stream)
            torch.cuda.synchronize()
            ms = max_over_ranks(e0.elapsed_time(e1))
            st = ctx.last_stats()
            h = hashlib.sha256(b"".join(np.ascontiguousarray(out[k]).tobytes() for k in sorted(out))).hexdigest()
            mhz = float(peaks()[0].get("sm_max_mhz", 1965.0))
            rl = topsis_roofline(st, ms, mhz, "") if method == "topsis" else ahp_roofline(st, ms, mhz)
            res[f"{method} {name}"] = {"pods_per_s": st["pod_steps"] / (ms / 1e3), "ms": ms,
                                       "us_per_pod_step": ms * 1e3 / max(1, st["pod_steps"]),
                                       "pod_steps": st["pod_steps"], "placements_sha256": h[:16],
                                       "roofline": {k: rl[k] for k in ("bound", "achieved", "peak", "unit", "frac")}}
            ctx.close()
    same = {m: len({v["placements_sha256"] for k, v in res.items() if k.startswith(m)}) == 1 for m in C5_REQUESTS}
    if world > 1:  # every rank holds the same placements (replicated commit), equal to unsharded
        import torch.distributed as dist
        mine = {k: v["placements_sha256"] for k, v in res.items()}
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        same = {m: same[m] and all(a == allh[0] for a in allh) for m in C5_REQUESTS}
    return {"workload": "C5: fat-tree k=64 (65536 servers), sequential Flat scheduling of "
                        f"{C5_REQUESTS['topsis']} (TOPSIS) / {C5_REQUESTS['ahp']} (AHP) requests, servers sharded "
                        f"over {world} rank(s)", "scaling": "strong", "modes": res,
            "identical_placements_across_modes": same}


PATH_QUERIES = 1 << 20   # queries per GPU per step (weak scaling)


def path_workload(rank: int):
    """The paper's DC (fat-tree k=20, 2000 servers) as an explicit graph with warm link
    residuals, and 2^20 random server pairs per GPU with demand ~U{1..50} Mbps."""
    g = gen.fat_tree_graph(gen.snapshot(20, 20))
    q = gen.path_queries(g, PATH_QUERIES, 7000 + rank)
    return g, q


def measure_paths(args, ctx, dev, stream, flush, barrier, max_over_ranks, sum_over_ranks, rank, local):
    import torch
    from paper_1909_07673_b200 import nacs
    g, q = path_workload(rank)
    ctx.load_graph(g)
    d = {k: torch.from_numpy(v).to(dev) for k, v in q.items()}
    nq = q["src"].size
    mh = 8
    out = (torch.empty(nq, dtype=torch.int32, device=dev), torch.empty(nq, dtype=torch.int32, device=dev),
           torch.empty((nq, mh + 1), dtype=torch.int32, device=dev))
    lb = torch.empty(g["n_servers"], dtype=torch.int64, device=dev)

    def timed(fn):
        for _ in range(args.warmup):
            flush.zero_()
            fn()
        torch.cuda.synchronize(dev)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            fn()
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        return max_over_ranks(sum(a.elapsed_time(b) for a, b in ev) / args.steps)

    ms = timed(lambda: ctx.widest_paths(d["src"], d["dst"], d["demand"], max_hops=mh, out=out, flags=nacs.NACS_ASYNC))
    edges = ctx.last_stats()["edges_scanned"]
    ms_lb = timed(lambda: ctx.logical_bandwidth(out=lb, flags=nacs.NACS_ASYNC))
    edges_lb = ctx.last_stats()["edges_scanned"]
    # e2e: host arrays through the public API (staging copies inside the timed region)
    hout = (np.zeros(nq, np.int32), np.zeros(nq, np.int32), np.zeros((nq, mh + 1), np.int32))
    ctx.widest_paths(q["src"], q["dst"], q["demand"], max_hops=mh, out=hout)
    barrier()
    t = time.perf_counter()
    for _ in range(args.steps):
        ctx.widest_paths(q["src"], q["dst"], q["demand"], max_hops=mh, out=hout)
    el = max_over_ranks(time.perf_counter() - t)
    total = sum_over_ranks(nq)
    ns = g["n_servers"]
    return {"workload": "fat-tree k=20 (2000 servers, 2500 vertices, P:396) as a general graph, warm links; "
                        f"{nq} random server pairs/GPU, demand U{{1..50}} Mbps (P:398)",
            "value": total / (ms / 1e3), "unit": "paths/s", "ms_per_step": ms,
            "edges_scanned_per_query": edges / nq,
            "e2e": {"value": total * args.steps / el, "unit": "paths/s", "h2d_bytes_per_step": 12 * nq,
                    "d2h_bytes_per_step": 4 * nq * (mh + 3)},
            "logical_bandwidth": {"value": sum_over_ranks(ns * (ns - 1)) / (ms_lb / 1e3), "unit": "server pairs/s",
                                  "ms_per_step": ms_lb, "edges_scanned_per_source": edges_lb / ns},
            "kernel": "k_paths_grouped_cta (a CTA per destination group: one BFS, smem atomicMin labels; walks per thread)"}


# T5: events, average runtime (s), U(ij), U(i) per algorithm on the paper's GPU
T5 = {"bf": (2462, 79.38, 1.0, 0.9689), "wf": (1007, 47.80, 1.0, 0.9941),
      "ahp flat": (949, 9.45, 1.0, 0.9822), "ahp clustering": (936, 7.51, 1.0, 0.9910),
      "ahp network": (928, 6.90, 1.0, 0.9841), "topsis flat": (894, 3.67, 1.0, 0.9885),
      "topsis clustering": (916, 3.84, 1.0, 0.9901), "topsis network": (892, 3.48, 1.0, 0.9894)}


def measure_sim(ctx):
    """The E2 campaign: fresh k=20 fat-tree, 6000 requests of 4 containers arriving
    over 500 ticks, durations up to 250 ticks, through nacs_simulate for the 8 rows of T5.
    Runtime = wall time inside the scheduling attempts (T5 "Average Runtime"), U(i) = mean over
    accepted containers of Eq. 1, U(ij) = mean over accepted inter-container vlinks of Eq. 2."""
    snap = gen.snapshot(20, warm=False)
    reqs, arrival, duration = gen.sim_workload()
    rows = {}
    for name in ("bf", "wf", "ahp flat", "ahp clustering", "ahp network", "topsis flat", "topsis clustering",
                 "topsis network"):
        method, schema = (name.split() + ["flat"])[:2]
        ctx.load_topology(snap)
        r = ctx.simulate(reqs, arrival, duration, method, schema, max_ticks=5000)
        pl = r["placements"]
        acc_c = pl["server_of_container"] >= 0
        ui = 0.5 * (pl["cpu_alloc"][acc_c] / reqs["cpu_max"][acc_c] + pl["ram_alloc"][acc_c] / reqs["ram_max"][acc_c])
        vsrv = pl["server_of_container"][reqs["container_off"][:-1].repeat(np.diff(reqs["vlink_off"]))
                                         + reqs["vl_src"]]
        acc_v = vsrv >= 0
        uij = pl["bw_alloc"][acc_v] / reqs["bw_max"][acc_v]
        st = r["start"]
        ok = st >= 0
        t5 = T5[name]
        rows[name] = {"events": r["totals"]["events"], "attempts": r["totals"]["attempts"],
                      "accepted": r["totals"]["accepted"], "runtime_s": r["sched_seconds"],
                      "wall_s": r["wall_seconds"], "U_ij": float(uij.mean()) if uij.size else None,
                      "U_i": float(ui.mean()) if ui.size else None,
                      "mean_delay": float((st[ok] - arrival[ok]).mean()) if ok.any() else None,
                      "max_F_servers": float(r["tick_servers"].max() / 2000),
                      "max_F_links": float(r["tick_links"].max() / 6000),
                      "pod_steps": ctx.last_stats()["pod_steps"], "retries": ctx.last_stats()["retries"],
                      "paper_T5": {"events": t5[0], "runtime_s": t5[1], "U_ij": t5[2], "U_i": t5[3]}}
    return {"workload": "E2 (P:396-398): fresh fat-tree k=20 (2000 servers), 6000 requests x 4 containers, "
                        "arrivals U{0..499}, durations U{1..250} ticks, pairs <= 50 Mbps; nacs_simulate, "
                        "FIFO with head-of-line blocking (R28)",
            "rows": rows,
            "note": "paper_T5 = the paper's numbers on its unnamed CUDA 10.1 GPU with its own unpublished "
                    "workload draw: context, not a like-for-like target"}


def cpu_baseline_paths(budget_s=4.0):
    """The oracle's modified Dijkstra (one O(V^2) label-setting search per query, OpenMP over
    queries) on a sample of the paths workload."""
    from oracle import oracle as O
    cores = len(os.sched_getaffinity(0))
    g, q = path_workload(0)
    nq = 256
    while True:
        t = time.perf_counter()
        O.graph_paths(g, q["src"][:nq], q["dst"][:nq], q["demand"][:nq], max_hops=8, nthreads=cores)
        el = time.perf_counter() - t
        if el > budget_s / 4 or nq >= 1 << 16:
            break
        nq *= 4
    return {"value": nq / el, "unit": "paths/s", "cores": cores, "kind": "oracle",
            "sample": f"first {nq} queries of the workload, C++ oracle Dijkstra per query, {el:.1f} s"}


def cpu_baseline_sim(n_req=1000):
    """The oracle's event loop (TOPSIS Flat) on the first n_req requests of the E2 campaign."""
    from oracle import oracle as O
    snap = gen.snapshot(20, warm=False)
    reqs, arrival, duration = gen.sim_workload()
    sub = gen.subset(reqs, np.arange(n_req))
    t = time.perf_counter()
    r = O.simulate(snap, sub, arrival[:n_req], duration[:n_req], "topsis", "flat", max_ticks=5000)
    el = time.perf_counter() - t
    return {"value": r["totals"]["attempts"] / el, "unit": "attempts/s", "cores": 1, "kind": "oracle",
            "sample": f"E2, first {n_req} requests, TOPSIS Flat, sequential C++ oracle, {el:.1f} s "
                      f"({r['totals']['pod_steps']} pod steps)"}


def cpu_baseline(snap, reqs, budget_s=15.0, method="topsis"):
    """The oracle as it stands, on the host cores, on a bounded sample of the workload."""
    from oracle import oracle as O
    cores = len(os.sched_getaffinity(0))
    n_req = 64
    while True:
        sub = gen.subset(reqs, np.arange(n_req))
        t = time.perf_counter()
        _, cnt, _ = O.schedule(snap, sub, method, "flat", sequential=False, nthreads=cores)
        el = time.perf_counter() - t
        if el > budget_s / 4 or n_req >= reqs["n_requests"]:
            break
        n_req = min(reqs["n_requests"], int(n_req * max(2.0, budget_s / max(el, 1e-3) / 2)))
    return {"value": cnt["pod_steps"] / el, "unit": "pods/s", "cores": cores, "kind": "oracle",
            "sample": f"first {n_req} requests of the workload ({cnt['pod_steps']} pod steps), "
                      f"{method} flat, C++ double oracle, OpenMP over requests, {el:.1f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    snap, reqs, name = workload(0, "topsis")
    from oracle import oracle as O
    O.build()
    cores = len(os.sched_getaffinity(0))
    sample = gen.subset(reqs, np.arange(256))
    for _ in range(args.warmup):
        O.schedule(snap, gen.subset(reqs, np.arange(16)), "topsis", "flat", sequential=False, nthreads=cores)
    t = time.perf_counter()
    pods = 0
    for _ in range(args.steps):
        _, cnt, _ = O.schedule(snap, sample, "topsis", "flat", sequential=False, nthreads=cores)
        pods += cnt["pod_steps"]
    el = time.perf_counter() - t
    value = pods / el
    desc = f"first 256 requests of the workload per step ({pods // max(args.steps, 1)} pod steps), C++ double oracle"
    print(json.dumps({"impl": "reference", "metric": "pods placed/sec (and servers ranked/sec)", "value": value,
                      "unit": "pods/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                      "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
                      "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                      "config": {"workload": name, "k": 32, "method": "topsis", "schema": "flat"},
                      "cpu_baseline": {"value": value, "unit": "pods/s", "cores": cores, "kind": "oracle",
                                       "sample": desc},
                      "e2e": {"value": value, "unit": "pods/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def self_launch(args) -> int:
    """--gpus N > 1 without a torchrun environment: launch N ranks (one process per GPU) with
    torchrun on 127.0.0.1 and pass the JSON line through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the communicator lines name the N ranks
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    rank, world, local = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
