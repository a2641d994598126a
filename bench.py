#!/usr/bin/env python
"""Benchmark of the FD block-preconditioner application (BASELINE.json metric: preconditioner
applications/s and DOF/s in FP64, % of the FP64 tensor-core roofline).

One step = one block_precond_apply (P_D^{-1} r, or (P_D^G)^{-1} r for config 3) over one batch of
synthetic RHS already resident in HBM: the whole hot path. Default workload
= BASELINE.json configs[4] (config 5: 3D Raviart-Thomas p=4, 512^3 elements, 548.8 M dofs), the
largest configuration that fits one GPU and the one the FP64 tensor-core target is about (SURVEY.md
§8(d) D-3); --config selects the others (parity-test cases, not bench lines).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl {fdp,reference}]

N > 1 runs under torchrun, one rank per GPU. Config 5 is slab-decomposed (i3 planes split over
the ranks, exchanges fused into the contraction epilogues as NVLink peer stores; strong scaling);
configs 1-3 have no natural sharding ("replicas only": each rank applies the preconditioner to its
own RHS stream); config 4 shards its batch of 8 RHS across ranks.
--impl reference times the CPU oracle (the reference arm of this tier) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--rt-reading", default="paper", choices=["paper", "literal"],
                    help="RT own-direction regularity: the paper's alpha+1 (default) or configs 3/5's "
                         "literal 'C^3' wording, alpha (SURVEY.md C-3; a secondary row)")
    ap.add_argument("--impl", default="fdp", choices=["fdp", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="budget of the oracle sample")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------------------------
# workload description (counts only; no method arithmetic beyond sizes)
# ----------------------------------------------------------------------------------------------
_RT_LITERAL = False


def RT_OWN_ALPHA(w):
    """RT own-direction regularity for --rt-reading literal, else the paper's."""
    return (w.p - 1) if (_RT_LITERAL and w.disc == "RT") else None


def l2_policy(n_total, batch):
    """L2 handling of the timed loop, a function of the workload only (the same string in both
    arms): working sets below 2x the 126 MB L2 are flushed before every timed step."""
    ws = 2 * 8 * n_total * batch
    if ws < 2 * (126 << 20):
        return True, "flushed before every timed step (512 MB written, then read back)"
    return False, f"working set {ws / 1e9:.2f} GB > L2 (126 MB): no flush needed"


def batch_layout(cid, w, gpus, rank=0):
    """(items of this rank, global batch) -- config 5 at N > 1: one RHS slab-sharded; config 4:
    its 8 RHS dealt round-robin; configs 1-3: every rank its own replica stream."""
    if cid == 5 and gpus > 1:
        return [0], 1
    if cid == 4:
        return list(range(rank, w.batch, gpus)), w.batch
    return list(range(w.batch)), w.batch * gpus


def workload_config(cid, w, n_total, gpus):
    items, batch_total = batch_layout(cid, w, gpus)
    _, l2 = l2_policy(n_total, len(items))
    return {
        "workload": w.name + ("_literal_c3" if (_RT_LITERAL and w.disc == "RT") else ""),
        "config_index": cid,
        "discretization": f"{w.dim}D {w.disc} pressure p={w.p}, velocity p={w.p + 1}, alpha=p-1, {w.n_el}^{w.dim} elements",
        "preconditioner": "P_D^G (D_V=nu, D_Q=1/nu at dofs)" if w.variable_nu else "P_D",
        "dofs_per_rhs": n_total,
        "global_batch": batch_total,
        "parallelism": (("slab-" + os.environ.get("FDP_SLAB_EXCHANGE", "peer")) if cid == 5 and gpus > 1
                        else "batch-shard" if cid == 4 else "replicas") + f"x{gpus}",
        "l2": l2,
        "rhs": f"numpy default_rng(seed={w.seed}).standard_normal, FP64",
    }


def nvml_sampler(stop, out, dev):
    """Fast NVML polling (~1 kHz) so that even a millisecond-scale timed region gets samples;
    each sample is (host time, SM MHz, max SM MHz, reason flags as 'Active' / 'Not Active')."""
    import pynvml
    pynvml.nvmlInit()
    try:
        h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        bits = [getattr(pynvml, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
                getattr(pynvml, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                getattr(pynvml, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                getattr(pynvml, "nvmlClocksThrottleReasonSwPowerCap", 0x4)]
        while not stop.is_set():
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            flags = ["Active" if rs & b else "Not Active" for b in bits]
            out.append((time.perf_counter(), [str(sm), str(mx), str(rs)] + flags))
            stop.wait(0.001)
    finally:
        pynvml.nvmlShutdown()


def clock_sampler(stop, out, dev):
    try:
        nvml_sampler(stop, out, dev)
    except Exception:
        nvsmi_sampler(stop, out, dev)


def nvsmi_sampler(stop, out, dev):
    q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    while not stop.is_set():
        try:
            r = subprocess.run(["nvidia-smi", f"--id={dev}", f"--query-gpu={q}",
                                "--format=csv,noheader,nounits"], capture_output=True, text=True,
                               timeout=5)
            if r.returncode == 0 and r.stdout.strip():
                out.append((time.perf_counter(), [x.strip() for x in r.stdout.strip().split(",")]))
        except Exception:
            pass
        stop.wait(0.2)


def summarize_clocks(samples, t0=None, t1=None):
    """Median SM clock and the throttle reasons seen, from the samples taken inside the timed
    region [t0, t1] (host clock); the nearest samples around it if none fell inside."""
    inside = [s for t, s in samples if t0 is None or t0 <= t <= t1]
    if not inside and samples:
        inside = [min(samples, key=lambda ts: abs(ts[0] - (t0 or 0.0)))[1]]
    samples = inside
    if not samples:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
    sm = [float(s[0]) for s in samples if s[0].replace(".", "").isdigit()]
    mx = [float(s[1]) for s in samples if s[1].replace(".", "").isdigit()]
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    reasons = set()
    for s in samples:
        for nm, v in zip(names, s[3:7]):
            if v.lower() == "active":
                reasons.add(nm)
    return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
            "reasons": sorted(reasons), "samples": len(samples)}


# ----------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# ----------------------------------------------------------------------------------------------
def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip() + f" x {os.cpu_count()} threads"
    except Exception:
        pass
    return None


def oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(w, budget_s, max_steps=None):
    """Time the oracle's block-preconditioner apply on this workload's RHS, one RHS per call,
    for about budget_s seconds. Returns (applies/s, dofs/apply, n_calls, seconds, setup_s)."""
    from oracle import precond, spaces
    t0 = time.perf_counter()
    od = spaces.build(w.dim, w.disc, w.p, w.n_el, rt_own_alpha=RT_OWN_ALPHA(w))
    dv = dq = None
    if w.variable_nu:
        dv, dq = spaces.nu_scalings(od, synth.viscosity)
    P = precond.BlockPrecond(od, dv, dq)
    setup = time.perf_counter() - t0
    r = synth.rhs(w.seed, od.n_total, 1)[0]
    P.apply(r)  # warm
    n, t = 0, 0.0
    times = []
    while (t < budget_s or n == 0) and (max_steps is None or n < max_steps):
        a = time.perf_counter()
        P.apply(r)
        dt = time.perf_counter() - a
        times.append(dt)
        t += dt
        n += 1
    return n / t, od.n_total, n, t, setup, times


def run_reference(args, w, cid):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    # rank 0 runs alone: give the oracle every host core (torchrun sets OMP_NUM_THREADS=1)
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=os.cpu_count() or 1)
    except Exception:
        pass
    # each step = one oracle application to one RHS (bounded: the whole run stays within minutes)
    steps, warm = args.steps, max(args.warmup, 3)  # the GPU arm's warm-up floor
    from oracle import precond, spaces
    od = spaces.build(w.dim, w.disc, w.p, w.n_el, rt_own_alpha=RT_OWN_ALPHA(w))
    dv = dq = None
    if w.variable_nu:
        dv, dq = spaces.nu_scalings(od, synth.viscosity)
    P = precond.BlockPrecond(od, dv, dq)
    r = synth.rhs(w.seed, od.n_total, 1)[0]
    # every step is one full oracle application to one RHS of the workload (batch item 0): the run
    # honours --steps / --warmup exactly, so its line is comparable step for step with the GPU
    # arm's (config 5: ~24 s per application on 16 host cores, ~10 min for 20 + 5 steps)
    for _ in range(warm):
        P.apply(r)
    t0 = time.perf_counter()
    for _ in range(steps):
        P.apply(r)
    dt = time.perf_counter() - t0
    value = steps / dt
    cores = oracle_threads()
    line = {
        "impl": "reference", "metric": "preconditioner_applications_per_s", "value": value,
        "unit": "apply/s", "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": 1e3 * dt / steps, "higher_is_better": True, "scaling": "strong" if cid in (4, 5) else "weak",
        # BASELINE.md §2.1 holds the paper's own per-apply time at config 2's size (P_D, 866,750
        # dofs: 9.94 s / 166 applications = 59.9 ms on one Haswell-E thread):
        # context from another machine, not a target
        "vs_baseline": (value / (166 / 9.94)) if cid == 2 else None,
        "vs_baseline_source": ("BASELINE.md §2.1: 59.9 ms per P_D apply at config 2's size (paper, "
                               "MATLAB, one Haswell-E thread)") if cid == 2 else None, "dtype": "f64", "data": "synthetic",
        "dof_per_s": value * od.n_total,
        "config": workload_config(cid, w, od.n_total, args.gpus),
        "cpu_baseline": {"value": value, "unit": "apply/s", "cores": cores, "kind": "oracle",
                         "sample": f"{steps} oracle applications (numpy/scipy FP64) to one RHS of {w.name} "
                                   f"(batch item 0), after {warm} untimed ones; one application = one "
                                   f"step of the GPU arm's workload per RHS"},
        "e2e": {"value": value, "unit": "apply/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------------------------
def main():
    global _RT_LITERAL
    args = parse()
    _RT_LITERAL = args.rt_reading == "literal"
    cid = args.config
    w = synth.CONFIGS[cid]
    if args.impl == "reference":
        run_reference(args, w, cid)
        return

    import torch
    import torch.distributed as dist
    import paper_1712_00403_b200 as fdp

    rank, world, local = dist_env()
    if world > 1:
        # FDP_BENCH_SHARED_GPU=1 (host-logic check only): every rank on cuda:0 with gloo
        # collectives, for exercising the multi-rank code path on a one-GPU box; not a measurement
        if os.environ.get("FDP_BENCH_SHARED_GPU"):
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    torch.cuda.init()

    # ---- setup (excluded from timing) ----
    t0 = time.perf_counter()
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el, rt_own_alpha=RT_OWN_ALPHA(w))
    dv = dq = None
    if w.variable_nu:
        dv, dq = fdp.nu_scalings(gd, synth.viscosity_separable(gd.D))
    P = fdp.build_block(gd, device=dev, dscale_vel=dv, dscale_pres=dq)
    setup_s = time.perf_counter() - t0
    n_total = gd.n_total

    # config 5 at N > 1: slab decomposition with NCCL all-to-all exchanges (strong scaling)
    slab = cid == 5 and world > 1
    exchange = None
    if slab:
        from paper_1712_00403_b200 import dist as fdist
        # default: exchanges fused into the contraction epilogues (peer stores over NVLink,
        # DESIGN.md §9); FDP_SLAB_EXCHANGE=nccl selects the NCCL all-to-all baseline
        exchange = os.environ.get("FDP_SLAB_EXCHANGE", "peer")
        SB = None
        if exchange == "peer":
            try:
                SB = fdist.PeerSlabBlockPrecond(P)
                ok = 1.0
            except Exception as e:  # no CUDA IPC / peer access between the ranks' GPUs
                print(f"peer-store exchange unavailable ({e}); using NCCL all-to-all", file=sys.stderr)
                ok = 0.0
            flag = torch.tensor([ok], device=f"cuda:{dev}")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)  # every rank takes the same path
            if flag.item() < 1.0:
                if SB is not None:
                    SB.close()
                SB = None
                exchange = "nccl"
        if SB is None:
            SB = fdist.SlabBlockPrecond(P)
    # batch per rank: config 4 shards its 8 RHS across ranks; others replicate one RHS stream
    items, batch_total = batch_layout(cid, w, world, rank)
    batch = len(items)
    if batch == 0:
        raise SystemExit("more ranks than RHS for this config")
    if slab:
        # timing workload: this rank's slabs drawn from its own seeded stream (FD cost is
        # data-independent; slab parity is tested separately against the oracle)
        r_host = synth.rhs(w.seed + 1000 * rank, SB.local_n, 1)
        ws = SB.ws
    else:
        rhs_all = synth.rhs(w.seed + (rank if cid != 4 else 0), n_total, w.batch)
        r_host = np.ascontiguousarray(rhs_all[items])
        del rhs_all
        ws = P.workspace(batch)
    r = torch.from_numpy(r_host).to(dev)
    s = torch.empty_like(r)
    flush, _ = l2_policy(n_total, batch)
    flush_buf = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev) if flush else None
    stream = torch.cuda.current_stream()

    def flush_l2():
        # write a buffer 4x the L2, then read it back: the timed step starts on an L2 full of
        # clean lines (a write-only flush leaves ~126 MB of dirty lines whose write-back would
        # compete with the step's own traffic and made config-2 timings vary by 15%)
        flush_buf.zero_()
        torch.sum(flush_buf, dtype=torch.int64)

    def step():
        if slab:
            SB.apply(r[0], s[0], stream=stream)
        else:
            P.apply(r, s, batch=batch, workspace=ws, stream=stream)

    # ---- warmup ----
    for _ in range(max(args.warmup, 3)):
        if flush:
            flush_l2()
        step()
    torch.cuda.synchronize()

    # ---- timed region (device events per step; L2 flushed between steps when resident) ----
    stop = threading.Event()
    samples = []
    th = threading.Thread(target=clock_sampler, args=(stop, samples, dev), daemon=True)
    th.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    wall0 = time.perf_counter()
    for i in range(args.steps):
        if flush:
            flush_l2()
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    dev_ms = float(sum(step_ms))

    # ---- per-launch roofline pass (events between launches, same graph path) ----
    prof_runs = []
    if not slab:
        P.profile(True)
        for i in range(max(3, min(args.steps, 20))):
            if flush:
                flush_l2()
            step()
            torch.cuda.synchronize()
            if i >= 1:
                prof_runs.append(P.profile_read())
        P.profile(False)

    # ---- end-to-end through the public host-buffer API (H2D + apply + D2H inside) ----
    # page-locked buffers from libfdp (cudaMallocHost): H2D from torch's pinned allocator ran at
    # 14 GB/s vs 54 GB/s from these on the B200 boxes (probes/pcie_bw.py, probes/h2d_bw.cu)
    r_np = fdp.host_empty(r_host.shape)
    r_np[...] = r_host
    s_np = fdp.host_empty(r_host.shape)
    r_pin = torch.from_numpy(r_np)
    s_pin = torch.from_numpy(s_np)

    def e2e_step():
        if slab:  # Python-level public API: pinned H2D, sharded apply, D2H, sync
            r.copy_(r_pin, non_blocking=True)
            SB.apply(r[0], s[0], stream=stream)
            s_pin.copy_(s, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        else:
            P.apply_host(r_pin.numpy(), s_pin.numpy(), batch=batch)

    e2e_step()
    torch.cuda.synchronize()
    e2e_steps = max(3, min(args.steps, 20))
    if world > 1:
        dist.barrier()
    e0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = time.perf_counter() - e0
    stop.set()
    th.join(timeout=5)

    # ---- reduce over ranks ----
    stats = torch.tensor([dev_ms, e2e_s, wall], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    dev_ms_max, e2e_max, wall_max = [float(x) for x in stats.cpu()]
    apps_total = batch_total * args.steps
    value = apps_total / (dev_ms_max * 1e-3)
    e2e_value = batch_total * e2e_steps / e2e_max

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel (K1 mode contraction): algorithmic flops / event duration
    peaks = json.load(open(PEAKS_FILE))
    fp64_peak = peaks["dmma_tflops_w32"]
    k1_ms = k1_fl = 0.0
    k1_n = 0
    tot_ms = 0.0
    per_kind = {0: 0.0, 1: 0.0, 2: 0.0}
    k3_ms = k3_by = 0.0
    for run in prof_runs:
        for kind, ms, fl, by in run:
            tot_ms += ms
            per_kind[kind] += ms
            if kind == 0:
                k1_ms += ms
                k1_fl += fl
                k1_n += 1
            if kind == 2:
                k3_ms += ms
                k3_by += by
    k1_family = (k1_fl / (k1_ms * 1e-3)) / 1e12 if k1_ms > 0 else None
    # the dominant kernel: the K1-family launch with the largest share of the profiled step
    # (launch positions are the same in every profiled apply); its executed flops / mean duration
    dom = None
    if prof_runs:
        nl = min(len(r) for r in prof_runs)
        means = []
        for i in range(nl):
            ms_i = float(np.mean([r[i][1] for r in prof_runs]))
            fl_i = float(np.mean([r[i][2] for r in prof_runs]))
            means.append((ms_i, fl_i, prof_runs[0][i][0], i))
        k1 = [m for m in means if m[2] == 0 and m[1] > 0]
        if k1:
            ms_i, fl_i, _, idx = max(k1)
            dom = {"launch_index": idx, "mean_ms": ms_i, "flops_per_launch": fl_i,
                   "share_of_step": ms_i / (tot_ms / len(prof_runs)) if tot_ms else None,
                   "achieved": fl_i / (ms_i * 1e-3) / 1e12,
                   # ordinal among the step's FD-transform launches (K1t on configs 4-5: forward
                   # modes 1, 2, 3 (Lambda), backward modes 3, 2, 1)
                   "transform_ordinal": [m[3] for m in k1].index(idx)}
    achieved = dom["achieved"] if dom else k1_family
    # the dense FD's work (4 N_k sum_d n_d per component and RHS) at the same
    # K1 time: what the even-odd folding saves shows as dense_equiv > achieved
    dense_fl = sum(4.0 * float(np.prod(d)) * sum(d) for d in gd.comp_dims) * batch_total / world
    dense_equiv = (dense_fl * len(prof_runs) / (k1_ms * 1e-3)) / 1e12 if k1_ms > 0 else None
    # DRAM traffic per K1 launch from the committed ncu --set full capture of this config
    traffic = traffic_src = None
    ncu_json = ""
    for tag in ("r02g", "r02", "r01"):  # the newest committed capture of this config
        ncu_json = os.path.join(ROOT, "profiles", f"{tag}_ncu_cfg{cid}.json")
        if os.path.exists(ncu_json):
            break
    if os.path.exists(ncu_json):
        # the dominant launch's kernel: the plane kernel (plane path) or the folded K1 forward
        # (FOLD = 1, the fourth template argument); else every FD-transform kernel captured
        allk = [k for k in json.load(open(ncu_json)).get("kernels", []) if "mode_" in k["kernel"]]
        ks = [k for k in allk if "mode_plane" in k["kernel"]]
        if not ks and dom is not None and dom.get("transform_ordinal", 9) < 6:
            # K1t: the captures of the dominant pass's kernel mode_tma_kernel<KMAJ, FOLD, STAGES>
            # (passes: fwd 1 <1,1>, fwd 2 <0,1>, fwd 3 + Lambda <0,1> (also reads the 1/Lambda
            # table: DRAM reads > 1.5x writes), bwd 3 <0,2>, bwd 2 <0,2>, bwd 1 <1,2>)
            o = dom["transform_ordinal"]
            km, fo = [("1", "1"), ("0", "1"), ("0", "1"), ("0", "2"), ("0", "2"), ("1", "2")][o]
            def targ(k):
                a = k["kernel"].split("mode_tma_kernel<")[1].split(",")
                return a[0].strip(), a[1].strip()
            ks = [k for k in allk if "mode_tma_kernel<" in k["kernel"] and targ(k) == (km, fo)]
            if o in (1, 2):
                lam = lambda k: (k["dram_read_bytes"] or 0) > 1.5 * (k["dram_write_bytes"] or 1)
                ks = [k for k in ks if lam(k) == (o == 2)]
        if not ks:
            ks = [k for k in allk if "fold_kernel<" in k["kernel"]
                  and k["kernel"].split("fold_kernel<")[1].split(",")[3].strip() == "1"]
        what = "dominant kernel"
        if not ks:
            ks, what = allk, "all captured FD-transform kernels"
        if ks:
            traffic = float(np.mean([(k["dram_read_bytes"] or 0) + (k["dram_write_bytes"] or 0) for k in ks]))
            traffic_src = (f"{os.path.relpath(ncu_json, ROOT)} (DRAM read + write per launch, mean of "
                           f"{len(ks)} captured launches of the {what}; ncu --set full, cold cache)")
    launches = P.launch_count(batch)
    roof_kind = "per-launch CUDA events of K1 inside the apply graph"
    if slab:
        # K1 algorithmic flops of one full apply / G per rank over the whole step time
        # (a lower bound: includes the two exchanges)
        fl = sum(4.0 * float(np.prod(d)) * sum(d) for d in gd.comp_dims)
        achieved = fl / world / (dev_ms_max / args.steps * 1e-3) / 1e12
        per_kind[0] = tot_ms = 1.0
        launches = 3 * 7 + 5
        roof_kind = "K1 flops / step time per rank (includes exchanges; lower bound)"
    
    clocks = summarize_clocks(samples, wall0, wall0 + wall)
    cpu = None
    if not args.no_cpu_baseline:
        os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
        v, nd, n, t, setup_o, _ = oracle_sample(w, args.cpu_seconds)
        cpu = {"value": v, "unit": "apply/s", "cores": oracle_threads(), "kind": "oracle",
               "sample": f"{n} oracle applications (numpy/scipy FP64) to one RHS of {w.name} in {t:.1f} s; setup {setup_o:.2f} s excluded",
               "cpu_model": cpu_model()}
        if cid in (1, 2, 3):
            # also one thread, the paper's protocol
            try:
                from threadpoolctl import threadpool_limits
                with threadpool_limits(limits=1):
                    v1, _, n1, t1, _, _ = oracle_sample(w, min(args.cpu_seconds, 8.0))
                cpu["one_thread"] = {"value": v1, "unit": "apply/s", "cores": 1,
                                     "sample": f"{n1} oracle applications in {t1:.1f} s"}
            except Exception as e:  # pragma: no cover - threadpoolctl missing
                cpu["one_thread"] = {"unavailable": str(e)}
    line = {
        "metric": "preconditioner_applications_per_s",
        "value": value,
        "unit": "apply/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": dev_ms_max / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if cid in (4, 5) else "weak",
        # BASELINE.md §2.1 holds the paper's own per-apply time at config 2's size (P_D, 866,750
        # dofs: 9.94 s / 166 applications = 59.9 ms on one Haswell-E thread):
        # context from another machine, not a target
        "vs_baseline": (value / (166 / 9.94)) if (cid == 2 and not slab) else None,
        "vs_baseline_source": ("BASELINE.md §2.1: 59.9 ms per P_D apply at config 2's size (paper, "
                               "MATLAB, one Haswell-E thread)") if (cid == 2 and not slab) else None,
        "dtype": "f64",
        "data": "synthetic",
        "dof_per_s": value * n_total,
        "config": workload_config(cid, w, n_total, world),
        "roofline": {
            "bound": "tensor",
            "kernel": "the dominant FD-transform launch of the step, the one with the largest mean "
                      "time (config 2/3: the plane kernel mode_plane_kernel; configs 4/5: a pass of "
                      "the TMA-fed folded transform mode_tma_kernel (K1t), dominant_launch."
                      "transform_ordinal = fwd modes 1, 2, 3, bwd modes 3, 2, 1); FP64 mma.sync "
                      "m8n8k4 -> DMMA",
            "achieved": achieved,
            "dominant_launch": dom,
            "k1_family": {"achieved": k1_family,
                          "frac": (k1_family / fp64_peak) if k1_family else None,
                          "what": "all FD-transform launches of the step: executed flops / their time"},
            "peak": fp64_peak,
            "unit": "TFLOP/s",
            "frac": (achieved / fp64_peak) if achieved else None,
            "flops_counted": "as executed: 2 R (ne^2 + no^2) per folded m-mode product, 2 R n^2 "
                             "per dense one (DESIGN.md §8)",
            "dense_fd_equiv": {"achieved": dense_equiv,
                               "frac": (dense_equiv / fp64_peak) if dense_equiv else None,
                               "flops_per_apply": dense_fl / max(1, batch_total / world),
                               "source": "SURVEY.md §8(d) D-4 dense FD flops over the same K1 time"},
            "traffic": traffic,
            "traffic_source": traffic_src,
            "peak_source": "measured all-SM DMMA register loop, profiles/r01_fp64_peaks.json (MEASURED_PEAKS.json has no FP64 entry)",
            "measured_as": roof_kind,
            "k1_share_of_step": per_kind[0] / tot_ms if tot_ms else None,
            "k1_launches_per_step": k1_n // max(1, len(prof_runs)),
            "k3_mass_gbs": (k3_by / (k3_ms * 1e-3) / 1e9) if k3_ms else None,
            "step_ms_profiled": tot_ms / max(1, len(prof_runs)),
        },
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "apply/s",
                "h2d_bytes_per_step": int(r_host.nbytes), "d2h_bytes_per_step": int(r_host.nbytes),
                "api": (f"pinned H2D + slab apply ({exchange} exchange) + D2H + sync" if slab
                        else "block_precond_apply_host (pinned host buffers, H2D+apply+D2H+sync)")},
        "gpu_launches": launches * args.steps,
        "clocks": clocks,
        "setup_s": setup_s,
        "wall_s_timed_region": wall_max,
        "step_ms_p50": float(np.median(step_ms)),
        "step_ms_p10": float(np.percentile(step_ms, 10)),
        "step_ms_p90": float(np.percentile(step_ms, 90)),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
