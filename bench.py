#!/usr/bin/env python
"""Benchmark of the Δ-matrix SA hot path (arXiv 1208.2675) on B200.

BASELINE.json metric: "SA iterations/s (1 chain, N=100); chain-iterations/s at 1/2/4/8 B200".

  N = 1 (default): headline = one whole config-3 job per step: qap_reset (device-resident p0) +
      qap_delta_init + qap_sa_run over I = 1e8 iterations of the N=100 tai100a-shaped instance.
      The config-5 ensemble (8192 chains x 1e7) is reported nested under "ensemble".
  N > 1: headline = BASELINE config 5, chain-iterations/s of 8192 independent N=100 chains x 1e7
      iterations split over the N ranks (dist.ensemble_distributed: chain-keyed start
      permutations generated on each device, one NCCL min-reduce of (best cost, chain) and a
      broadcast of the winning permutation) -> strong scaling, identical best cost / chain for
      every N.  The single-chain figure is nested under "single_chain" (one replica per rank).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--dry-run]

--gpus N > 1 without WORLD_SIZE in the environment relaunches itself under
torch.distributed.run with N ranks (127.0.0.1 rendezvous).  --dry-run exercises only the host
path (launch, rank environment, chain partition, collectives on gloo, JSON line) with no GPU work.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from qap_inputs import SA_SEED, config  # noqa: E402

METRIC_1 = "SA iterations/s (1 chain, N=100)"
UNIT_1 = "iterations/s"
METRIC_N = "chain-iterations/s (8192 x N=100 chains, BASELINE config 5)"
UNIT_N = "chain-iterations/s"
SMEM_BYTES_PER_CLK = 128          # per SM, B300_MICROARCH.md "smem crossbar BW 128/N B/cyc/SM"
BYTES_PER_PROPOSAL = 4            # one int32 Δ read per proposed swap


def bytes_per_accept(n: int, sa: int = 1, sb: int = 1) -> int:
    """Algorithmic on-chip bytes one accepted swap must move:
    disjoint Δ read+write, touching Δ writes, rows A_v/B'_v of every touching v, rows r,s,
    staging writes, B' row/column exchange.  60.4 KB at N = 100 (8-bit A, B)."""
    disjoint = (n - 2) * (n - 3) // 2
    touching = 2 * n - 3
    return (8 * disjoint + 4 * touching + (n - 2) * n * (sa + sb) + 2 * n * (sa + sb)
            + 4 * n + 4 * n * sb + 4 * n * sb)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- clocks --
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        mhz, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                mhz.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(mhz)}


# ------------------------------------------------------------ peaks -----
def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def profile_summary(kernel):
    """ncu-derived facts of a kernel from the committed summary (profiles/ncu_summary.json):
    dram bytes per launch (--set full), issue-slot utilisation, SM cycles per accepted swap."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get("kernels", {}).get(kernel, {})
    except Exception:
        return {}


def smem_peak(clocks, peaks, sms=1):
    """One (or `sms`) SM's shared-memory bandwidth: 128 B/clk/SM (B300_MICROARCH.md, B200_PROFILING
    fallback: no measured shared-memory peak in MEASURED_PEAKS.json) x the SM clock measured under
    load during the timed region (nvidia-smi median), else sm_max_mhz."""
    mhz = (clocks or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    src = ("128 B/clk/SM (B300_MICROARCH.md 'smem crossbar 128/N B/cyc/SM'; MEASURED_PEAKS.json has "
           f"no shared-memory peak) x {mhz:.0f} MHz (SM clock measured during the timed region)"
           + (f" x {sms} SMs" if sms > 1 else ", one SM"))
    return SMEM_BYTES_PER_CLK * mhz * 1e6 * sms / 1e9, src, mhz


def host_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


# -------------------------------------------------------- distributed ---
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args, argv):
    """--gpus N > 1 outside torchrun: relaunch this script with N ranks (one per GPU)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")             # communicator lines show the N ranks
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *argv]
    log("bench: launching", " ".join(cmd))
    return subprocess.call(cmd, env=env)


# ---------------------------------------------------------- reference ---
def run_reference(args):
    """The oracle (oracle/, plain C, as it stands) on the host cores, bounded samples of the
    workload of our arm at this N (config 3 at N = 1, config 5 at N > 1)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O
    host = host_info()
    times = []
    if ws == 1:
        A, B, p0, cfg = config(3)
        I = cfg["iters"]
        sch = O.geometric_schedule_for(A, B, p0, I)
        sample = args.ref_sample
        for step in range(args.warmup + args.steps):
            run = O.Run(A, B, p0, mode=O.MODE_SCRATCH)
            t = time.perf_counter()
            run.run(0, sample, sch, SA_SEED)
            dt = time.perf_counter() - t
            if step >= args.warmup:
                times.append(dt)
        ms = 1e3 * statistics.mean(times)
        value = sample / (ms / 1e3)
        metric, unit, cores = METRIC_1, UNIT_1, 1
        desc = (f"oracle SCRATCH-mode sequential SA, iterations [0,{sample}) of config 3's "
                f"1e8-iteration schedule, 1 host thread")
        cfgd = {"workload": "config3 tai100a-shaped N=100, 1 chain (sampled prefix)", "n": 100,
                "iters_per_step": sample}
    else:
        A, B, _, cfg = config(5)
        n, I = cfg["n"], cfg["iters"]
        cores = os.cpu_count() or 1
        count = max(cores, args.ref_chains)
        sch = O.geometric_schedule_for(A, B, O.start_perm(n, SA_SEED, 0), I)
        for step in range(args.warmup + args.steps):
            t = time.perf_counter()
            O.ensemble_run(A, B, None, 0, I, sch, SA_SEED, threads=cores, mode=O.MODE_SCRATCH,
                           count=count)
            dt = time.perf_counter() - t
            if step >= args.warmup:
                times.append(dt)
        ms = 1e3 * statistics.mean(times)
        value = count * I / (ms / 1e3)
        metric, unit = METRIC_N, UNIT_N
        desc = (f"oracle thread pool ({cores} threads), chains 0..{count - 1} of config 5 "
                f"(1e7 iterations each, SCRATCH mode)")
        cfgd = {"workload": f"config5 ensemble N=100 (sampled: {count} of 8192 chains)", "n": n,
                "chains_per_step": count, "iters_per_chain": I}
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if ws == 1 else "strong", "vs_baseline": None, "dtype": "int32+f64",
        "data": "synthetic", "config": dict(cfgd, l2="n/a (host)"),
        "cpu_baseline": dict({"value": value, "unit": unit, "cores": cores, "kind": "oracle",
                              "sample": desc}, **host),
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(sample):
    """Config 3: the oracle (SCRATCH mode, one thread) over a bounded prefix of the schedule."""
    import oracle as O
    A, B, p0, cfg = config(3)
    sch = O.geometric_schedule_for(A, B, p0, cfg["iters"])
    run = O.Run(A, B, p0, mode=O.MODE_SCRATCH)
    t = time.perf_counter()
    run.run(0, sample, sch, SA_SEED)
    dt = time.perf_counter() - t
    return dict({"value": sample / dt, "unit": UNIT_1, "cores": 1, "kind": "oracle",
                 "sample": f"oracle SCRATCH mode, iterations [0,{sample}) of config 3's 1e8 schedule "
                           f"({dt:.1f} s, 1 thread)"}, **host_info())


def cpu_baseline_ensemble(chains):
    """Config 5: the oracle's thread pool (all host cores, SCRATCH mode) over a bounded sample of
    chains, each its full 1e7 iterations."""
    import oracle as O
    A, B, _, cfg = config(5)
    n, I = cfg["n"], cfg["iters"]
    cores = os.cpu_count() or 1
    count = max(cores, chains)
    sch = O.geometric_schedule_for(A, B, O.start_perm(n, SA_SEED, 0), I)
    t = time.perf_counter()
    O.ensemble_run(A, B, None, 0, I, sch, SA_SEED, threads=cores, mode=O.MODE_SCRATCH, count=count)
    dt = time.perf_counter() - t
    return dict({"value": count * I / dt, "unit": UNIT_N, "cores": cores, "kind": "oracle",
                 "sample": f"oracle thread pool, chains 0..{count - 1} of config 5 x 1e7 iterations "
                           f"({dt:.1f} s, {cores} threads)"}, **host_info())


# --------------------------------------------------------------- ours ---
def single_chain(args, Q, local, stream, pg, ws):
    """Config 3 (N=100, 1e8 iterations), one chain per rank; returns the measured facts."""
    import torch
    A, B, p0, cfg = config(3)
    n, I = cfg["n"], cfg["iters"]
    s = Q.Solver(A, B, p0, device=local, stream=stream.cuda_stream)
    s.delta_init()
    t0, tf = s.schedule_bounds()                     # R2 rule on the device
    sch = Q.make_schedule(Q.QAP_COOL_GEOMETRIC, t0, tf, I)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def step():
        s.reset()                                    # p0 already resident in HBM
        s.delta_init()
        return s.run(0, I, sch, SA_SEED)

    for _ in range(args.warmup):
        step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kern_ms, sc, stats = [], [], []
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()                            # L2 flush between timed steps (outside events)
            ev[i][0].record(stream)
            st = step()
            ev[i][1].record(stream)
            stats.append(st)
            kern_ms.append(s.last_kernel_time()[0])
            sc.append(s.last_scratch_time())
        torch.cuda.synchronize()
    if pg:
        pg.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    if pg:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    launches = (2 + s.last_kernel_time()[1]) * args.steps

    # e2e through the public API with host buffers (create copies A, B, p0; state read back)
    e2e_ms = []
    for _ in range(max(1, args.e2e_steps)):
        torch.cuda.synchronize()
        t = time.perf_counter()
        with Q.Solver(A, B, p0, device=local, stream=stream.cuda_stream) as s2:
            s2.delta_init()
            s2.run(0, I, sch, SA_SEED)
            s2.state(want_delta=False)
        e2e_ms.append(1e3 * (time.perf_counter() - t))
    e2e_t = statistics.median(e2e_ms)
    if pg:
        t = torch.tensor([e2e_t], device="cuda", dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_t = float(t.item())
    engine = s.uses_tensor_core()
    s.close()
    return dict(n=n, I=I, t0=t0, tf=tf, ms_per_step=ms_per_step, kern_ms=kern_ms, scratch=sc,
                stats=stats, clocks=clk.summary(), launches=launches, e2e_ms=e2e_t,
                tensor_memory=engine)


def single_chain_roofline(sc, peaks):
    """SURVEY §8(d) byte basis for the dominant kernel of the config-3 step: (4 B x proposals +
    bytes_per_accept(N) x accepted swaps) / kernel time, against one SM's shared-memory bandwidth
    (the chain runs on one SM) at the measured clock.  The scratch phase (k_sa_scratch) is the
    dominant kernel when it ran; its proposals are the iterations it covered."""
    n, I = sc["n"], sc["I"]
    kms = statistics.mean(sc["kern_ms"])
    sc_ms = statistics.mean(x[0] for x in sc["scratch"])
    sc_k = sc["scratch"][-1][1]
    sc_acc = sc["scratch"][-1][2]
    acc = sc["stats"][-1]["accepted"]
    peak, src, mhz = smem_peak(sc["clocks"], peaks)
    bpa = bytes_per_accept(n)
    if sc_ms > 0:
        kname, kt, props, accs = "k_sa_scratch", sc_ms, sc_k, sc_acc
    else:
        kname, kt, props, accs = "k_sa_tc", kms, I, acc
    algo = BYTES_PER_PROPOSAL * props + bpa * accs
    achieved = algo / (kt / 1e3) / 1e9
    prof = profile_summary(kname)
    step_algo = BYTES_PER_PROPOSAL * I + bpa * acc
    out = {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
           "frac": achieved / peak, "traffic": prof.get("dram_bytes_per_launch"),
           "kernel": kname, "kernel_ms": kt, "peak_source": src,
           "algorithmic_bytes_per_launch": algo,
           "bytes_per_proposal": BYTES_PER_PROPOSAL, "bytes_per_accept": bpa,
           "proposals": props, "accepted": accs,
           "share_of_step": kt / sc["ms_per_step"],
           "whole_step": {"achieved": step_algo / (sc["ms_per_step"] / 1e3) / 1e9,
                          "frac": step_algo / (sc["ms_per_step"] / 1e3) / 1e9 / peak},
           "cycles_per_accept": (kt / 1e3) * mhz * 1e6 / max(1, accs),
           "ncu": prof or None}
    if sc_ms > 0:
        d_ms = kms - sc_ms
        d_props, d_acc = I - sc_k, acc - sc_acc
        out["delta_engine"] = {"kernel": "k_sa_tc (+ k_delta_init)", "ms": d_ms, "proposals": d_props,
                               "accepted": d_acc,
                               "proposals_per_s": d_props / (d_ms / 1e3) if d_ms > 0 else None,
                               "frac": (BYTES_PER_PROPOSAL * d_props + bpa * d_acc) / (d_ms / 1e3) / 1e9 / peak
                               if d_ms > 0 else None,
                               "ncu": profile_summary("k_sa_tc") or None}
    return out


def run_ensemble(args, Q, pg, ws, rank, local, stream, timed_steps, warmup):
    """BASELINE config 5: 8192 chains x 1e7 iterations split over ranks + NCCL min-reduce, through
    the product's distributed driver; start permutations generated on the device (R14b)."""
    import torch
    from paper_1208_2675_b200.dist import chain_range, ensemble_distributed
    A, B, _, cfg = config(5)
    C, I = args.ens_chains, args.ens_iters
    n = cfg["n"]
    s = Q.Solver(A, B, np.arange(n, dtype=np.int32), device=local, stream=stream.cuda_stream)
    p00 = s.start_perms(SA_SEED, 0, 1)[0]             # chain 0's start permutation (R19)
    s.reset(p00)
    s.delta_init()
    t0, tf = s.schedule_bounds()
    sch = Q.make_schedule(Q.QAP_COOL_GEOMETRIC, t0, tf, I)
    begin, end = chain_range(rank, ws, C)
    kern = {}

    def runner(A_, B_, b, p0s, iters, schedule, seed, count):
        res = s.ensemble(b, p0s, iters, schedule, seed, count=count)
        kern["ms"], kern["launches"] = s.last_kernel_time()
        return res

    def one():
        return ensemble_distributed(A, B, C, I, sch, SA_SEED, p0_fn=None, local_runner=runner)

    for _ in range(warmup):
        one()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(timed_steps)]
    kms, res = [], None
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(timed_steps):
            flush.zero_()
            ev[i][0].record(stream)
            res = one()
            ev[i][1].record(stream)
            kms.append(kern.get("ms", 0.0))
        torch.cuda.synchronize()
    if pg:
        pg.barrier()
    step_ms = sum(a.elapsed_time(b) for a, b in ev) / timed_steps
    kmean = statistics.mean(kms)
    tt = torch.tensor([step_ms, kmean], device="cuda", dtype=torch.float64)
    if pg:
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
    step_ms, kmean = float(tt[0]), float(tt[1])
    # e2e through the public API with host buffers: qap_create (A, B, p0 copied in), the ensemble
    # (start permutations generated on the device), best permutation and statistics read back
    torch.cuda.synchronize()
    t = time.perf_counter()
    with Q.Solver(A, B, p00, device=local, stream=stream.cuda_stream) as s2:
        s2.ensemble(begin, None, I, sch, SA_SEED, count=end - begin)
    e2e_ms = 1e3 * (time.perf_counter() - t)
    te = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
    if pg:
        pg.all_reduce(te, op=pg.ReduceOp.MAX)
    e2e_ms = float(te.item())
    s.close()
    return dict(C=C, I=I, n=n, t0=t0, tf=tf, step_ms=step_ms, kern_ms=kmean, res=res,
                clocks=clk.summary(), launches=kern.get("launches", 0) * timed_steps,
                e2e_ms=e2e_ms, local_chains=end - begin,
                tensor_memory=True)


def ensemble_roofline(e, peaks, sms):
    """SURVEY §8(d) byte basis over all SMs of one GPU: (4 B x chain-iterations + bytes_per_accept
    x accepted swaps) / kernel time / (SMs x 128 B/clk x measured clock); the HBM traffic the
    north_star asks for comes from ncu (expected << 1% of the HBM peak)."""
    res = e["res"]
    ws = max(1, e.get("ws", 1))
    props = e["C"] * e["I"]
    algo = BYTES_PER_PROPOSAL * props + bytes_per_accept(e["n"]) * res.accepted
    peak, src, _ = smem_peak(e["clocks"], peaks, sms=sms * ws)
    achieved = algo / (e["kern_ms"] / 1e3) / 1e9
    prof = profile_summary("k_ens_scratch")
    hbm = None
    if prof.get("dram_bytes_per_launch"):
        gbs = prof["dram_bytes_per_launch"] / (prof["time_ms"] / 1e3) / 1e9 if prof.get("time_ms") else None
        hbm = {"dram_gbs": gbs, "peak_gbs": peaks.get("hbm_gbs", 6538.6),
               "frac": gbs / peaks.get("hbm_gbs", 6538.6) if gbs else None,
               "source": prof.get("capture")}
    return {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": prof.get("dram_bytes_per_launch"),
            "kernel": "k_ens_scratch + k_sa_tc (ensemble launches)", "kernel_ms": e["kern_ms"],
            "peak_source": src, "algorithmic_bytes_per_launch": algo,
            "accepted": res.accepted, "chain_iterations": props, "hbm": hbm, "ncu": prof or None}


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    pg = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    from paper_1208_2675_b200 import qapsa as Q
    stream = torch.cuda.current_stream()
    peaks = measured_peaks()
    sms = torch.cuda.get_device_properties(local).multi_processor_count

    sc = None
    if ws == 1 or not args.no_single:
        sc = single_chain(args, Q, local, stream, pg, ws)
    ens = None
    if ws > 1 or not args.no_ensemble:
        ens = run_ensemble(args, Q, pg, ws, rank, local, stream,
                           timed_steps=args.steps if ws > 1 else args.ens_steps,
                           warmup=args.warmup if ws > 1 else 1)
        ens["ws"] = ws
    cfg4 = None
    if rank == 0 and ws == 1 and not args.no_config4:
        cfg4 = run_config4(args, Q)
    cpu = cpu_ens = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_sample)
        if ens is not None:
            cpu_ens = cpu_baseline_ensemble(args.cpu_ens_chains)

    if rank == 0:
        sc_obj = None
        if sc is not None:
            I, n = sc["I"], sc["n"]
            acc = sc["stats"][-1]["accepted"]
            sc_obj = {
                "metric": METRIC_1, "value": ws * I * 1e3 / sc["ms_per_step"], "unit": UNIT_1,
                "ms_per_step": sc["ms_per_step"],
                "value_without_init": I * 1e3 / statistics.mean(sc["kern_ms"]),
                "engine": ("tensor-memory: scratch phase (k_sa_scratch) then Δ (k_sa_tc)"
                           if sc["tensor_memory"] else "shared-memory (k_sa_chain)"),
                "config": {"workload": "config3 tai100a-shaped N=100, 1 chain, 1e8 iterations"
                                       + (" (one replica per rank)" if ws > 1 else ""),
                           "n": n, "iters_per_step": I,
                           "schedule": {"kind": "geometric", "t0": sc["t0"], "tf": sc["tf"]},
                           "l2": "flushed between timed steps (256 MiB write)"},
                "clocks": sc["clocks"], "gpu_launches": sc["launches"],
                "roofline": single_chain_roofline(sc, peaks),
                "e2e": {"value": ws * I / (sc["e2e_ms"] / 1e3), "unit": UNIT_1,
                        "h2d_bytes_per_step": 2 * n * n * 4 + 4 * n,
                        "d2h_bytes_per_step": 2 * 4 * n + 2 * 48},
                "acceptance_rate": acc / I, "accepted": acc, "best_cost": sc["stats"][-1]["best_cost"],
                "digest": str(sc["stats"][-1]["digest"]), "cpu_baseline": cpu,
            }
        ens_obj = None
        if ens is not None:
            res, C, I, n = ens["res"], ens["C"], ens["I"], ens["n"]
            ens_obj = {
                "metric": METRIC_N, "value": C * I * 1e3 / ens["step_ms"], "unit": UNIT_N,
                "ms_per_step": ens["step_ms"], "kernel_ms": ens["kern_ms"],
                "value_kernel_only": C * I * 1e3 / ens["kern_ms"],
                "engine": "tensor-memory: k_start_perms, k_reset, k_ens_scratch (4 chains per SM), k_delta_init, k_sa_tc "
                          "over all chains, then k_ens_collect + k_ens_reduce and the NCCL min-reduce",
                "config": {"workload": "config5 ensemble: 8192 chains x N=100 tai100a-shaped x 1e7 iterations",
                           "chains": C, "iters_per_chain": I, "n": n,
                           "chains_per_rank": ens["local_chains"],
                           "start_perms": "chain-keyed Fisher-Yates on the device (R14b)",
                           "schedule": {"kind": "geometric", "t0": ens["t0"], "tf": ens["tf"]},
                           "l2": "flushed between timed steps (256 MiB write)",
                           "parallelism": f"chains split over {ws} rank(s), NCCL min-reduce"},
                "clocks": ens["clocks"], "gpu_launches": ens["launches"],
                "roofline": ensemble_roofline(ens, peaks, sms),
                "e2e": {"value": C * I / (ens["e2e_ms"] / 1e3), "unit": UNIT_N,
                        "h2d_bytes_per_step": 2 * n * n * 4 + 4 * n,
                        "d2h_bytes_per_step": 4 * n + 48 + 64},
                "best_cost": res.best_cost, "best_chain": res.best_chain, "accepted": res.accepted,
                "near_ties": res.near_ties, "cpu_baseline": cpu_ens,
            }
        if ws == 1:
            line = dict(sc_obj)
            line.update({"n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                         "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                         "dtype": "int32+f64",
                         "data": "synthetic (seeded tai100a-shaped instance, BASELINE config 3)"})
            line["config"] = dict(line["config"], parallelism="replicas1")
            if ens_obj is not None:
                line["ensemble"] = ens_obj
        else:
            line = dict(ens_obj)
            line.update({"n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                         "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                         "dtype": "int32+f64",
                         "data": "synthetic (seeded tai100a-shaped instance, BASELINE config 5)"})
            if sc_obj is not None:
                line["single_chain"] = sc_obj
        if cfg4 is not None:
            line["config4_prefix"] = cfg4
        line = {k: line[k] for k in ["metric", "value", "unit", "n_gpus", "steps", "warmup",
                                     "ms_per_step", "higher_is_better", "scaling", "vs_baseline",
                                     "dtype", "data", "config"] if k in line} | line
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    return 0


def run_config4(args, Q):
    """BASELINE config 4 (N=256 grey density, 16-bit B, 1e9-iteration schedule): device time of
    its first args.cfg4_iters iterations on the relabel engine (rank 0, one call, after one
    warm-up call on a separate context).  A prefix, not the whole run: the schedule's hot start."""
    A, B, p0, cfg = config(4)
    I = args.cfg4_iters
    for rep in range(2):
        s4 = Q.Solver(A, B, p0)
        s4.delta_init()
        t0, tf = s4.schedule_bounds()
        sch = Q.make_schedule(Q.QAP_COOL_GEOMETRIC, t0, tf, cfg["iters"])
        g = s4.run(0, I if rep else min(I, 10**5), sch, SA_SEED)
        ms, launches = s4.last_kernel_time()
        eng = s4.engine()
        s4.close()
    return {"workload": "config4 tai256c-shaped N=256 (uint16 B), iterations [0, %d) of 1e9" % I,
            "metric": "SA iterations/s (1 chain, N=256)", "unit": "iterations/s",
            "value": I / (ms / 1e3), "kernel_ms": ms,
            "engine": {Q.QAP_ENGINE_RELABEL: "relabel (k_sa_relabel)",
                       Q.QAP_ENGINE_SHARED_MEMORY: "shared-memory (k_sa_chain)"}.get(eng, str(eng)),
            "accepted": g["accepted"], "cost": g["cost"], "gpu_launches": launches}


# ----------------------------------------------------------- dry run ---
def run_sweep(args):
    """Fig. 2 of the paper (Eq.(4)): for a BASELINE instance and I = 1e4 ... Imax, one
    chain with an I-iteration schedule on the GPU (device time of the call, through the C-ABI) and
    the non-parallel Delta-matrix SA of the paper's ref. [17] -- the oracle in DELTA mode, one host
    core (the cpu_baseline role) -- on the same I; P = t_non-parallel / t_parallel.  Both sides
    must end with the same best cost (bit-exact trajectories).  One JSON line."""
    import torch
    import oracle as O
    from paper_1208_2675_b200 import qapsa as Q
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    A, B, p0, cfg = config(args.sweep)
    rows = []
    I = 10**4
    while I <= args.sweep_imax:
        with Q.Solver(A, B, p0) as s:
            s.delta_init()
            t0, tf = s.schedule_bounds()
            s.run(0, min(I, 10**4), Q.make_schedule(Q.QAP_COOL_GEOMETRIC, t0, tf, I), SA_SEED)   # warm-up
        with Q.Solver(A, B, p0) as s:
            s.delta_init()
            t0, tf = s.schedule_bounds()
            g = s.run(0, I, Q.make_schedule(Q.QAP_COOL_GEOMETRIC, t0, tf, I), SA_SEED)
            ms, _ = s.last_kernel_time()
            eng = s.engine()
        sch = O.geometric_schedule_for(A, B, p0, I)
        run = O.Run(A, B, p0, mode=O.MODE_DELTA)
        t = time.perf_counter()
        st = run.run(0, I, sch, SA_SEED)
        t_np = time.perf_counter() - t
        row = {"I": I, "t_parallel_s": ms / 1e3, "t_non_parallel_s": t_np, "P": t_np / (ms / 1e3),
               "accepted": g["accepted"], "best_cost": g["best_cost"],
               "oracle_best_cost": int(st["best_cost"]), "engine": eng}
        if row["best_cost"] != row["oracle_best_cost"]:
            raise SystemExit(f"sweep: best cost differs from the oracle at I = {I}")
        rows.append(row)
        log(json.dumps(row))
        I *= 10
    host = host_info()
    print(json.dumps({"sweep": "Fig. 2 / Eq.(4): P = t_non-parallel / t_parallel against I",
                      "config": args.sweep, "instance": cfg["name"], "seed": SA_SEED,
                      "non_parallel": "oracle DELTA mode (the non-parallel Delta-matrix SA, P:44-50), 1 host core",
                      "parallel": "this library, 1 B200 (device time of the call, threshold precompute included)",
                      "cpu_model": host.get("cpu_model"), "rows": rows}), flush=True)
    return 0


def run_dry(args):
    """Host path only (no GPU, no method arithmetic): rank environment, chain partition, the
    ensemble driver's collectives on gloo with a stub rank runner, and rank 0's JSON line."""
    import torch.distributed as dist
    from paper_1208_2675_b200.dist import chain_range, ensemble_distributed
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    C, n = args.ens_chains, 100
    begin, end = chain_range(rank, ws, C)

    def stub(A_, B_, b, p0s, iters, schedule, seed, count):
        # a placeholder result that depends only on the global chain ids (no SA is run)
        costs = [(c * 7919) % 1000003 for c in range(b, b + count)]
        i = int(np.argmin(costs))
        return dict(best_cost=costs[i], best_chain=b + i, best_perm=np.arange(n, dtype=np.int32),
                    stats=dict(iterations=count * iters, accepted=0, near_ties=0))

    A = np.zeros((n, n), np.int32)
    res = ensemble_distributed(A, A, C, args.ens_iters, None, SA_SEED, p0_fn=None, local_runner=stub,
                               device="cpu")
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": ws, "chains": C, "rank0_chains": [begin, end],
                          "best_cost": res.best_cost, "best_chain": res.best_chain,
                          "iterations": res.iterations}), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dry-run", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3, help="end-to-end steps (median reported)")
    ap.add_argument("--no-ensemble", action="store_true")
    ap.add_argument("--no-single", action="store_true", help="N > 1: skip the nested single chain")
    ap.add_argument("--ens-chains", type=int, default=8192)
    ap.add_argument("--ens-iters", type=int, default=10**7)
    ap.add_argument("--ens-steps", type=int, default=2, help="N = 1: timed ensemble runs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config4", action="store_true")
    ap.add_argument("--cfg4-iters", type=int, default=10**7)
    ap.add_argument("--cpu-sample", type=int, default=3 * 10**7)
    ap.add_argument("--cpu-ens-chains", type=int, default=16)
    ap.add_argument("--ref-sample", type=int, default=10**7)
    ap.add_argument("--ref-chains", type=int, default=8)
    ap.add_argument("--sweep", type=int, default=0, help="Fig. 2 sweep (Eq.(4)) on this BASELINE config")
    ap.add_argument("--sweep-imax", type=int, default=10**8)
    args = ap.parse_args()
    if args.sweep:
        return run_sweep(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args, sys.argv[1:])
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
