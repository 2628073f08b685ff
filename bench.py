#!/usr/bin/env python
"""Benchmark of the Δ-matrix SA hot path (arXiv 1208.2675) on B200.

Headline (BASELINE.json metric "SA iterations/s (1 chain, N=100)"): one step =
one whole config-3 job: qap_reset (device-resident p0) + qap_delta_init +
qap_sa_run over I = 1e8 iterations of the N=100 tai100a-shaped instance.
Under torchrun (N>1) every rank runs its own replica of that chain ("replicas
only": a single chain does not shard) -> weak scaling.
The "ensemble" object is BASELINE config 5: 8192 independent N=100 chains x
1e7 iterations split over the ranks, NCCL min-reduce of the best cost and
permutation (strong scaling, fixed total work).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
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

from qap_inputs import SA_SEED, config, start_perms  # noqa: E402

METRIC = "SA iterations/s (1 chain, N=100)"
UNIT = "iterations/s"
SMEM_BYTES_PER_CLK = 128          # per SM, B300_MICROARCH.md "smem crossbar BW 128/N B/cyc/SM"


def bytes_per_accept(n: int, sa: int = 1, sb: int = 1) -> int:
    """Algorithmic on-chip bytes one accepted swap must move:
    disjoint Δ read+write, touching Δ writes, rows A_v/B'_v of every touching v,
    rows r,s, staging writes, B' row/column exchange."""
    disjoint = (n - 2) * (n - 3) // 2
    touching = 2 * n - 3
    return (8 * disjoint + 4 * touching + (n - 2) * n * (sa + sb) + 2 * n * (sa + sb)
            + 4 * n + 4 * n * sb + 4 * n * sb)


BYTES_PER_PROPOSAL = 4            # one int32 Δ read per proposed swap


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


def profile_traffic(which):
    """Per-launch dram bytes of the dominant kernel from the committed ncu summary, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get("sa_tc_dram_bytes_per_launch" if which == "tc" else "sa_chain_dram_bytes_per_launch")
    except Exception:
        return None


# -------------------------------------------------------- distributed ---
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------- reference ---
def run_reference(args):
    """The oracle (oracle/, plain C, as it stands) on the host cores, config-3 samples."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O
    A, B, p0, cfg = config(3)
    I = cfg["iters"]
    sch = O.geometric_schedule_for(A, B, p0, I)
    sample = args.ref_sample
    times = []
    for step in range(args.warmup + args.steps):
        run = O.Run(A, B, p0, mode=O.MODE_SCRATCH)
        t = time.perf_counter()
        run.run(0, sample, sch, SA_SEED)
        dt = time.perf_counter() - t
        if step >= args.warmup:
            times.append(dt)
    ms = 1e3 * statistics.mean(times)
    value = sample / (ms / 1e3)
    desc = (f"oracle SCRATCH-mode sequential SA, iterations [0,{sample}) of config 3's "
            f"1e8-iteration schedule, 1 host thread")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32+f64", "data": "synthetic",
        "config": {"workload": "config3 tai100a-shaped N=100, 1 chain (sampled prefix)",
                   "n": 100, "iters_per_step": sample, "l2": "n/a (host)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(sample):
    import oracle as O
    A, B, p0, cfg = config(3)
    sch = O.geometric_schedule_for(A, B, p0, cfg["iters"])
    run = O.Run(A, B, p0, mode=O.MODE_SCRATCH)
    t = time.perf_counter()
    run.run(0, sample, sch, SA_SEED)
    dt = time.perf_counter() - t
    return {"value": sample / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"oracle SCRATCH mode, iterations [0,{sample}) of config 3's 1e8 schedule "
                      f"({dt:.1f} s, 1 thread)"}


# --------------------------------------------------------------- ours ---
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

    A, B, p0, cfg = config(3)
    n, I = cfg["n"], cfg["iters"]
    stream = torch.cuda.current_stream()
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
    kern_ms, stats = [], []
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
        torch.cuda.synchronize()
    if pg:
        pg.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if pg:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = ws * I * args.steps / (total_ms / 1e3)
    acc = stats[-1]["accepted"]
    clocks = clk.summary()

    # roofline of the dominant kernel.  Tensor-memory engine (k_sa_tc): every
    # accepted swap is two int8 tensor-core MMAs (Δ += L R^T: 128x128x32; [G|H] += 128x256x32), the
    # algorithmic O(N^2) work of the update; peak = one SM's share of the dense int8 tensor peak
    # (the chain runs on one SM).  Shared-memory engine (k_sa_chain): algorithmic on-chip bytes
    # against one SM's shared-memory bandwidth.
    kms = statistics.mean(kern_ms)
    peaks = measured_peaks()
    mhz = peaks.get("sm_max_mhz", 1965.0)
    sms = peaks.get("sm_count", 148)
    if s.uses_tensor_core():
        # dominant kernel: the scratch phase (k_sa_scratch) when it ran, else the Δ engine (k_sa_tc)
        sc_ms, sc_k, sc_acc = s.last_scratch_time()
        bf16 = peaks.get("bf16_tflops")          # burst: the chain kernel is timed on its own
        if bf16:
            chip_i8, src = 2.0 * float(bf16), ("of measured: MEASURED_PEAKS.json bf16_tflops x 2 "
                                               "(int8:bf16 nominal ratio 4.5:2.25)")
        else:
            chip_i8, src = 2.0 * 1590.0, "of fallback: 1.59 PFLOP/s bf16 (B200_PROFILING.md) x 2"
        peak = chip_i8 / sms
        if sc_ms > 0:
            ops_per_accept = 2 * 128 * 256 * 32        # [G|H] += rank-1 (M=128, N=256, K=32)
            algo, kname, kt = sc_acc * ops_per_accept, "k_sa_scratch", sc_ms
        else:
            ops_per_accept = 2 * 128 * (128 + 256) * 32  # Δ (N=128) and [G|H] (N=256), K=32
            algo, kname, kt = acc * ops_per_accept, "k_sa_tc", kms
        achieved = algo / (kt / 1e3) / 1e12
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS (int8)",
                    "frac": achieved / peak, "traffic": profile_traffic("tc"),
                    "kernel": kname, "kernel_ms": kt,
                    "peak_source": f"{src}, one SM of {sms}",
                    "algorithmic_ops_per_launch": algo,
                    "ops_per_accept": ops_per_accept,
                    "share_of_step": kt / ms_per_step,
                    "scratch_phase": {"ms": sc_ms, "k_reached": sc_k, "accepted": sc_acc,
                                      "delta_engine_ms": kms - sc_ms},
                    "note": "latency-bound sequential chain: the tensor work of an accept is ~0.1-0.25 us; "
                            "the rest is the window / stage dependency chain on one SM"}
    else:
        sa = s_ta = 1
        algo_bytes = BYTES_PER_PROPOSAL * I + acc * bytes_per_accept(n, sa, s_ta)
        achieved = algo_bytes / (kms / 1e3) / 1e9
        peak = SMEM_BYTES_PER_CLK * mhz * 1e6 / 1e9   # one SM: the chain runs on one SM
        roofline = {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": profile_traffic("chain"),
                    "kernel": "k_sa_chain", "kernel_ms": kms,
                    "peak_source": f"128 B/clk/SM (B300_MICROARCH.md) x sm_max_mhz {mhz} "
                                   f"(MEASURED_PEAKS.json), one SM",
                    "algorithmic_bytes_per_launch": algo_bytes,
                    "share_of_step": kms / ms_per_step}

    # e2e through the public API with host buffers (create copies A, B, p0; state read back)
    e2e_ms = []
    for i in range(max(1, args.e2e_steps)):
        torch.cuda.synchronize()
        t = time.perf_counter()
        with Q.Solver(A, B, p0, device=local, stream=stream.cuda_stream) as s2:
            s2.delta_init()
            s2.run(0, I, sch, SA_SEED)
            p_out, bp_out, _ = s2.state(want_delta=False)
        e2e_ms.append(1e3 * (time.perf_counter() - t))
    e2e_t = statistics.mean(e2e_ms)
    if pg:
        t = torch.tensor([e2e_t], device="cuda", dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e = {"value": ws * I / (e2e_t / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": 2 * n * n * 4 + 4 * n,
           "d2h_bytes_per_step": 2 * 4 * n + 2 * 48}

    ens = None
    if not args.no_ensemble:
        ens = run_ensemble(args, Q, s, pg, ws, rank, sch_t0tf=(t0, tf))

    cfg4 = None
    if rank == 0 and not args.no_config4:
        cfg4 = run_config4(args, Q)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_sample)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32+f64",
            "data": "synthetic (seeded tai100a-shaped instance, BASELINE config 3)",
            "engine": ("tensor-memory: scratch phase (k_sa_scratch) then Δ (k_sa_tc)" if s.uses_tensor_core()
                       else "shared-memory (k_sa_chain)"),
            "config": {"workload": "config3 tai100a-shaped N=100, 1 chain, 1e8 iterations"
                                   + (" (one replica per rank)" if ws > 1 else ""),
                       "n": n, "iters_per_step": I, "chains_per_rank": 1,
                       "schedule": {"kind": "geometric", "t0": t0, "tf": tf},
                       "l2": "flushed between timed steps (256 MiB write)",
                       "parallelism": f"replicas{ws}"},
            "clocks": clocks,
            "gpu_launches": (2 + s.last_kernel_time()[1]) * args.steps,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "acceptance_rate": acc / I,
            "accepted": acc,
            "best_cost": stats[-1]["best_cost"],
        }
        if ens is not None:
            line["ensemble"] = ens
        if cfg4 is not None:
            line["config4_prefix"] = cfg4
        print(json.dumps(line), flush=True)
    s.close()
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
    out = {}
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


def run_ensemble(args, Q, s, pg, ws, rank, sch_t0tf):
    """BASELINE config 5: 8192 chains x 1e7 iterations split over ranks + NCCL min-reduce,
    through the product's distributed driver (paper_1208_2675_b200.dist)."""
    import torch
    from paper_1208_2675_b200.dist import chain_range, ensemble_distributed
    A, B, _, cfg = config(5)
    C, I = args.ens_chains, args.ens_iters
    n = cfg["n"]
    t0, tf = sch_t0tf
    sch = Q.make_schedule(Q.QAP_COOL_GEOMETRIC, t0, tf, I)
    warm = Q.make_schedule(Q.QAP_COOL_GEOMETRIC, t0, tf, 10**5)
    begin, end = chain_range(rank, ws, C)
    p0_local = start_perms(n, SA_SEED, begin, end - begin)
    for _ in range(args.warmup):
        s.ensemble(begin, p0_local[: min(end - begin, 1024)], 10**5, warm, SA_SEED)
    kern = {}

    def runner(A_, B_, b, p0s, iters, schedule, seed):
        res = s.ensemble(b, p0s, iters, schedule, seed)
        kern["ms"] = s.last_kernel_time()[0]
        return res

    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = ensemble_distributed(A, B, C, I, sch, SA_SEED,
                               p0_fn=lambda b, c: p0_local if b == begin else start_perms(n, SA_SEED, b, c),
                               local_runner=runner)
    torch.cuda.synchronize()
    wall_ms = 1e3 * (time.perf_counter() - t)
    tt = torch.tensor([kern.get("ms", 0.0), wall_ms], device="cuda", dtype=torch.float64)
    if pg:
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
    kms, wall_ms = float(tt[0]), float(tt[1])
    return {"metric": "chain-iterations/s (8192 x N=100 chains)", "unit": "chain-iterations/s",
            "value": C * I / (kms / 1e3), "value_incl_reduce": C * I / (wall_ms / 1e3),
            "kernel_ms": kms, "chains": C, "iters_per_chain": I, "n_gpus": ws,
            "engine": ("tensor-memory: k_sa_scratch + k_delta_init + k_sa_tc over all chains, one SM per chain"
                       if s.uses_tensor_core() else "shared-memory: k_ensemble, several chains per SM"),
            "gpu_launches": s.last_kernel_time()[1],
            "scaling": "strong", "best_cost": res.best_cost, "best_chain": res.best_chain,
            "accepted": res.accepted, "near_ties": res.near_ties,
            "warmup": f"{args.warmup} x (<=1024 chains x 1e5 it)", "timed_runs": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-ensemble", action="store_true")
    ap.add_argument("--ens-chains", type=int, default=8192)
    ap.add_argument("--ens-iters", type=int, default=10**7)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config4", action="store_true")
    ap.add_argument("--cfg4-iters", type=int, default=10**6)
    ap.add_argument("--cpu-sample", type=int, default=3 * 10**7)
    ap.add_argument("--ref-sample", type=int, default=10**7)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
