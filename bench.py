#!/usr/bin/env python3
"""bench.py -- FP64 POBTAF + POBTASI (Serinv, arXiv 2503.17528) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference|library]

One step = one pass of the whole hot path: POBTAF followed
by POBTASI of a synthetic SPD BTA matrix (generator G1, seed 0) -- the fused
`serinv_selinv` task graph at N = 1, the distributed PPOBTAF -> all-gather ->
PPOBTASI at N > 1 (weak scaling: every rank owns the configured n blocks).
Metric (BASELINE.json): FP64 TFLOP/s of POBTAF + POBTASI, algorithmic flop count
(LAPACK conventions, sequential count for distributed runs),
device-timed with CUDA events; fraction of the measured FP64 DMMA peak.

--impl reference times the CPU oracle (oracle/, numpy/scipy FP64) on a bounded
sample of the same workload (the paper's code does not exist).
--impl library times the paper's own GPU design on the same B200 and input: one
cuSOLVER / cuBLAS call per block operation (tools/library_arm.py);
a bench-only comparator, N = 1.
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

CONFIGS = {  # BASELINE.json configs
    "C1": dict(n=8, b=4, a=2),
    "C2": dict(n=128, b=1024, a=64),
    "C3": dict(n=365, b=2048, a=4),
    "C4": dict(n=256, b=512, a=16),
    "C5": dict(n=16384, b=64, a=8),
}
METRIC = "FP64 seconds & TFLOP/s for POBTAF+POBTASI (1/2/4/8 B200), fraction of FP64 peak"
FP64_PEAK_TFLOPS = 37.1   # measured DMMA peak, profiles/fp64_peaks_r01.json
L2_BYTES = 126 * 2 ** 20


def flops_pobtaf(n, b, a):
    return (n - 1) * (7 / 3 * b ** 3 + 3 * a * b * b + a * a * b) + b ** 3 / 3 + a * b * b + a * a * b + a ** 3 / 3


def flops_pobtasi(n, b, a):
    return ((n - 1) * (14 / 3 * b ** 3 + 6 * a * b * b + 2 * a * a * b)
            + 2 * b ** 3 / 3 + 2 * a * b * b + 2 * a * a * b + 2 * a ** 3 / 3)


def src_sha() -> str:
    """sha256 (16 hex) of the library sources (csrc/ + include/serinv.h): the build a
    committed ncu capture was taken of."""
    import hashlib
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2503_17528_b200", "csrc")
    for f in sorted(os.listdir(csrc)) + ["../../../include/serinv.h"]:
        p = os.path.normpath(os.path.join(csrc, f))
        if os.path.isfile(p):
            h.update(os.path.basename(p).encode())
            with open(p, "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()[:16]


def ncu_traffic(config, engine="exec"):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the executor from a committed
    ncu --set full capture of this config (profiles/r*/ncu_<C>/summary.json) whose src_sha
    matches the library sources being timed; else (None, reason)."""
    import glob
    sha = src_sha()
    seen = []
    sub = f"ncu_{config}" if engine == "exec" else f"ncu_{config}_{engine}"
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", sub, "summary.json")), reverse=True):
        try:
            with open(p) as f:
                d = json.load(f)
        except (OSError, ValueError):
            continue
        seen.append(os.path.relpath(p, ROOT))
        if d.get("src_sha") == sha and "dram_bytes_per_launch" in d:
            return d["dram_bytes_per_launch"], os.path.relpath(p, ROOT)
    return None, (f"no ncu capture of src_sha {sha} (stale: {', '.join(seen)})" if seen else "no ncu capture")


def bench_config(name, cfg):
    """The workload both arms report (per GPU for N > 1: weak scaling)."""
    n, b, a = cfg["n"], cfg["b"], cfg["a"]
    return {"workload": f"{name} n={n} b={b} a={a} per GPU", "n": n, "b": b, "a": a, "generator": "g1 seed 0",
            "l2": (f"inputs {bta_bytes(n, b, a) / 1e9:.2f} GB per GPU > 126 MB L2 (no flush needed)"
                   if bta_bytes(n, b, a) > L2_BYTES else "inputs fit in L2 (parity-size case)")}


def algorithmic_bytes(n, b, a):
    """read + write of the whole BTA per phase (2 * 8 * (n(2b^2 + ab) - b^2 + a^2)),
    F + SI = 2 phases."""
    return 2 * 2 * 8 * (n * (2 * b * b + a * b) - b * b + a * a)


HBM_PEAK_GBS = 6549.1     # MEASURED_PEAKS.json hbm_gbs (copy bandwidth on this pool's B200s)


def bta_bytes(n, b, a):
    return 8 * (n * b * b + (n - 1) * b * b + n * a * b + a * a)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS),
                    help="BASELINE.json config; default C3 = the north-star climate shape")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference", "library"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="use the distributed path (NCCL process group, serinv_ppobtaf_q / _q) even at N = 1 "
                         "(exercises the N > 1 code path on a one-GPU box)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-phases", action="store_true",
                    help="skip the standalone serinv_pobtaf / serinv_pobtasi phase timings")
    ap.add_argument("--r", default="auto",
                    help="N > 1: blocks of the first / last rank relative to a middle rank (serinv_plan_ends); "
                         "'auto' = distributed.auto_r(b)")
    ap.add_argument("--q", default="auto",
                    help="N > 1: sub-partitions per rank (serinv_ppobtaf_q); 'auto' = serinv_dist_auto_q")
    ap.add_argument("--engine", default="auto", choices=["auto", "exec", "sb"],
                    help="N = 1: 'sb' = the small-block engine (serinv_sb_selinv, b <= 64, a <= 16), "
                         "'exec' = the tile-task executor; 'auto' = sb where it applies")
    ap.add_argument("--partitions", default="auto",
                    help="N = 1: intra-GPU partitions, e.g. 1 (sequential), 8, 256x16 (nested); "
                         "'auto' = the library's plan (serinv_auto_partitions)")
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled every ~5 ms DURING the timed region
    (NVML; nvidia-smi as a fallback)."""
    NVML_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                 "hw_thermal_slowdown": 0x40}
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []      # (sm_mhz, sm_max_mhz, {reasons})
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except AttributeError:  # older binding name
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        return float(sm), float(mx), {k for k, v in self.NVML_BITS.items() if bits & v}

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        f = [x.strip() for x in out.split(",")]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        return float(f[0]), float(f[1]), {names[k] for k in range(4) if f[2 + k].lower().startswith("active")}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample_nvml() if self._nvml else self._sample_smi())
            except Exception:
                pass
            self._stop.wait(0.005 if self._nvml else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*(s[2] for s in self.samples))),
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


# --------------------------------------------------------------------------- statistics
def median_ci95(xs):
    """Median and a distribution-free 95 % confidence interval of the median (order
    statistics of Binomial(n, 1/2); PAPER.md P:717 reports median + 95 % CI)."""
    from math import comb
    v = sorted(xs)
    n = len(v)
    med = statistics.median(v)
    if n < 6:
        return med, v[0], v[-1]
    cdf = [sum(comb(n, i) for i in range(k + 1)) / 2 ** n for k in range(n + 1)]
    # [v[i], v[n-1-i]] covers the median with probability 1 - 2 P(B <= i), B ~ Bin(n, 1/2):
    # the largest i with P(B <= i) <= 0.025
    i = max([k for k in range(n // 2) if cdf[k] <= 0.025] or [0])
    return med, v[i], v[n - 1 - i]


def stats_line(times_s, flops):
    med, lo, hi = median_ci95(times_s)
    return {"seconds_median": round(med, 6), "seconds_ci95": [round(lo, 6), round(hi, 6)],
            "seconds_mean": round(statistics.mean(times_s), 6), "samples": len(times_s),
            "tflops_median": round(flops / med / 1e12, 4),
            "tflops_ci95": [round(flops / hi / 1e12, 4), round(flops / lo / 1e12, 4)]}


# --------------------------------------------------------------------------- CPU oracle
def cpu_oracle_sample(cfg, budget_s):
    """n' for a bounded oracle sample: the largest power of two (>= 2, <= n) whose
    oracle selinv is predicted to take about budget_s (per-block cost is constant)."""
    import btagen
    from oracle import sequential as seq
    n, b, a = cfg["n"], cfg["b"], cfg["a"]
    nprime = 2
    t0 = time.perf_counter()
    seq.selinv(btagen.g1(0, nprime, b, a))
    dt = time.perf_counter() - t0
    while nprime * 2 <= n and dt * 2 <= budget_s:
        nprime *= 2
        dt *= 2
    return nprime


def cpu_oracle_run(cfg, nprime):
    """One oracle selinv (POBTAF + POBTASI, numpy/scipy FP64, as it stands) on the first
    n' blocks of the configured (b, a); returns seconds."""
    import btagen
    from oracle import sequential as seq
    A = btagen.g1(0, nprime, cfg["b"], cfg["a"])
    t0 = time.perf_counter()
    seq.selinv(A)
    return time.perf_counter() - t0


def cpu_oracle_rate(cfg, budget_s=20.0):
    """Time the oracle (as it stands) on a bounded sample.  Returns (TFLOP/s, seconds, n', cores)."""
    b, a = cfg["b"], cfg["a"]
    cores = len(os.sched_getaffinity(0))
    nprime = cpu_oracle_sample(cfg, budget_s)
    dt = cpu_oracle_run(cfg, nprime)
    fl = flops_pobtaf(nprime, b, a) + flops_pobtasi(nprime, b, a)
    return fl / dt / 1e12, dt, nprime, cores


def reference_arm(args, cfg):
    """The reference arm is the CPU oracle (there is no reference code, only PAPER.md):
    each step = one oracle selinv on a bounded sample of the workload (n' blocks, about
    3 s), so --steps K --warmup W ends within a few minutes.  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n, b, a = cfg["n"], cfg["b"], cfg["a"]
    cores = len(os.sched_getaffinity(0))
    nprime = cpu_oracle_sample(cfg, budget_s=3.0)
    times = []
    for it in range(args.warmup + args.steps):
        dt = cpu_oracle_run(cfg, nprime)
        if it >= args.warmup:
            times.append(dt)
    fl = flops_pobtaf(nprime, b, a) + flops_pobtasi(nprime, b, a)
    med, lo, hi = median_ci95(times)
    value = fl / med / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(med * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.config, cfg),
        "stats": stats_line(times, fl),
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": f"oracle selinv (numpy/scipy FP64) on n'={nprime} of the {n} blocks, same b, a; "
                                   f"TFLOP/s of that sample"},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def library_arm(args, cfg):
    """The paper's per-block cuSOLVER/cuBLAS design on this B200, same input,
    same timing rules as our arm; reports its max block error against our library."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import torch
    import btagen
    import paper_2503_17528_b200 as sb
    from tools import library_arm as la
    n, b, a = cfg["n"], cfg["b"], cfg["a"]
    torch.cuda.set_device(0)
    fl = flops_pobtaf(n, b, a) + flops_pobtasi(n, b, a)
    pristine = btagen.g1_torch(0, n, b, a, device="cuda:0")
    work = {k: v.clone() for k, v in pristine.items()}

    def restore():
        for k in work:
            work[k].copy_(pristine[k])

    def step():
        ld = la.pobtaf(work)
        la.pobtasi(work)
        return ld

    for _ in range(args.warmup):
        restore()
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    times = []
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            restore()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ld_lib = step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    sec = statistics.median(times)
    # agreement with our library on the same input (relative Frobenius, per sampled block)
    ours = {k: v.clone() for k, v in pristine.items()}
    ld_ours = sb.selinv(ours["diag"], ours["lower"], ours["arrow"], ours["tip"])
    errs = []
    for k, idx in (("diag", [0, n // 2, n - 1]), ("lower", [0, (n - 1) // 2, n - 2]), ("arrow", [0, n - 1]),
                   ("tip", [None])):
        for i in idx:
            if (k == "lower" and n < 2) or (k in ("arrow", "tip") and a == 0):
                continue
            x, y = (work[k], ours[k]) if i is None else (work[k][i], ours[k][i])
            errs.append(float(torch.linalg.norm(x - y) / torch.linalg.norm(y)))
    line = {
        "impl": "library", "metric": METRIC, "value": round(fl / sec / 1e12, 4), "unit": "TFLOP/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.config, cfg),
        "design": "per-block cusolverDnDpotrf / cublasDtrsm / cublasDgemm via torch.linalg (paper P:646-650)",
        "fraction_of_fp64_peak": round(fl / sec / 1e12 / FP64_PEAK_TFLOPS, 4),
        "max_rel_block_err_vs_ours": max(errs), "logdet_diff_vs_ours": abs(float(ld_lib) - float(ld_ours)),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm
def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg)
    if args.impl == "library":
        return library_arm(args, cfg)
    import torch
    import torch.distributed as dist
    import btagen
    import paper_2503_17528_b200 as sb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch N > 1 with "
                         f"`python -m torch.distributed.run --nproc-per-node {args.gpus} bench.py --gpus {args.gpus}`")
    N = world
    torch.cuda.set_device(local)
    dpath = world > 1 or args.dist   # distributed path (one process per GPU)
    if dpath:
        if "RANK" not in os.environ:  # --dist at world size 1 without torchrun
            os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=os.environ.get("MASTER_PORT", "29533"))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n_loc, b, a = cfg["n"], cfg["b"], cfg["a"]
    n = n_loc * world
    fl_f, fl_si = flops_pobtaf(n, b, a), flops_pobtasi(n, b, a)
    fl = fl_f + fl_si
    h = sb.default_handle(local)
    stream = torch.cuda.current_stream()

    def barrier():
        if dpath:
            dist.barrier()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def max_over_ranks(rows):
        """rows: per-step lists of seconds on this rank -> per-step max over ranks."""
        t = torch.tensor(rows, dtype=torch.float64, device="cuda")
        if dpath:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.cpu().tolist()

    # ---- inputs resident in HBM (pristine copy restored between steps, untimed); the
    # generator's torch twin builds G1 directly in HBM, bit-identical to btagen.g1
    Ps = [1]
    use_sb = (not dpath and (args.engine == "sb" or (args.engine == "auto" and b <= 64 and a <= 16)))
    if not dpath:
        if use_sb:
            Ps = (sb.sb_auto_plan(n, b, a) if args.partitions == "auto"
                  else [int(x) for x in args.partitions.split("x") if int(x) > 1])
        else:
            Ps = (sb.auto_partitions(n, b) if args.partitions == "auto"
                  else [int(x) for x in args.partitions.split("x")])
        pristine = btagen.g1_torch(0, n, b, a, device=f"cuda:{local}")
        work = {k: v.clone() for k, v in pristine.items()}
        W = (work["diag"], work["lower"], work["arrow"], work["tip"])

        def step():
            if use_sb:
                return sb.selinv_sb(*W, Ps, handle=h, check=False)
            if Ps == [1]:
                return sb.selinv(*W, handle=h, check=False)
            return sb.pselinv(*W, Ps, handle=h, check=False)
    else:
        from paper_2503_17528_b200 import distributed as sd
        # twisted scheme (reading R14): first and last rank are fill-in free, so they
        # take r x a middle rank's blocks (flop/chain balance)
        r_end = sd.auto_r(b) if args.r == "auto" else float(args.r)
        parts = sb.plan_ends(n, world, r_end)
        s, e = parts[rank]
        # sub-partitions per rank (intra-GPU partitioning of each rank's chain), the
        # same on every rank: the library's default for the smallest rank
        Q = (sd.dist_auto_q(min(e_ - s_ for s_, e_ in parts), b) if args.q == "auto" else int(args.q))
        pristine = btagen.g1_torch(0, n, b, a, device=f"cuda:{local}", start=s, end=e)
        if pristine["lower"].shape[0] == 0:
            pristine["lower"] = torch.zeros((1, b, b), dtype=torch.float64, device=f"cuda:{local}")
        work = {k: v.clone() for k, v in pristine.items()}
        # the library's own NCCL communicator carries the exchange (serinv_ppobtaf / serinv_ppobtasi)
        comm = sd.Comm(world, rank, local)
        ctx = sd.DistContext(h, world, rank, n, s, e - s, b, a, device=local, Q=Q, comm=comm)

        def step():
            return sd.pselinv_step(ctx, work, check=False)

    def restore():
        for k in work:
            work[k].copy_(pristine[k])

    # ---- warmup
    for _ in range(args.warmup):
        restore()
        step()
    torch.cuda.synchronize()
    info, logdet = (h.scalars() if not dpath else (ctx.info, ctx.logdet))
    if int(info.item()) != 0:
        raise SystemExit(f"factorisation failed: info={int(info.item())}")
    logdet_ref = float(logdet.item())

    # ---- timed steps (device events on the library stream; per step max over ranks)
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            restore()
            barrier()
            torch.cuda.synchronize()
            e0 = ev()
            step()
            e1 = ev()
            torch.cuda.synchronize()
            barrier()
            times.append(e0.elapsed_time(e1) / 1e3)
    launches = h.last_launches() * (1 if not dpath else 2)  # distributed: ppobtaf + ppobtasi
    times = [r[0] for r in max_over_ranks([[t] for t in times])]
    st = stats_line(times, fl)
    sec_per_step = st["seconds_median"]
    value = fl / sec_per_step / 1e12

    step_name = ("serinv_sb_selinv" if use_sb else "serinv_selinv" if Ps == [1] else "serinv_pselinv_nested")
    # ---- phases: factorisation and selected inversion timed as separate launches
    phases = None
    if not args.no_phases and not dpath:
        # the literal C-ABI path: serinv_pobtaf (Alg. 1, one-sided order, L is part of
        # the contract) then serinv_pobtasi (Alg. 2) on its output, one launch each
        tf, ts = [], []
        for it in range(args.warmup + args.steps):
            restore()
            torch.cuda.synchronize()
            e0 = ev()
            sb.pobtaf(*W, handle=h, check=False)
            e1 = ev()
            sb.pobtasi(*W, handle=h, check=False)
            e2 = ev()
            torch.cuda.synchronize()
            if it >= args.warmup:
                tf.append(e0.elapsed_time(e1) / 1e3)
                ts.append(e1.elapsed_time(e2) / 1e3)
        if int(info.item()) != 0:
            raise SystemExit(f"serinv_pobtasi failed: info={int(info.item())}")
        phases = {"pobtaf": stats_line(tf, fl_f), "pobtasi": stats_line(ts, fl_si),
                  "pobtaf_plus_pobtasi": stats_line([x + y for x, y in zip(tf, ts)], fl),
                  "fused_selinv": {"seconds_median": st["seconds_median"], "tflops_median": st["tflops_median"],
                                   "step": step_name},
                  "note": "pobtaf / pobtasi: standalone serinv_pobtaf and serinv_pobtasi launches (Alg. 1 and "
                          "Alg. 2 order); the headline value is the fused one-launch step"}
    elif not args.no_phases and dpath:
        # phase split through the transport-agnostic pair (serinv_ppobtaf_q, torch.distributed
        # NCCL all-gather, serinv_ppobtasi_q): same kernels and records, events between the phases
        ctx_p = sd.DistContext(h, world, rank, n, s, e - s, b, a, device=local, Q=Q)
        rows = []
        for it in range(args.warmup + args.steps):
            restore()
            barrier()
            torch.cuda.synchronize()
            e0 = ev()
            sd.ppobtaf(ctx_p, work)
            e1 = ev()
            sd.exchange(ctx_p.send, ctx_p.recv, ctx_p.group)
            e2 = ev()
            sd.ppobtasi(ctx_p, work)
            e3 = ev()
            torch.cuda.synchronize()
            if it >= args.warmup:
                rows.append([e0.elapsed_time(e1) / 1e3, e1.elapsed_time(e2) / 1e3, e2.elapsed_time(e3) / 1e3])
        rows = max_over_ranks(rows)
        phases = {"ppobtaf": stats_line([r[0] for r in rows], fl_f),
                  "exchange": stats_line([r[1] for r in rows], 1.0),
                  "ppobtasi": stats_line([r[2] for r in rows], fl_si),
                  "note": "per phase max over ranks; the exchange line's tflops fields are meaningless; "
                          "ppobtasi includes the redundant reduced solve (POBTARSSI)"}
        del phases["exchange"]["tflops_median"], phases["exchange"]["tflops_ci95"]
        del ctx_p
        torch.cuda.empty_cache()

    # ---- end to end through the public API with host buffers (pinned H2D, D2H of X + logdet)
    e2e = None
    if not args.no_e2e:
        pinned = {k: v.cpu().pin_memory() for k, v in pristine.items()}
        out = {k: torch.empty_like(v).pin_memory() for k, v in pinned.items()}
        ld_host = torch.empty(1, dtype=torch.float64).pin_memory()
        h2d = sum(v.numel() * 8 for v in pinned.values())
        et = []
        for it in range(args.warmup + args.steps):
            barrier()
            torch.cuda.synchronize()
            e0 = ev()
            if not dpath and Ps == [1] and not use_sb:
                # public API with host buffers: H2D / D2H stream with the computation
                sb.selinv_host(pinned, work, out, handle=h, check=False)
            else:  # partitioned / distributed: H2D, the step, D2H on the stream
                for k in work:
                    work[k].copy_(pinned[k], non_blocking=True)
                step()
                for k in work:
                    out[k].copy_(work[k], non_blocking=True)
            ld_host.copy_(logdet, non_blocking=True)
            e1 = ev()
            torch.cuda.synchronize()
            if it >= args.warmup:
                et.append(e0.elapsed_time(e1) / 1e3)
        et = [r[0] for r in max_over_ranks([[t] for t in et])]
        tb = torch.tensor([float(h2d)], dtype=torch.float64, device="cuda")
        if dpath:
            dist.all_reduce(tb, op=dist.ReduceOp.SUM)
        h2d_all = int(tb.item())
        em = statistics.median(et)
        if abs(float(ld_host.item()) - logdet_ref) > 1e-9 * abs(logdet_ref):
            raise SystemExit(f"e2e log det {float(ld_host.item())} != device-path {logdet_ref}")
        e2e = {"value": round(fl / em / 1e12, 4), "unit": "TFLOP/s",
               "h2d_bytes_per_step": h2d_all, "d2h_bytes_per_step": h2d_all + 8 * world,
               "ms_per_step": round(em * 1e3, 3),
               "api": "serinv_selinv_host (streaming H2D/D2H)" if (not dpath and Ps == [1] and not use_sb) else
                      "H2D + step + D2H on the library stream"}

    # ---- CPU baseline (oracle as it stands), rank 0, N = 1 only, bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, dt, nprime, cores = cpu_oracle_rate(cfg, budget_s=20.0)
        cpu = {"value": round(rate, 6), "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
               "sample": f"oracle selinv (numpy/scipy FP64) on n'={nprime} of the {n} blocks (b={b}, a={a}), "
                         f"{dt:.1f} s"}

    if rank == 0:
        traffic, traffic_src = (ncu_traffic(args.config, "sb" if use_sb else "exec") if not dpath
                                else (None, "distributed run"))
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": "TFLOP/s", "n_gpus": N,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec_per_step * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": bench_config(args.config, cfg),
            "plan": {"n_global": n, "end_ratio_r": r_end if dpath else None,
                     "parallelism": f"partitions{world}x{Q}" if dpath else
                     ("small-block engine, partitions per level " + "x".join(map(str, Ps)) if use_sb else
                      "single" if Ps == [1] else "intra-GPU partitions " + "x".join(map(str, Ps))),
                     "step": ("PPOBTAF+POBTARSSI+PPOBTASI, nested, 2 kernels per level (serinv_sb_selinv)"
                              if use_sb else "POBTAF+POBTASI (serinv_selinv)" if Ps == [1] else
                              "PPOBTAF+POBTARSSI+PPOBTASI in one launch (serinv_pselinv_nested)")
                             if not dpath else
                             "serinv_ppobtaf (incl. the library's ncclAllGather) + serinv_ppobtasi"},
            "stats": st,
            "seconds_per_step": round(sec_per_step, 6),
            "tflops_pobtaf_plus_pobtasi": round(value, 4),
            "fraction_of_fp64_peak": round(value / (FP64_PEAK_TFLOPS * N), 4),
            "roofline": {"bound": "tensor", "achieved": round(value / N, 4), "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": round(value / N / FP64_PEAK_TFLOPS, 4),
                         "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": ("sb_factor_kernel + sb_inverse_kernel (all launches of the step, one stream)"
                                    if use_sb else "serinv_exec_kernel (persistent, 1 launch per step)"),
                         "peak_source": "measured DMMA f64 peak, profiles/fp64_peaks_r01.json "
                                        "(MEASURED_PEAKS.json has no FP64 entry)"},
            # small-b evidence: algorithmic HBM bytes per step / step time
            "roofline_hbm": {"bound": "hbm", "achieved": round(algorithmic_bytes(n, b, a) / sec_per_step / 1e9 / N, 2),
                             "peak": HBM_PEAK_GBS, "unit": "GB/s",
                             "frac": round(algorithmic_bytes(n, b, a) / sec_per_step / 1e9 / N / HBM_PEAK_GBS, 4),
                             "bytes_per_step": algorithmic_bytes(n, b, a),
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            "clocks": clk.summary(),
            "gpu_launches": launches * args.steps,
            "logdet": logdet_ref,
        }
        if phases:
            line["phases"] = phases
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dpath:
        comm.close()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
