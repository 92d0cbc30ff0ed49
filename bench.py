"""Benchmark: Vecchia log-likelihood evaluations per second (BASELINE.json).

Workload (BASELINE config 2): n = 1,000,000 uniform locations in [0,1]^2,
m = 60, random ordering (seed 0), Matérn nu = 1.5, sigma^2 = 1,
beta = 0.052537 (vg/kernels.py:118), FP64; observations drawn by the device
Vecchia forward simulation at those parameters.  One "step" =
one full log-likelihood evaluation (all n - m + 1 blocks, fused kernel +
ordered reduction) of the same plan.  Inputs (32 MB points + 240 MB int32
neighbour table + the 18 GB distance cache) exceed the 126 MB L2, so no
explicit flush is needed between steps.  The cpu_baseline leg doubles as
the run's parity check (`parity`: the oracle over the same blocks, the
oracle's neighbour table over the first 200k targets).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU: blocks are sharded in fixed
4096-entry chunks and one NCCL all-reduce per evaluation combines the
partials (strong scaling: the problem size is fixed).

`--impl reference` times the reference algorithm's CPU implementation on the
host cores: the C restatement under oracle/ (the reference itself is Python
and does not travel to the GPU box), on a prefix sample of the same ordered
problem, extrapolated per block (time is linear in n, reference acceptance
criterion C8).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "r01_fp64_peak.jsonl")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def fp64_peak():
    """Builder-measured FP64 peak (DMMA.8x8x4 stream on all 148 SMs; MEASURED_PEAKS.json
    carries no FP64 figure): the best dmma_m8n8k4 line of profiles/r01_fp64_peak.jsonl."""
    best = None
    try:
        with open(FP64_PEAK_FILE) as f:
            for line in f:
                rec = json.loads(line)
                if rec.get("kernel") == "dmma_m8n8k4":
                    best = max(best or 0.0, float(rec["tflops"]))
    except OSError:
        pass
    if best is None:
        return 37.0, "fallback 37.0 TFLOP/s (profiles/r01_fp64_peak.jsonl missing)"
    return best, ("of builder-measured DMMA peak: tools/fp64_peak.cu DMMA.8x8x4 stream, "
                  "148 SMs @1965 MHz (profiles/r01_fp64_peak.jsonl)")


# joint block, fused block kernel, chunk partials (+ the ordered total in its
# last CTA); general nu adds the per-evaluation K_nu table build
KERNELS_PER_EVAL = 3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--m", type=int, default=60)
    ap.add_argument("--nu", type=float, default=1.5)
    ap.add_argument("--beta", type=float, default=0.052537)
    ap.add_argument("--locations", default="uniform", choices=["uniform", "clustered"],
                    help="clustered: config-5 'soil-moisture-shaped' irregular locations")
    ap.add_argument("--ordering", default="random", choices=["random", "maxmin", "morton"],
                    help="maxmin: exact device maxmin ordering (config 5)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--variant", type=int, default=-1,
                    help="kernel variant (-1 auto; see vgp_plan_set_variant in include/vecchia_b200.h)")
    return ap.parse_args()


def synthetic(n, seed=0, kind="uniform"):
    """Locations of the workload (observations come from simulate_vecchia)."""
    rng = np.random.default_rng(seed)
    if kind == "clustered":
        # 200 Gaussian clusters (sd 0.02) holding 80% of the points, 20% uniform
        centers = rng.random((200, 2))
        k = int(0.8 * n)
        locs = np.concatenate([centers[rng.integers(0, 200, k)] + 0.02 * rng.standard_normal((k, 2)),
                               rng.random((n - k, 2))])
    else:
        locs = rng.random((n, 2))
    return locs


Y_SEED = 1  # z ~ N(0, I) of the Vecchia forward simulation


def simulated_dataset(vg, locs, plan, args):
    """Observations drawn from the Vecchia model of the plan at the evaluation
    parameters (model-consistent y keeps the 1e-9 CPU/GPU gate
    meaningful; white noise does not).  Runs on the GPU (vgp_simulate)."""
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, args.beta, args.nu))
    y = vg.simulate_vecchia(vg.Dataset(locs, np.zeros(locs.shape[0])), plan, spec, Y_SEED)
    return vg.Dataset(locs, y)


def workload(args):
    locs = ("U[0,1]^2 seed 0" if args.locations == "uniform" else
            "clustered seed 0: 80% in 200 Gaussian clusters (sd 0.02), 20% U[0,1]^2")
    ordering = {"random": "random(seed=0)", "maxmin": "maxmin (exact, device)",
                "morton": "morton"}[args.ordering]
    return {"workload": "vecchia_loglik", "n": args.n, "m": args.m, "kernel": "matern",
            "nu": args.nu, "sigma_sq": 1.0, "beta": args.beta, "ordering": ordering,
            "locations": locs, "observations": f"Vecchia forward simulation at the evaluation "
            f"parameters (vgp_simulate, z seed {Y_SEED})",
            "l2": "inputs > L2 (272 MB), no flush"}


def flop_count(n, m):
    return float(n - m + 1) * (m**3 / 3.0 + 2.0 * m**2 + 4.0 * m)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU baseline

def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


PORT_NOTE = ("oracle/vecchia_oracle.c: the reference algorithm restated in C (fixed-chunk "
             "threads like vg/parallel.py); its POTRF updates the lower triangle only where "
             "the reference's _potrf_sweep updates the full trailing block "
             "(vg/batchla.py:146-156), so it is faster than the reference's own code "
             "(94.6 s/eval on 8 cores, SURVEY.md §3.1)")


def cpu_baseline(args, ordered, table, gpu_res):
    """Oracle C restatement (oracle/vecchia_oracle.c) on a prefix of the same
    ordered problem: the first n' ordered points form exactly the first
    n' - m + 1 blocks.  Also the parity check of the run: the oracle's total
    on that prefix against the GPU's per-block results over the same blocks,
    and the oracle's neighbour table on a prefix against the GPU's."""
    import hashlib

    from oracle import oracle as O

    import paper_2403_07412_b200 as vg

    threads = os.cpu_count() or 1
    m = args.m
    locs, obs = ordered.locations, ordered.observations
    closed = args.nu in (0.5, 1.5, 2.5)

    def run(nn):
        t0 = time.perf_counter()
        r = O.loglik(locs[:nn], obs[:nn], m, table[: nn - m], "matern", 1.0, args.beta,
                     args.nu, threads=threads)
        dt = time.perf_counter() - t0
        if r.status != 0:
            raise RuntimeError(f"oracle evaluation failed: status {r.status}")
        return r, dt

    n_cal = min(args.n, 20000 if closed else 3000)
    r, t_cal = run(n_cal)
    per_block = t_cal / (n_cal - m + 1)
    n_s = int(min(args.n, max(n_cal, args.cpu_seconds / per_block + m - 1)))
    if n_s > n_cal:
        r, t_s = run(n_s)
    else:
        t_s = t_cal
    blocks_s = n_s - m + 1
    sec_per_eval = t_s / blocks_s * (args.n - m + 1)
    sample = (f"prefix n'={n_s} of the ordered problem ({blocks_s} of {args.n - m + 1} blocks, "
              f"{t_s:.1f}s), extrapolated per block")
    # parity over the same blocks: total == block_first + _ordered_sum(block_rest)
    k = n_s - m
    gpu_prefix = gpu_res.block_first + vg.vecchia._ordered_sum(gpu_res.block_rest[:k])
    rest_rel = np.abs(gpu_res.block_rest[:k] - r.block_rest) / np.maximum(np.abs(r.block_rest), 1e-300)
    n_knn = int(min(args.n, 200000))
    t0 = time.perf_counter()
    knn_ref = O.knn_pred(locs[:n_knn], m, threads)
    knn_s = time.perf_counter() - t0
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()
    parity = {
        "rel_err": abs(gpu_prefix - r.total) / abs(r.total),
        "blocks": blocks_s, "of_blocks": args.n - m + 1,
        "gpu_total": gpu_prefix, "oracle_total": r.total,
        "block_rest_max_rel_err": float(rest_rel.max()) if k else 0.0,
        "knn_rows": n_knn - m, "knn_table_sha256_equal": sha(knn_ref) == sha(table[: n_knn - m]),
        "knn_oracle_s": round(knn_s, 2),
        "gate": "rel_err <= 1e-9 (BASELINE north_star)",
    }
    model, nproc = cpu_info()
    base = {"value": 1.0 / sec_per_eval, "unit": "evals/s", "cores": threads, "kind": "port",
            "sample": sample, "cpu_model": model, "nproc": nproc, "note": PORT_NOTE}
    return base, parity


# ------------------------------------------------------------------ arms

def config_key(args):
    return f"n{args.n}_m{args.m}_nu{args.nu}_{args.locations}_{args.ordering}"


def ncu_traffic(args):
    """DRAM bytes per launch of THIS config's dominant kernel, from the committed
    ncu --set full capture (profiles/ncu_traffic.json), or None if never captured."""
    try:
        with open(TRAFFIC_FILE) as f:
            rec = json.load(f).get(config_key(args))
    except (OSError, ValueError):
        return None, None
    if not rec:
        return None, None
    return rec.get("dram_bytes_per_launch"), rec.get("source")


def run_reference(args, rank, world):
    """`--impl reference`: the reference algorithm on host cores (oracle port)."""
    if rank != 0:
        return
    from oracle import oracle as O

    # (the reference has no maxmin ordering; its per-block cost does not
    # depend on the ordering or on the observation values, so the sample is
    # randomly ordered with N(0,1) observations — no GPU on this arm)
    locs = synthetic(args.n, kind=args.locations)
    y = np.random.default_rng(Y_SEED).standard_normal(args.n)
    perm = np.random.default_rng(0).permutation(args.n)
    ol, oy = locs[perm], y[perm]
    threads = os.cpu_count() or 1
    m = args.m
    t0 = time.perf_counter()
    n_cal = min(args.n, 20000 if args.nu in (0.5, 1.5, 2.5) else 3000)
    table_cal = O.knn_pred(ol[:n_cal], m, threads)
    r = O.loglik(ol[:n_cal], oy[:n_cal], m, table_cal, "matern", 1.0, args.beta, args.nu, threads)
    per_block = (time.perf_counter() - t0) / (n_cal - m + 1)
    budget = max(2.0, min(15.0, 120.0 / max(1, args.steps + args.warmup)))
    n_s = int(min(args.n, max(n_cal, budget / per_block)))
    table = O.knn_pred(ol[:n_s], m, threads)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = O.loglik(ol[:n_s], oy[:n_s], m, table, "matern", 1.0, args.beta, args.nu, threads)
        dt = time.perf_counter() - t0
        if r.status != 0:
            raise RuntimeError("reference evaluation failed")
        if i >= args.warmup:
            times.append(dt)
    blocks_s = n_s - m + 1
    step_s = statistics.mean(times)
    sec_per_eval = step_s / blocks_s * (args.n - m + 1)
    value = 1.0 / sec_per_eval
    sample = (f"prefix n'={n_s} of the ordered problem ({blocks_s} of {args.n - m + 1} blocks "
              f"per step, {step_s:.2f} s), extrapolated per block to n={args.n}")
    model, nproc = cpu_info()
    line = {
        "impl": "reference", "metric": "vecchia_loglik_evals_per_s", "value": value,
        "unit": "evals/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * step_s, "ms_per_eval_extrapolated": 1000.0 * sec_per_eval,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload(args),
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port",
                         "sample": sample, "cpu_model": model, "nproc": nproc,
                         "note": PORT_NOTE},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


VARIANT_NAMES = {0: "generic", 1: "warp-dmma-allreg", 4: "warp-specialised+dcache",
                 7: "ws-scheduler-aware",
                 8: "ws-scheduler-aware+dcache", 11: "large-m-cta", 12: "large-m-cta+dcache",
                 13: "thread-per-block"}


def roofline(args, k_avg_ms, flops, n_gpus=1):
    peak, peak_src = fp64_peak()
    achieved = flops / (k_avg_ms * 1e-3) / 1e12
    traffic, traffic_src = ncu_traffic(args)
    return {"bound": "tensor", "pipe": "fp64 (DMMA + DFMA share one pipe)", "achieved": achieved,
            "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
            "traffic_source": traffic_src, "peak_source": peak_src,
            "algorithmic": "flop_count(n,m)=(n-m+1)(m^3/3+2m^2+4m) per launch "
                           "(vg/vecchia.py:241-251), covariance generation excluded",
            "kernel_ms": k_avg_ms}


def run_ours_single(args):
    import torch

    import paper_2403_07412_b200 as vg

    dev = 0
    vg._native.set_device(dev)
    torch.cuda.set_device(dev)
    locs = synthetic(args.n, kind=args.locations)
    t0 = time.perf_counter()
    plan = vg.make_plan(vg.Dataset(locs, np.zeros(args.n)), args.m, args.ordering, seed=0)
    knn_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    data = simulated_dataset(vg, locs, plan, args)
    sim_s = time.perf_counter() - t0
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, args.beta, args.nu))
    dp = plan.device_plan(dev)
    dp.set_data(data)
    dp.set_variant(args.variant)
    stream = torch.cuda.ExternalStream(dp.stream)

    for _ in range(args.warmup):
        dp.launch(spec)
    total, st, _ = dp.fetch()
    if st != 0:
        raise RuntimeError(f"evaluation failed with status {st}")

    dp.set_timing(True)
    dp.kernel_time()  # reset
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            dp.launch(spec)
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    k_ms, k_launches = dp.kernel_time()
    dp.set_timing(False)
    total2, st2, _ = dp.fetch()
    if st2 != 0 or total2 != total:
        raise RuntimeError("non-deterministic or failed evaluation in the timed region")
    k_avg_ms = k_ms / max(k_launches, 1)

    # e2e: the public drop-in call with host buffers (upload + full LogLikResult back);
    # the warm-up holds each result like the timed loop, so the page-locked
    # result pool reaches its steady state (two live generations) untimed
    for _ in range(max(3, args.warmup)):
        res = vg.vecchia_loglik(data, plan, spec)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        res = vg.vecchia_loglik(data, plan, spec)
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    if res.total != total:
        raise RuntimeError("e2e total differs from device-resident total")
    h2d = args.n * 16 + args.n * 8
    d2h = 3 * (args.n - args.m) * 8 + 24

    rl = roofline(args, k_avg_ms, flop_count(args.n, args.m))
    rl["kernel_share"] = k_avg_ms / ms
    line = {
        "metric": "vecchia_loglik_evals_per_s", "value": 1000.0 / ms, "unit": "evals/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload(args),
        "roofline": rl,
        "e2e": {"value": 1.0 / e2e_s, "unit": "evals/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "api": "paper_2403_07412_b200.vecchia_loglik(dataset, plan, spec)"},
        "gpu_launches": (KERNELS_PER_EVAL + (args.nu not in (0.5, 1.5, 2.5))) * args.steps,
        "clocks": clk.summary(),
        "plan_s": round(knn_s, 3), "simulate_s": round(sim_s, 3), "total": total,
        "kernel_variant": VARIANT_NAMES.get(dp.kernel_variant, str(dp.kernel_variant)),
    }
    if args.nu not in (0.5, 1.5, 2.5):
        # general-nu Matern: covariance generation is outside the flop model
        # (SURVEY.md H2); report its throughput beside it — distinct entries
        # (lower triangle of Sigma_e plus v_e) per evaluation
        per_eval = (args.n - args.m) * (args.m * (args.m + 1) // 2 + args.m)
        line["generation"] = {"matern_entries_per_eval": per_eval,
                              "matern_entries_per_s": per_eval * 1000.0 / ms,
                              "method": "per-evaluation degree-7 polynomial table of "
                                        "s2 2^(1-nu)/Gamma(nu) u^nu K_nu(u), 64 segments per "
                                        "binade (csrc/vgp_ktab.cuh)"}
    if not args.no_cpu_baseline:
        ordered = data.permute(plan.permutation)
        base, parity = cpu_baseline(args, ordered, plan.neighbors.neighbors, res)
        line["cpu_baseline"] = base
        line["parity"] = parity
    print(json.dumps(line), flush=True)


def run_ours_multi(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2403_07412_b200 as vg
    from paper_2403_07412_b200.distributed import ShardedVecchia, make_shard_plan

    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    vg._native.set_device(local)
    # communicator lines (nranks, NVLS/ring choice) on stderr, so a scaling run
    # records what NCCL built; stdout stays the one JSON line
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    nccl_log = f"/tmp/vgp_nccl.{os.getpid()}.log"
    os.environ.setdefault("NCCL_DEBUG_FILE", nccl_log)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    locs = synthetic(args.n, kind=args.locations)
    t0 = time.perf_counter()
    plan = vg.make_plan(vg.Dataset(locs, np.zeros(args.n)), args.m, args.ordering, seed=0)
    knn_s = time.perf_counter() - t0
    data = simulated_dataset(vg, locs, plan, args)
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, args.beta, args.nu))
    # the rank's own plan: ordering everywhere, conditioning sets only for its
    # targets (the full plan above only generates the synthetic observations)
    t0 = time.perf_counter()
    sp = make_shard_plan(data, args.m, args.ordering, 0, rank, world)
    shard_plan_s = time.perf_counter() - t0
    sh = ShardedVecchia(data, sp, device=local)
    sp_t = torch.tensor([shard_plan_s], dtype=torch.float64, device="cuda")
    dist.all_reduce(sp_t, op=dist.ReduceOp.MAX)
    shard_plan_s = float(sp_t.item())
    for _ in range(args.warmup):
        total = sh.total(spec)
    sys.stderr.write(f"[bench] rank {rank}/{world}: NCCL {torch.cuda.nccl.version()} communicator, "
                     f"device {local}, blocks [{sh.block_lo}, {sh.block_hi})\n")
    try:  # the communicator NCCL built (nranks, channels), echoed to stderr
        with open(nccl_log) as fh:
            for ln in fh:
                if "nranks" in ln or "NVLS" in ln or "Channel" in ln and "comm" in ln:
                    sys.stderr.write(ln)
    except OSError:
        pass
    if sh.dplan is not None:
        sh.dplan.set_timing(True)
        sh.dplan.kernel_time()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            t = sh.total(spec)
        ev1.record()
        torch.cuda.synchronize()
    dist.barrier()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    k_ms, k_n = sh.dplan.kernel_time() if sh.dplan is not None else (0.0, 0)
    mx = torch.tensor([ms_local, k_ms / max(k_n, 1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    ms, k_avg_ms = (float(v) for v in mx.cpu().tolist())
    if t != total:
        raise RuntimeError("non-deterministic sharded total")
    # e2e: dataset re-upload + sharded evaluation through the public API
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        sh.set_data(data)
        sh.total(spec)
    e2e_local = (time.perf_counter() - t0) / args.e2e_steps
    e2e_t = torch.tensor([e2e_local], dtype=torch.float64, device="cuda")
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_t.item())
    if rank == 0:
        nshard = max(1, sh.block_hi - sh.block_lo)
        flops_rank = flop_count(args.n, args.m) * nshard / (args.n - args.m + 1)
        achieved = flops_rank / (k_avg_ms * 1e-3) / 1e12
        line = {
            "metric": "vecchia_loglik_evals_per_s", "value": 1000.0 / ms, "unit": "evals/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": dict(workload(args), parallelism=f"blocks{world}"),
            "roofline": dict(roofline(args, k_avg_ms, flops_rank),
                             note="rank-0 shard kernel, max over ranks"),
            "e2e": {"value": 1.0 / e2e_s, "unit": "evals/s",
                    "h2d_bytes_per_step": args.n * 24, "d2h_bytes_per_step": 8 * (sh.buf.numel()),
                    "api": "paper_2403_07412_b200.distributed.ShardedVecchia"},
            "gpu_launches": (KERNELS_PER_EVAL + 1 + (args.nu not in (0.5, 1.5, 2.5))) * args.steps,
            "clocks": clk.summary(), "plan_s": round(knn_s, 3),
            "shard_plan_s": round(shard_plan_s, 3), "total": total,
            "collective": "1 NCCL all_reduce(SUM) of 1+n_chunks fp64 per eval",
        }
        print(json.dumps(line), flush=True)
    sh.close()
    dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    # VGP_BENCH_FORCE_MULTI=1 runs the sharded NCCL path even at world size 1
    # (how the multi-GPU code path is exercised on a one-GPU box)
    if world > 1 or os.environ.get("VGP_BENCH_FORCE_MULTI") == "1":
        for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29517"), ("RANK", "0"),
                     ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0")):
            os.environ.setdefault(k, v)
        run_ours_multi(args, rank, world)
    else:
        run_ours_single(args)


if __name__ == "__main__":
    main()
