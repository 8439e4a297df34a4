#!/usr/bin/env python
"""Benchmark: BASELINE.json configs[1] — brute-force kNN, 1e6 x 128 fp32
database, 1e4 queries, k = 10, memory_limit = 1 GB per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full kNN call (all 1e4 queries against the whole database).
N > 1: launched under torchrun, one process per GPU; the database is sharded
over ranks (strong scaling: the job is always C2), each rank runs the fused
path on its shard and an NCCL all_gather + tb_topk_merge combines the exact
per-shard lists.  Timing: CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks.  Inputs (512 MB) exceed the
126 MB L2, so no explicit flush is needed between steps.

Prints one JSON line (rank 0).  --impl reference times the reference's own
CPU algorithm (the oracle port of tensorbudget's pipelined kNN: expanded-form
GEMM + full stable argsort, oracle/knn.py) on the host cores instead.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL's communicator INIT lines go to a per-process log file (NCCL prints to
# stdout otherwise, and stdout must stay the one JSON line); each rank
# forwards them to its stderr when it finishes (_forward_nccl_log).
if "NCCL_DEBUG_FILE" not in os.environ and \
        os.environ.get("NCCL_DEBUG", "WARN").upper() in ("WARN", "VERSION", ""):
    os.environ["NCCL_DEBUG"] = "INFO"
    os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
    os.environ["NCCL_DEBUG_FILE"] = f"/tmp/tb_bench_nccl.%h.{os.getpid()}.log"

N_DB, M_Q, DIM, K = 1_000_000, 10_000, 128, 10
LIMIT = 10**9
METRIC = "knn_queries_per_s"
UNIT = "queries/s"
WORKLOAD = "knn_c2_1e6x128_q1e4_k10_fp32_1GB"


def _traffic(kernel: str):
    """roofline.traffic: DRAM bytes per launch of `kernel` from the committed
    ncu --set full capture (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)[kernel]
        return t["traffic"], t["algorithmic_bytes"], t["ncu_rep"]
    except (OSError, KeyError):
        return None, None, None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0,
                "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
            return
        # nvidia-smi takes ~0.1-0.3 s to print its first line: wait for it so
        # the (short) timed region that follows is actually sampled
        t_end = time.time() + 3.0
        while not self.lines and time.time() < t_end and self.proc.poll() is None:
            time.sleep(0.01)
        self.lines.clear()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(x: np.ndarray, q: np.ndarray, k: int, n_queries: int, threads: int):
    """The reference's kNN algorithm (oracle/knn.py reference_port) on a
    bounded query sample, query chunks spread over `threads` host threads."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import knn as oknn
    sample = q[:n_queries]
    chunks = [c for c in np.array_split(sample, threads) if len(c)]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=len(chunks)) as ex:
        list(ex.map(lambda c: oknn.reference_port(x, c, k, split_bytes=600 * 10**6), chunks))
    dt = time.perf_counter() - t0
    return n_queries / dt, dt


def _profile_json(name: str):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


def host_info() -> dict:
    """CPU model and the BLAS thread pool numpy uses (BASELINE.md §2 asks
    for both next to a CPU number)."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        pools = [p for p in threadpool_info() if p.get("user_api") == "blas"]
        if pools:
            blas = {"library": pools[0].get("internal_api"), "threads": pools[0].get("num_threads")}
    except Exception:          # pragma: no cover - threadpoolctl missing
        pass
    return {"cpu_model": model, "blas": blas}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# SGPR (BASELINE.json configs[3]): ELBO evaluations/s at C4


SG_N, SG_D, SG_M = 2_000_000, 11, 10_000
SG_NTEST = 200_000          # predictive-mean test points (10 % split)


def sgpr_cpu_baseline(n_sample: int, threads: int):
    """fp64 numpy restatement (oracle/sgpr.py) on a bounded sample of N; the
    statistics are linear in N, so evals/s = 1 / (t_stats * N / n + t_tail)."""
    from oracle import sgpr as osgpr
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n_sample, SG_D))
    y = np.sin(X.sum(axis=1)) + 0.1 * rng.standard_normal(n_sample)
    Z = X[:SG_M] if n_sample >= SG_M else rng.standard_normal((SG_M, SG_D))
    t0 = time.perf_counter()
    S, v, yy = osgpr.sufficient_stats(X, y, Z, "rbf", 1.0, 1.0)
    t_stats = time.perf_counter() - t0
    t0 = time.perf_counter()
    osgpr.elbo_from_stats(S, v, yy, SG_N, osgpr.kuu(Z, "rbf", 1.0, 1.0), 0.01, 1.0)
    t_tail = time.perf_counter() - t0
    per_eval = t_stats * SG_N / n_sample + t_tail
    return {"value": 1.0 / per_eval, "unit": "elbo_evals/s", "cores": threads, "kind": "port",
            **host_info(),
            "sample": f"Sigma/v/yy over {n_sample} of N={SG_N} points ({t_stats:.1f}s, "
                      f"linear in N) + fp64 tail ({t_tail:.1f}s): oracle/sgpr.py (GPflow 2.3.1 "
                      "SGPR restatement, numpy/OpenBLAS fp64)"}


def run_sgpr(args, dev, world, rank, dist):
    import torch

    from paper_2206_14148_b200 import SGPR
    from paper_2206_14148_b200.distributed import shard_range
    start, stop = shard_range(SG_N, rank, world)
    g = torch.Generator(device=dev)
    g.manual_seed(77 + rank)
    X = torch.randn((stop - start, SG_D), generator=g, device=dev)
    y = (torch.sin(X.double().sum(1)) + 0.1 * torch.randn(stop - start, generator=g, device=dev,
                                                          dtype=torch.float64)).float()
    g.manual_seed(5)
    Z = torch.randn((SG_M, SG_D), generator=g, device=dev)       # same on every rank
    group = dist.group.WORLD if dist is not None else None
    # warm-up: one full-size evaluation (the first M=1e4 cuSOLVER/cuBLAS calls
    # pay seconds of one-time library initialisation), then time the next
    SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01, memory_limit=LIMIT, group=group).elbo()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    base = torch.cuda.memory_allocated(dev) - (X.numel() + y.numel() + Z.numel()) * 4
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    m = SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01, memory_limit=LIMIT, group=group)
    sampler = ClockSampler(dev.index or 0)
    sampler.start()
    e0.record()
    st = m.statistics()
    e1.record()
    torch.cuda.synchronize()
    peak_stats = torch.cuda.max_memory_allocated(dev) - base
    elbo = m.elbo()
    e2.record()
    torch.cuda.synchronize()
    peak_eval = torch.cuda.max_memory_allocated(dev) - base
    clocks = sampler.stop()
    stats_ms, total_ms = e0.elapsed_time(e1), e0.elapsed_time(e2)
    if dist is not None:
        t = torch.tensor([stats_ms, total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        stats_ms, total_ms = (float(v) for v in t.tolist())
    useful = SG_N * SG_M * (SG_M + 1)
    achieved = useful / (stats_ms / 1e3) / 1e12
    # denominator: the MEASURED sustained tcgen05 kind::i8 rate of the Gram's
    # own instruction on all SMs (profiles/r02_i8_peak.json, tools/probes/
    # i8_peak.py: >= 4 s under the power cap), / 9 u8 x u8 slice products per
    # useful MAC (exact 24-bit fixed-point Gram); also against the i8 floor
    # (16384 ops/cycle/SM) at the SM clock sampled during this run
    i8 = _profile_json("r02_i8_peak.json") or {}
    peak = i8.get("i8_tops_sustained", 3926.7) / 9.0
    sm_mhz = (clocks or {}).get("sm_mhz") or 0.0
    floor_at_clock = 16384 * 148 * sm_mhz * 1e6 / 1e12 / 9.0 if sm_mhz else None
    traffic, alg_bytes, rep = _traffic("sgpr_gram_i8")
    out = {"metric": "sgpr_elbo_evals_per_s", "value": 1e3 / total_ms, "unit": "elbo_evals/s",
           "ms_per_eval": total_ms, "stats_ms": stats_ms, "tail_ms": total_ms - stats_ms,
           "clocks": clocks,
           "elbo": elbo, "dtype": "f32 inputs; Kuf rounded once to 24-bit fixed point, exact "
                                   "integer Gram (u8 slices, s32 TMEM); fp64 accumulation and tail",
           "config": {"workload": "sgpr_c4_rbf_N2e6_d11_M1e4_1GB", "N": SG_N, "d": SG_D,
                      "M": SG_M, "kernel": "rbf", "lengthscale": 1.0, "noise": 0.01,
                      "memory_limit": LIMIT, "chunk_n": int(st.plan.chunk_n),
                      "engine": "i8", "chunk_buffers": int(st.plan.off[4]),
                      "Z": "M points drawn from the X distribution (same seed on every rank)",
                      "parallelism": f"N-shard{world}", "timed": "1 full evaluation (statistics + "
                      "fp64 tail) after one untimed full-size warm-up evaluation"},
           "peak_stats_mb": peak_stats / 1e6, "planned_peak_mb": st.plan.peak_bytes / 1e6,
           "peak_eval_mb": peak_eval / 1e6,
           "peak_note": "max_memory_allocated incl. X, y, Z; peak_eval covers statistics AND the "
                        "packed in-place O(M^3) tail (tb_sgpr_tail_run)",
           "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                        "frac": achieved / peak, "traffic": traffic,
                        "traffic_note": None if traffic is None else
                        f"DRAM bytes per 7808-point chunk launch from {rep}; algorithmic "
                        f"{alg_bytes} B",
                        "kernel": "sgpr_gram_i8 (exact fixed-point Gram on INT8 tcgen05) + "
                                  "overlapped kuf_quant; time = whole statistics pass",
                        "peak_source": "measured sustained tcgen05 kind::i8 "
                                       f"({i8.get('i8_tops_sustained', 3926.7):.0f} TOPS, "
                                       "profiles/r02_i8_peak.json) / 9 slice products per "
                                       "useful MAC",
                        "frac_of_i8_floor_at_run_clock": (achieved / floor_at_clock
                                                          if floor_at_clock else None),
                        "i8_issued_tops": 9.0 * achieved,
                        "frac_of_nominal": achieved / (4500.0 / 9.0),
                        "useful_flops": useful}}
    # predictive mean (BASELINE configs[3] "ELBO + predictive mean") at a
    # 10 % test split, each rank predicting its own shard of test points:
    # mu(X*) = K(X*, Z) w, the fp64 kernel-MVM kernel at d = 11
    nt0, nt1 = shard_range(SG_NTEST, rank, world)
    g.manual_seed(91 + rank)
    Xs = torch.randn((nt1 - nt0, SG_D), generator=g, device=dev)
    m.predict_mean(Xs[:1024])
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    p0.record()
    mu = m.predict_mean(Xs)
    p1.record()
    torch.cuda.synchronize()
    pred_ms = p0.elapsed_time(p1)
    if dist is not None:
        t = torch.tensor([pred_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        pred_ms = float(t.item())
    out["predict"] = {"n_test": SG_NTEST, "ms": pred_ms, "points_per_s": SG_NTEST / (pred_ms / 1e3),
                      "kernel_evals_per_s": SG_NTEST * SG_M / (pred_ms / 1e3),
                      "finite": bool(torch.isfinite(mu).all().item()),
                      "kernel": "kernel_mvm_fixed_kernel<float,11,RBF> (fp64 arithmetic)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = sgpr_cpu_baseline(args.sgpr_cpu_n, host_cores())
    del m, X, y, Z, Xs, mu
    return out


# ---------------------------------------------------------------------------
# Kernel MVM (the paper's §5.1 workload; reference
# build_kernel_mvm, frontend.py:34-54): y = K v, K the n x n SE kernel over
# 1-D inputs, n = 1e6, fp64.  Rows of K (x) are sharded over ranks.

MV_N = 1_000_000
MV_FP64_INST_PER_EVAL = 17     # counted in the SASS of kernel_mvm_fixed_kernel<double,1,RBF>


def mvm_cpu_baseline(n_rows: int, threads: int):
    """The reference's op order (oracle.mvm.se_mvm_reference, numpy) on a
    bounded sample of rows against all n columns; rows are independent, so
    MVM/s = evals/s / n^2."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import mvm as omvm
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, n_rows)
    y = rng.uniform(-1, 1, MV_N)
    v = rng.uniform(-1, 1, MV_N)
    parts = [p for p in np.array_split(x, threads) if len(p)]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=len(parts)) as ex:
        list(ex.map(lambda p: omvm.se_mvm_reference(p, y, v, 1.0, 0.1, chunk=16), parts))
    dt = time.perf_counter() - t0
    evals = n_rows * MV_N / dt
    return {"value": evals / MV_N ** 2, "unit": "mvm/s", "cores": len(parts), "kind": "port",
            **host_info(),
            "sample": f"{n_rows} of {MV_N} rows x all {MV_N} columns in {dt:.1f}s "
                      f"({evals:.3e} kernel evaluations/s): oracle/mvm.py se_mvm_reference "
                      "(reference op order, numpy fp64)"}


def run_mvm(args, dev, world, rank, dist):
    import torch

    from paper_2206_14148_b200 import mvm
    from paper_2206_14148_b200.distributed import shard_range
    start, stop = shard_range(MV_N, rank, world)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    x = (torch.rand((MV_N, 1), generator=g, device=dev, dtype=torch.float64) * 2 - 1)[start:stop]
    y = torch.rand((MV_N, 1), generator=g, device=dev, dtype=torch.float64) * 2 - 1
    v = torch.rand(MV_N, generator=g, device=dev, dtype=torch.float64) * 2 - 1
    mvm.kernel_mvm(x[:4096].contiguous(), y, v, "rbf", 1.0, 0.1)          # warm-up
    xs = x.contiguous()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    out = mvm.kernel_mvm(xs, y, v, "rbf", 1.0, 0.1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    rows = stop - start
    if dist is not None:
        t = torch.tensor([ms, float(rows)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, rows = float(t[0].item()), int(t[1].item())
    evals = rows * MV_N / (ms / 1e3)
    fp64 = _profile_json("r02_fp64_peak.json") or {}
    peak_inst = fp64.get("fp64_tflops", 36.97) / 2.0       # DFMA instructions/s (T)
    achieved_inst = evals * MV_FP64_INST_PER_EVAL / 1e12
    res = {"metric": "kernel_mvm_per_s", "value": 1e3 / ms, "unit": "mvm/s", "ms_per_mvm": ms,
           "kernel_evals_per_s": evals, "checksum": float(out.sum().item()),
           "config": {"workload": "se_kernel_mvm_n1e6_d1_f64", "n": MV_N, "dtype": "f64",
                      "kernel": "squared exponential, variance 1, lengthscale 0.1",
                      "parallelism": f"row-shard{world}",
                      "memory": "O(n): K is never formed (the reference materialises 8 TB "
                                "naive, 125-row slices at a 1 GB split)"},
           "roofline": {"bound": "fp64", "achieved": achieved_inst, "peak": peak_inst,
                        "unit": "T fp64-pipe instructions/s", "frac": achieved_inst / peak_inst,
                        "kernel": "kernel_mvm_fixed_kernel<double, 1, RBF, 4>",
                        "per_unit": f"{MV_FP64_INST_PER_EVAL} fp64 instructions per kernel "
                                    "evaluation (SASS count: difference, square, exp range "
                                    "reduction + 11-term polynomial, accumulate)",
                        "peak_source": "measured DFMA rate (profiles/r02_fp64_peak.json, "
                                       "tools/probes/fp64_peak_probe.cu)"}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = mvm_cpu_baseline(args.mvm_cpu_rows, host_cores())
    return res


def _forward_nccl_log():
    """Copy this process's NCCL debug file (see NCCL_DEBUG_FILE above) to
    stderr, so the launcher sees the communicator lines (nranks, NVLS)."""
    import glob
    pat = os.environ.get("NCCL_DEBUG_FILE", "")
    if not pat.startswith("/tmp/tb_bench_nccl."):
        return
    for path in glob.glob(pat.replace("%h", "*")):
        try:
            with open(path) as fh:
                sys.stderr.write(fh.read())
            os.remove(path)
        except OSError:
            pass
    sys.stderr.flush()


def spawn_ranks(gpus: int, argv) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch this script as N ranks
    (one process per GPU) through torch.distributed.run on 127.0.0.1, the
    same launch the driver uses; rank 0's JSON line reaches our stdout."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *argv]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.run(cmd, env=env).returncode


def run_dry(args):
    """--dry-run: the launch plumbing only (CPU, gloo): every rank joins the
    group and all-reduces its rank; rank 0 prints what it saw.  Lets the
    N-rank spawn be tested without GPUs (tests/test_bench_launch.py)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([float(rank), 1.0])
        dist.all_reduce(t)
        ranks_sum, ranks = int(t[0].item()), int(t[1].item())
        dist.destroy_process_group()
    else:
        ranks_sum, ranks = 0, 1
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "requested_gpus": args.gpus,
                          "ranks": ranks, "rank_sum": ranks_sum}))
    return 0


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    rng = np.random.default_rng(2)
    x = rng.standard_normal((N_DB, DIM), dtype=np.float32)
    q = rng.standard_normal((M_Q, DIM), dtype=np.float32)
    threads = host_cores()
    per_step = max(threads, args.ref_queries)
    for _ in range(args.warmup):
        cpu_baseline(x, q, K, per_step, threads)
    times = []
    for _ in range(args.steps):
        _, dt = cpu_baseline(x, q, K, per_step, threads)
        times.append(dt)
    total = sum(times)
    value = per_step * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic N(0,1)",
        "config": {"workload": WORKLOAD, "n": N_DB, "m": M_Q, "d": DIM, "k": K,
                   "memory_limit": LIMIT, "step_sample_queries": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         **host_info(),
                         "sample": f"{per_step} queries/step vs the full 1e6x128 db: "
                                   "tensorbudget pipelined kNN (expanded-form GEMM + full "
                                   "stable argsort, oracle/knn.py reference_port)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2206_14148_b200 as tb
    from paper_2206_14148_b200 import distributed, neighbors

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TB_FORCE_DIST=1 exercises the NCCL gather/merge path even at world 1
    use_dist = world > 1 or os.environ.get("TB_FORCE_DIST") == "1"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if use_dist:
        dist.init_process_group("nccl", device_id=dev)
    start, stop = distributed.shard_range(N_DB, rank, world)
    rows = stop - start

    # synthetic data, generated on the device (same queries on every rank)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    x = torch.randn((rows, DIM), generator=g, device=dev, dtype=torch.float32)
    g.manual_seed(99)
    q = torch.randn((M_Q, DIM), generator=g, device=dev, dtype=torch.float32)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    base_alloc = torch.cuda.memory_allocated(dev) - (x.numel() + q.numel()) * 4

    out_dtype = np.float64 if use_dist else np.float32
    op = neighbors.KnnOperator(rows, M_Q, DIM, K, dtype=np.float32, out_dtype=out_dtype,
                               engine=args.engine, memory_limit=LIMIT, device=dev)
    plan = op.plan
    out = op.alloc_outputs()
    n_ev = 2 * int(plan.n_chunks)
    ev_sets = [[torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
               for _ in range(args.steps)]
    for evs in ev_sets:           # materialise the cudaEvent_t handles
        for e in evs:
            e.record()
    torch.cuda.synchronize()

    def step(events=None):
        if not use_dist:
            return op.run(x, q, out, events=events)
        return distributed.knn_sharded(x, q, K, index_base=start, operator=op, events=events)

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        step()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for s in range(args.steps):
        step(ev_sets[s])
    t1.record()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    clocks = sampler.stop()
    ms = t0.elapsed_time(t1)
    if use_dist:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    peak_dev = torch.cuda.max_memory_allocated(dev) - base_alloc
    # kernels this library launches per step, counted (CUPTI) on one extra
    # untimed step: every prep / candidate-engine / merge / re-rank kernel
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    launches_per_step = sum(1 for e in prof.events()
                            if e.device_type.name == "CUDA" and "tb::" in e.name)
    value = M_Q * args.steps / (ms / 1000.0)
    fb = op.fallback_count()

    # dominant kernel (candidate engine) time, measured inside the timed
    # region on every rank; N > 1: the slowest rank's (max over ranks)
    per = []
    for evs in ev_sets:
        per.append(sum(evs[2 * c].elapsed_time(evs[2 * c + 1])
                       for c in range(int(plan.n_chunks))))
    eng_ms = sum(per) / len(per)
    if use_dist:
        tt = torch.tensor([eng_ms, float(rows)], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        eng_ms, rows_max = float(tt[0].item()), int(tt[1].item())
    else:
        rows_max = rows

    # end to end through the public operator: pinned host inputs copied in,
    # results copied out, every step
    e2e = None
    if not args.no_e2e:
        # the reference-facing call with HOST buffers (tb_knn_run_host): pinned
        # x, q copied in (queries first, then the database chunk by chunk on
        # one copy stream, overlapped with compute) and dist, idx copied out,
        # every step.  Its plan caps chunks at n/20 so nineteen of the twenty
        # database copies overlap compute (tools/e2e_chunks.py: 4/8/12/16/24
        # chunks -> 0.89/0.97/0.99/1.00/0.85 M q/s on an early build; with the
        # current engine 12/16/20/24/32 -> 0.998/1.001/1.007/1.008/0.911 M q/s,
        # 20 keeps a margin below the cliff; the bound is PCIe).
        # N > 1: every rank copies its shard in, the per-shard lists meet on
        # the device (NCCL all_gather + merge) and the global result is copied
        # out on every rank (distributed.knn_sharded_host).
        xh = x.cpu().pin_memory()
        qh = q.cpu().pin_memory()
        op_h = neighbors.KnnOperator(rows, M_Q, DIM, K, dtype=np.float32, out_dtype=out_dtype,
                                     engine=args.engine, memory_limit=LIMIT, device=dev,
                                     max_chunk_rows=((rows + 19) // 20 + 255) // 256 * 256)
        staging = (x, q, out[0], out[1])      # device buffers refilled every step
        dh = torch.empty(out[0].shape, dtype=out[0].dtype).pin_memory()
        ih = torch.empty(out[1].shape, dtype=out[1].dtype).pin_memory()

        if use_dist:
            def e2e_step():
                distributed.knn_sharded_host(xh, qh, K, index_base=start, operator=op_h,
                                             staging=staging, out_host=(dh, ih))
        else:
            def e2e_step():
                op_h.run_host(xh, qh, (dh, ih), staging=staging)

        for _ in range(max(1, args.warmup)):
            e2e_step()
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        host_ms = (time.perf_counter() - h0) * 1000 / args.steps
        e1.record()
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if use_dist:
            dist.barrier()
            tt = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        if os.environ.get("TB_BENCH_TRACE") and not use_dist:   # diagnosis: CUPTI timeline
            from torch.profiler import profile, ProfilerActivity
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                for _ in range(2):
                    e2e_step()
                torch.cuda.synchronize()
            tl = sorted((e.time_range.start, e.time_range.end, e.name[:60])
                        for e in prof.events() if e.device_type.name == "CUDA")
            with open(os.environ["TB_BENCH_TRACE"], "w") as f:
                for a, b, nm in tl:
                    f.write(f"{(a - tl[0][0]) / 1000:9.3f} {(b - a) / 1000:8.3f}  {nm}\n")
        # the bound of this path: one pinned host->device copy of the same
        # bytes, alone (PCIe), timed the same way (this rank's bytes)
        hb = int(x.numel() * 4 + q.numel() * 4)
        e0.record()
        for _ in range(3):
            x.copy_(xh, non_blocking=True)
            q.copy_(qh, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        h2d_ms = e0.elapsed_time(e1) / 3
        hb_job, ob_job = hb, int(dh.numel() * dh.element_size() + ih.numel() * 8)
        if use_dist:
            tb_ = torch.tensor([hb_job, ob_job], device=dev, dtype=torch.float64)
            dist.all_reduce(tb_)
            hb_job, ob_job = (int(v) for v in tb_.tolist())
        e2e = {"value": M_Q * args.steps / (ems / 1000.0), "unit": UNIT,
               "h2d_only_ms": h2d_ms, "h2d_gbs": hb / h2d_ms / 1e6, "host_enqueue_ms": host_ms,
               "frac_of_h2d_bound": h2d_ms / (ems / args.steps),
               "h2d_bytes_per_step": hb_job,
               "d2h_bytes_per_step": ob_job,
               "ms_per_step": ems / args.steps,
               "chunks": int(op_h.plan.n_chunks),
               "path": ("distributed.knn_sharded_host: per rank KnnOperator.run_host -> "
                        "tb_knn_run_host (pinned shard + queries in), NCCL all_gather + "
                        "tb_topk_merge, global dist,idx out" if use_dist else
                        "KnnOperator.run_host -> tb_knn_run_host: pinned host x,q in "
                        "(per-chunk H2D overlapped with compute), dist,idx out")}
        del op_h

    peaks, peak_src = _peaks()
    roof = None
    if eng_ms:
        useful = 2.0 * M_Q * rows_max * DIM    # cross-term flops (largest shard)
        engine = {1: "tc3", 2: "simt", 3: "tc1"}[int(plan.engine)]
        passes = {"tc3": 3, "tc1": 1, "simt": 1}[engine]
        achieved = useful / (eng_ms / 1000.0) / 1e12
        # burst figure: one step is a few ms and the SM clock stays at its
        # maximum (no power-cap reason in `clocks`), i.e. a kernel timed alone
        peak = peaks["bf16_tflops"] / passes
        traffic, alg_bytes, rep = _traffic({"tc3": "knn_tc", "tc1": "knn_tc1"}.get(engine, ""))
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_note": None if traffic is None else
                f"DRAM bytes per chunk launch from {rep}; algorithmic {alg_bytes} B",
                "kernel": f"knn candidate engine ({engine})",
                "kernel_ms": eng_ms, "kernel_share_of_step": eng_ms / (ms / args.steps),
                "peak_source": f"{peak_src} bf16 burst / {passes} MMA passes per useful MAC",
                "frac_of_sustained": achieved / (peaks.get("bf16_tflops_sustained",
                                                           peaks["bf16_tflops"]) / passes)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = host_cores()
        xs = x.cpu().numpy()
        qs = q.cpu().numpy()
        nq = max(threads, args.cpu_queries)
        v, dt = cpu_baseline(xs, qs, K, nq, threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", **host_info(),
               "sample": f"{nq} queries vs the full 1e6x128 db in {dt:.1f}s "
                         "(tensorbudget pipelined kNN algorithm, oracle/knn.py)"}

    sgpr = None
    if not args.no_sgpr:
        del op
        torch.cuda.empty_cache()
        sgpr = run_sgpr(args, dev, world, rank, dist if use_dist else None)
    mvm_line = None
    if not args.no_mvm:
        torch.cuda.empty_cache()
        mvm_line = run_mvm(args, dev, world, rank, dist if use_dist else None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic N(0,1), generated on device",
            "config": {"workload": WORKLOAD, "n": N_DB, "m": M_Q, "d": DIM, "k": K,
                       "memory_limit": LIMIT, "engine": args.engine,
                       "parallelism": f"db-shard{world}",
                       "l2_policy": "inputs (512 MB) larger than L2; no flush",
                       "plan": {"engine": int(plan.engine), "cand": int(plan.cand),
                                "slices": int(plan.slices), "chunks": int(plan.n_chunks),
                                "chunk_rows": int(plan.chunk_rows),
                                "workspace_mb": plan.workspace_bytes / 1e6,
                                "planned_peak_mb": plan.peak_bytes / 1e6}},
            "peak_device_mb": peak_dev / 1e6,
            "peak_device_note": "torch max_memory_allocated over the timed region "
                                "(inputs + workspace + outputs) vs memory_limit",
            "fallback_queries": fb,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "sgpr": sgpr,
            "mvm": mvm_line,
        }
        print(json.dumps(line))
    if use_dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--engine", default="auto")
    ap.add_argument("--cpu-queries", type=int, default=384)
    ap.add_argument("--ref-queries", type=int, default=384)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sgpr", action="store_true")
    ap.add_argument("--sgpr-cpu-n", type=int, default=16384)
    ap.add_argument("--no-mvm", action="store_true")
    ap.add_argument("--mvm-cpu-rows", type=int, default=2048)
    ap.add_argument("--dry-run", action="store_true",
                    help="launch plumbing only (gloo, no GPU work)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return spawn_ranks(args.gpus, sys.argv[1:])
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    try:
        return run_ours(args)
    finally:
        _forward_nccl_log()


if __name__ == "__main__":
    sys.exit(main())
