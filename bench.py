#!/usr/bin/env python
"""bench.py — FastPFP outer iterations/s on B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c5|c2|c4] [--precision P]

A step = one FastPFP outer iteration (Algorithm 1 lines 3-9): GEMM1 (U = A' X^T),
GEMM2 (Y = A U^T + lambda K), the projection loop (20 sweeps at c5), blend + rescale. The default
workload is BASELINE.json configs[4] (c5: n = n' = 16384, d = 64, fixed 20 x 20), whose inputs
(A, A', Y: 1.07 GB each) are larger than the 126 MB L2, so no L2 flush is needed between steps.
With N > 1 GPUs c5 is row-sharded over the ranks (one pair, strong scaling) and
`--workload c4` splits BASELINE configs[3]'s 8192 pairs evenly (no communication).
`python bench.py --gpus N` without a torchrun environment re-launches itself under
`torch.distributed.run` with N ranks on 127.0.0.1.

Timing: W untimed warm-up steps, then exactly K steps between barrier + cuda.synchronize on both
sides, timed with CUDA events on the handle's stream (torch's current stream), max over ranks.
Per-kernel device time (GEMM vs projection) comes from the library's own CUDA events on the same
stream (FASTPFP_OPT_PROFILE). nvidia-smi clocks are sampled during the timed region.

Roofline bookkeeping: GEMM flops 2nn'(n+n') per outer iteration;
projection ALGORITHMIC bytes 8 m^2 k (one read + one write of Y per sweep) + 12 n n' (the finalize
reads X and Y's X block and writes X) — anything else the kernel moves (the sums pass after the
GEMM, the second finalize pass, X's digit planes) is overhead, visible in `traffic` (ncu DRAM bytes).

--impl reference runs the fp64 CPU oracle (oracle/, the only other place bench.py executes it) on
a bounded sample of the same workload (rank 0 only) and prints the same JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FastPFP outer iters/s at n=1000 & 16384 (1–8 GPU); TFLOP/s & HBM GB/s vs peak"
UNIT = "outer_iters/s"
SMS = 148
# tcgen05 issue rates measured on this part (profiles/r01_tcgen05_peak_micro.txt), MAC/clk/SM
I8_MAC_CLK, TF32_MAC_CLK = 8192, 2048


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return mp, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md "clocks DURING the timed region")
# ------------------------------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int, period_ms: int = 50):
        self.idx = device_index
        self.period = period_ms
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.15)          # the first sample lands before the timed region starts
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


BAD_REASONS = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


# ------------------------------------------------------------------------------------------------
# distributed plumbing
# ------------------------------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def maybe_init_pg(world, backend):
    if world > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group(backend=backend)


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if (torch.cuda.is_available() and dist.get_backend() == "nccl") else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(argv, gpus: int) -> int:
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU) with torch.distributed.run
    on 127.0.0.1, the same launch the driver uses; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd, cwd=ROOT)


def finish_pg(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------------------------------------
# workload and roofline bookkeeping
# ------------------------------------------------------------------------------------------------
def make_problem(workload: str):
    from paper_1207_1114_b200 import inputs
    if workload == "c5":
        return inputs.config5()
    if workload == "c2":
        return inputs.config2()
    raise SystemExit(f"unknown workload {workload}")


def workload_desc(p, workload):
    if workload == "c5":
        return (f"c5 (BASELINE configs[4]): n=n'={p.n}, d={p.d}, ER p=0.1 U(0,1) + N(0,0.05^2) edge noise, "
                f"planted permutation, lambda={p.lam}, alpha={p.alpha}, fixed {p.max_iter2} sweeps per outer")
    return (f"c2 (BASELINE configs[1]): n=n'={p.n}, d={p.d}, ER p=0.5, lambda={p.lam}, alpha={p.alpha}, "
            f"eps1=eps2={p.eps1}, I0=I1={p.max_iter1}")


def proj_alg_bytes(n, npr, sweeps):
    """SURVEY §8(d) algorithmic bytes of the projection + finalize of one outer iteration: each
    sweep reads and writes Y once (8 m^2), the finalize reads X and Y[0:n,0:n'] and writes X (12 nn')."""
    m = max(n, npr)
    return 8 * m * m * sweeps + 12 * n * npr


def step_alg_bytes(n, npr, sweeps, lam_k):
    """SURVEY §8(d) B_alg per outer iteration: 4 (n^2 + n'^2 + 7 n n' [+ n n' for K]) + 8 m^2 k."""
    return 4 * (n * n + npr * npr + 7 * n * npr + (n * npr if lam_k else 0)) + 8 * max(n, npr) ** 2 * sweeps


def precision_name(prec):
    return {0: "tf32x3", 1: "tf32", 2: "fp32_simt", 3: "int8_ozaki"}[prec]


def gemm_peak(mp, src, prec):
    """Algorithmic-flop peak of one fp32-accurate product in the GEMM's own dtype (B200_PROFILING.md:
    another dtype's measured peak x the guide's nominal ratio; the sustained figure for a kernel
    timed inside a long step). int8 = bf16 x 4.5/2.25, 6 int8 MMAs per product; TF32 = bf16 x
    1.1/2.25, 3 MMAs per product for 3xTF32. SIMT fp32: 148 SMs x 128 FMA/clk x 2 x 1.965 GHz."""
    bf = mp["bf16_tflops_sustained"]
    if prec == 2:
        return SMS * 128 * 2 * 1.965e9 / 1e12, "alu", "fp32 FFMA peak 74.4 TF/s (148 SMs x 128 lanes x 2 flop x 1.965 GHz, derived)"
    if prec == 3:
        i8 = bf * 4.5 / 2.25
        return i8 / 6.0, "tensor", (f"int8 Ozaki: ({src} bf16 sustained {bf} x 4.5/2.25 nominal int8/bf16 dense ratio "
                                    f"= {i8:.0f} TOPS) / 6 int8 MMAs per fp32-accurate product")
    tf32 = bf * 1.1 / 2.25
    if prec == 1:
        return tf32, "tensor", f"tf32 = {src} bf16 sustained {bf} x 1.1/2.25 (nominal dense ratio)"
    return tf32 / 3.0, "tensor", (f"3xTF32: ({src} bf16 sustained {bf} x 1.1/2.25 nominal tf32/bf16 dense ratio) / 3 "
                                  f"TF32 MMAs per fp32-accurate product")


def pipe_peak(prec, sm_mhz):
    """The same kernel against the tcgen05 issue rate measured on this part at the median SM clock
    seen during the timed region (algorithmic flops: 6 int8 / 3 TF32 MMAs per fp32-accurate product)."""
    mac = {3: I8_MAC_CLK / 6.0, 0: TF32_MAC_CLK / 3.0, 1: float(TF32_MAC_CLK)}.get(prec)
    if not mac or not sm_mhz:
        return None
    return SMS * mac * 2 * sm_mhz * 1e6 / 1e12


def ncu_traffic(kernel_key):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from the committed ncu
    --set full capture summarised in profiles/ncu_summary.json."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get(kernel_key, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------------------------------------
# our arm: c5 (default) / c2 on the fixed schedule
# ------------------------------------------------------------------------------------------------
def timed_steps(s, p, inner, steps, world, local, stream, clock_ms=50):
    """Exactly `steps` outer iterations between barrier + synchronize, CUDA events on the stream."""
    import torch
    s.reset_stats()
    barrier(world)
    torch.cuda.synchronize()
    clk = Clocks(local, clock_ms)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    done = 0
    while done < steps:
        k = min(64, steps - done)
        _, rep = s.iterate(p.alpha, p.lam, 0.0, 0.0, k, inner, want_x=False, trace=0)
        if rep.iterations == 0 or rep.degenerate:
            raise SystemExit(f"bench: degenerate iterate after {done} steps (max X~ <= 1e-300)")
        done += rep.iterations
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    c = clk.stop()
    return e0.elapsed_time(e1), c, s.stats()


def run_ours(args):
    import torch

    import paper_1207_1114_b200 as F
    from paper_1207_1114_b200 import dist as D

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    maybe_init_pg(world, "nccl")
    mp, src = load_peaks()

    p = make_problem(args.workload)
    inner = p.max_iter2 if args.workload == "c5" else 20
    sharded = (world > 1 or args.force_shard) and args.workload == "c5"
    if sharded:
        # row-sharded pair (BASELINE configs[4]): this rank owns n/P rows; NCCL over NVLink
        shard = D.row_partition(p.n, p.n_prime, world, rank)
        s = D.make_solver(p.n, p.n_prime, p.d)
        A_l, Ap_l, B_l, Bp_l = D.local_inputs(p, shard)
    else:
        shard = None
        s = F.Solver(p.n, p.n_prime, p.d)
        A_l, Ap_l, B_l, Bp_l = p.A, p.Ap, p.B, p.Bp
    stream = torch.cuda.current_stream()
    s.set_option(F.OPT_STREAM, stream.cuda_stream)
    if args.precision is not None:
        s.set_option(F.OPT_PRECISION, args.precision)
    prec = s.get_option(F.OPT_PRECISION)        # the library default unless --precision is given
    s.set_option(F.OPT_CHECK_EVERY, 64)
    s.set_graphs(A_l, Ap_l, B_l, Bp_l)
    if p.X0 is not None:
        s.set_x0(p.X0 if not sharded else np.ascontiguousarray(p.X0[shard.sl]))

    # warm-up (untimed)
    s.iterate(p.alpha, p.lam, 0.0, 0.0, max(args.warmup, 1), inner, want_x=False)
    s.set_option(F.OPT_PROFILE, 1)
    ms, clocks, st = timed_steps(s, p, inner, args.steps, world, local, stream)
    if set(clocks.get("reasons", [])) & BAD_REASONS:
        ms, clocks, st = timed_steps(s, p, inner, args.steps, world, local, stream)   # re-measure once
        clocks["remeasured"] = True
    ms_max = max_over_ranks(ms, world)
    # sharded: the ranks cooperate on ONE pair (strong scaling); else every rank runs its own pair
    value = args.steps / (ms_max / 1e3) if sharded else args.steps * world / (ms_max / 1e3)
    step_ms = ms / args.steps
    rows_local = shard.rows if sharded else p.n

    roofline = gemm_roofline(mp, src, prec, st, step_ms, clocks, sharded, args.workload == "c5")
    pbytes = proj_alg_bytes(p.n, p.n_prime, inner) * rows_local // p.n
    proj_ms = st["proj_ms"] / max(st["proj_launches"], 1)
    proj_gbs = pbytes / (proj_ms / 1e3) / 1e9
    roofline["secondary"] = {
        "kernel": "proj_kernel (sums pass + 20 sweeps + finalize, one launch)" if not sharded else
                  "projection phase (sums + 20 sweep launches + finalize, NCCL all-reduces between)",
        "bound": "hbm", "achieved": round(proj_gbs, 1), "peak": mp["hbm_gbs"], "unit": "GB/s",
        "frac": round(proj_gbs / mp["hbm_gbs"], 4), "bytes_per_launch": pbytes,
        "bytes_rule": "SURVEY 8(d): 8 m^2 k (sweeps) + 12 n n' (finalize); sums pass, second finalize "
                      "pass and X digit planes are overhead (in traffic); single GPU: checkpointed sweeps "
                      "store Y after every other sweep only (DESIGN.md 6), so traffic is below these bytes",
        "ms_per_launch": round(proj_ms, 4), "share_of_step": round(proj_ms / step_ms, 4),
        "traffic": ncu_traffic("proj_kernel") if args.workload == "c5" and not sharded else None,
        "peak_source": f"{src} hbm_gbs (burst copy; the projection runs inside a long step)"}
    # SURVEY 8(d) composite: T_roof = max(F/peak_tensor, B/BW), T_seq = F/peak + B/BW (per rank)
    F_step = 2.0 * rows_local * p.n_prime * (p.n + p.n_prime)
    B_step = step_alg_bytes(p.n, p.n_prime, inner, p.lam != 0 and p.d > 0) * rows_local / p.n
    t_tensor = F_step / (roofline["peak"] * 1e12) * 1e3
    t_hbm = B_step / (mp["hbm_gbs"] * 1e9) * 1e3
    composite = {"flops_per_step": F_step, "alg_bytes_per_step": B_step,
                 "t_tensor_ms": round(t_tensor, 3), "t_hbm_ms": round(t_hbm, 3),
                 "t_roof_ms": round(max(t_tensor, t_hbm), 3), "t_seq_ms": round(t_tensor + t_hbm, 3),
                 "t_step_ms": round(step_ms, 3), "frac_roof": round(max(t_tensor, t_hbm) / step_ms, 4),
                 "frac_seq": round((t_tensor + t_hbm) / step_ms, 4),
                 "note": "peaks: roofline.peak (tensor, per fp32-accurate product) and measured hbm_gbs"
                         + ("; all-gather bytes over NVLink not included" if sharded else "")}

    out = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": (workload_desc(p, args.workload) if args.workload == "c5" else
                                (f"c2 problem (BASELINE configs[1] recipe: n=n'={p.n}, d={p.d}, ER p=0.5, "
                                 f"lambda={p.lam}, alpha={p.alpha}) on c5's fixed schedule: eps = 0, "
                                 f"{inner} sweeps per outer (the converging c2 run is secondary_c2 of "
                                 f"the default line)")),
                   "n": p.n, "n_prime": p.n_prime, "d": p.d,
                   "inner_sweeps": inner, "gemm": precision_name(prec),
                   "parallelism": (f"rowshard{world} (NCCL all-gather of U + per-sweep all-reduce)" if sharded
                                   else ("replicas" if world > 1 else "single")),
                   "l2": "inputs larger than L2 (A, A', Y 1.07 GB each vs 126 MB L2); no flush needed"
                   if args.workload == "c5" else "working set L2-resident"},
        "roofline": roofline, "composite": composite, "clocks": clocks, "gpu_launches": int(st["launches"]),
    }

    # end to end through the public API with HOST buffers (pinned): upload graphs, full 20 x 20
    # solve, read X back
    if not args.no_e2e:
        out["e2e"] = e2e(s, p, inner, stream, world, shard)
    if args.workload == "c5" and not args.no_secondary:
        out["full_match"] = full_match(s, p, inner, stream, world, shard)
    s.close()
    if rank == 0 and world == 1 and args.workload == "c5" and not args.no_secondary:
        out["precision_lines"] = {precision_name(q): precision_line(p, q, inner, min(args.steps, 6), mp, src)
                                  for q in (0, 1)}
        out["secondary_c1"] = secondary_pair("c1")
        out["secondary_c1_batched"] = secondary_c1_batched()
        out["secondary"] = secondary_pair("c2")
        out["secondary_c3"] = secondary_pair("c3")
        out["secondary_c4"] = secondary_c4(mp, src)
        out["secondary_pg"] = secondary_pair("c2", method=1)
        out["secondary_fastga"] = secondary_ga()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.workload, p)
    if rank == 0:
        print(json.dumps(out), flush=True)
    finish_pg(world)


def gemm_roofline(mp, src, prec, st, step_ms, clocks, sharded, c5):
    """Roofline of the dominant kernel (the GEMM at c5: one kernel, two launches per step)."""
    gemm_ms = st["gemm_ms"] / max(st["gemm_launches"], 1)
    flops_launch = st["gemm_flops"] / max(st["gemm_launches"], 1)
    achieved_tf = flops_launch / (gemm_ms / 1e3) / 1e12
    peak, bound, peak_note = gemm_peak(mp, src, prec)
    pp = pipe_peak(prec, clocks.get("sm_mhz"))
    return {
        "kernel": f"gemm_{precision_name(prec)}", "bound": bound, "achieved": round(achieved_tf, 2),
        "peak": round(peak, 2), "unit": "TFLOP/s", "frac": round(achieved_tf / peak, 4),
        "traffic": ncu_traffic(f"gemm_{precision_name(prec)}") if c5 and not sharded else None,
        "flops_per_launch": flops_launch, "ms_per_launch": round(gemm_ms, 4),
        "share_of_step": round(st["gemm_launches"] * gemm_ms / max(st["outer_iterations"], 1) / step_ms, 4),
        "peak_source": peak_note,
        "vs_measured_pipe": None if pp is None else {
            "peak": round(pp, 1), "frac": round(achieved_tf / pp, 4),
            "source": f"measured tcgen05 issue rate x {SMS} SMs x median SM clock {clocks.get('sm_mhz')} MHz"},
        "note": ("gemm_ms spans both GEMM launches and the NCCL all-gather between them" if sharded
                 else "per GEMM launch (GEMM1 and GEMM2 have equal flops at n = n')"),
    }


def e2e(s, p, inner, stream, world, shard=None):
    import torch
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory() if a is not None else None
    rows = p.n if shard is None else shard.rows
    sl = slice(0, p.n) if shard is None else shard.sl
    A, Ap = pin(p.A[sl]), pin(p.Ap)
    B = pin(p.B[sl]) if p.B is not None else None
    Bp = pin(p.Bp)
    Xh = torch.empty((rows, p.n_prime), dtype=torch.float32).pin_memory()
    outer = p.max_iter1 if p.eps1 == 0.0 else 20

    def one():
        s.set_graphs(A, Ap, B, Bp)      # H2D from pinned host memory + validation + K = BB'^T
        s.set_x0(None if p.X0 is None else np.ascontiguousarray(p.X0[sl]))
        s.iterate(p.alpha, p.lam, 0.0, 0.0, outer, inner, want_x=False)
        s.copy_x(Xh)                    # D2H of the result
    one()                               # warm-up
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    one()
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = max_over_ranks(max(e0.elapsed_time(e1), wall * 1e3), world)
    h2d = sum(x.numel() * 4 for x in (A, Ap, B, Bp) if x is not None)
    per_rank_pairs = 1 if shard is not None else world
    return {"value": round(outer * per_rank_pairs / (ms / 1e3), 4), "unit": UNIT,
            "h2d_bytes_per_step": h2d // outer, "d2h_bytes_per_step": (rows * p.n_prime * 4) // outer,
            "what": f"fastpfp_set_graphs(pinned host A,A',B,B') + set_x0 + iterate({outer} outer x {inner} sweeps) "
                    f"+ fastpfp_copy_x(pinned host); bytes amortised over the {outer} outer steps of one solve",
            "ms_per_solve": round(ms, 3)}


def full_match(s, p, inner, stream, world, shard=None):
    """north_star's full-match wall time at c5: the whole 20 x 20 solve from X0 plus the greedy
    discretization (fastpfp_discretize) to a host assignment, inputs resident on the
    device (SURVEY 8(d) timing windows)."""
    import torch
    res = []
    for _ in range(2):
        s.set_x0(None if p.X0 is None else np.ascontiguousarray(p.X0[shard.sl if shard else slice(None)]))
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.iterate(p.alpha, p.lam, 0.0, 0.0, p.max_iter1, inner, want_x=False)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        assign = s.discretize()
        t2 = time.perf_counter()
        res.append((t2 - t0, t1 - t0, t2 - t1))
    wall, solve, disc = min(res)
    return {"wall_ms": round(max_over_ranks(wall * 1e3, world), 2), "solve_ms": round(solve * 1e3, 2),
            "discretize_ms": round(disc * 1e3, 2), "outer_iterations": p.max_iter1, "inner_sweeps": inner,
            "planted_recovery": float(np.mean(assign == p.perm)) if p.perm is not None else None,
            "what": "iterate(20 outer x 20 sweeps from X0) + fastpfp_discretize to a host assignment (wall clock)"}


def precision_line(p, prec, inner, steps, mp, src):
    """The same c5 step with another GEMM precision (north_star: 3xTF32, with plain TF32 reported
    separately; plain TF32 is NOT fp32-accurate)."""
    import torch

    import paper_1207_1114_b200 as F
    s = F.Solver(p.n, p.n_prime, p.d)
    stream = torch.cuda.current_stream()
    s.set_option(F.OPT_STREAM, stream.cuda_stream)
    s.set_option(F.OPT_PRECISION, prec)
    s.set_option(F.OPT_CHECK_EVERY, 64)
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    s.iterate(p.alpha, p.lam, 0.0, 0.0, 3, inner, want_x=False)
    s.set_option(F.OPT_PROFILE, 1)
    ms, clocks, st = timed_steps(s, p, inner, steps, 1, torch.cuda.current_device(), stream)
    s.close()
    r = gemm_roofline(mp, src, prec, st, ms / steps, clocks, False, True)
    return {"value": round(steps / (ms / 1e3), 4), "unit": UNIT, "steps": steps, "ms_per_step": round(ms / steps, 3),
            "gemm": {k: r[k] for k in ("kernel", "achieved", "peak", "frac", "ms_per_launch", "share_of_step",
                                       "vs_measured_pipe", "peak_source")},
            "clocks": clocks, "fp32_accurate": prec != 1}


def _pair_problem(name):
    from paper_1207_1114_b200 import inputs
    return {"c1": inputs.config1, "c2": inputs.config2, "c3": inputs.config3}[name]()


PAIR_DESC = {
    "c1": "c1 (BASELINE configs[0]): n=n'=64, ER p=0.3 U(0,1), exact planted isomorphism, lambda=0, X0=1/n ones, "
          "alpha=0.5, eps1=eps2=1e-6, I0=I1=100",
    "c3": "c3 (BASELINE configs[2]): n=800 vs n'=1000 (200 outliers), ER p=0.4, noise N(0,0.05^2), d=16, "
          "lambda=0.5, alpha=0.5, eps1=eps2=1e-4, I0=I1=300, slack rows persist",
}


def secondary_pair(name, method=0):
    """One BASELINE pair config solved to convergence (its eps / I caps) plus greedy discretization:
    outer iters/s of the solve and the full-match wall time (median of 4 runs)."""
    import torch

    import paper_1207_1114_b200 as F
    p = _pair_problem(name)
    s = F.Solver(p.n, p.n_prime, p.d)
    stream = torch.cuda.current_stream()
    s.set_option(F.OPT_STREAM, stream.cuda_stream)
    s.set_option(F.OPT_CHECK_EVERY, 8)
    s.set_option(F.OPT_METHOD, method)
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    s.set_x0(p.X0)
    res = []
    for _ in range(4):
        s.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, rep = s.iterate(p.alpha, p.lam, p.eps1, p.eps2, p.max_iter1, p.max_iter2, want_x=False)
        e1.record(stream)
        torch.cuda.synchronize()
        solve_ms = e0.elapsed_time(e1)
        assign = s.discretize()
        wall = time.perf_counter() - t0
        res.append((solve_ms, wall, rep))
    solve_ms, wall, rep = sorted(res, key=lambda r: r[0])[len(res) // 2]
    acc = float((assign == p.perm).mean())
    st = s.stats()
    s.close()
    desc = PAIR_DESC.get(name) or workload_desc(p, "c2")
    return {"workload": desc + (" [Projected Gradient {pg}, P:245-249]" if method else ""),
            "value": round(rep.iterations / (solve_ms / 1e3), 3),
            "unit": UNIT, "outer_iterations": rep.iterations, "total_sweeps": rep.total_sweeps,
            "converged": rep.converged,
            "solve_ms": round(solve_ms, 3), "full_match_wall_ms": round(wall * 1e3, 3),
            "planted_recovery": acc, "ms_per_sweep": round(solve_ms / max(rep.total_sweeps, 1), 5),
            "bound": "latency (L2/on-chip resident working set; one grid exchange per sweep)",
            "proj_kernel": (("on-chip tiles (%d CTAs, one tagged-record exchange per sweep, no grid barrier)"
                             % st["onchip_tiles"]) if st["onchip_tiles"] > 1 else
                            "on-chip, one CTA holds Y (no exchange)")
                           if st["onchip_launches"] else "streaming (2 grid barriers per sweep)",
            "paper_context": "a few seconds for 1000-node graphs on a 3 GHz Core2 PC in MATLAB (PAPER.md:33-34)"}


def secondary_c1_batched():
    """BASELINE configs[0] through the batched small-pair kernel as a batch of one (the whole solve
    in one CTA slot: products on the int8 tensor cores, sweeps in registers) — the
    path a caller with many or tiny pairs uses; the same problem, eps and caps as secondary_c1."""
    import torch

    import paper_1207_1114_b200 as F
    from paper_1207_1114_b200 import inputs
    p = inputs.config1()
    s = F.BatchedSolver(1, p.n, p.n_prime, 0)
    stream = torch.cuda.current_stream()
    s.set_option(F.OPT_STREAM, stream.cuda_stream)
    s.set_graphs(p.A[None], p.Ap[None])
    res = []
    for _ in range(4):
        s.set_x0(p.X0[None])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, rep = s.iterate(p.alpha, p.lam, p.eps1, p.eps2, p.max_iter1, p.max_iter2, want_x=False)
        e1.record(stream)
        torch.cuda.synchronize()
        solve_ms = e0.elapsed_time(e1)
        assign = s.discretize()
        res.append((solve_ms, (time.perf_counter() - t0) * 1e3, rep))
    solve_ms, wall_ms, rep = sorted(res, key=lambda r: r[0])[len(res) // 2]
    s.close()
    iters, sweeps = int(rep.iterations[0]), int(rep.sweeps[0])
    return {"workload": PAIR_DESC["c1"] + " [batched small-pair kernel, batch of one]",
            "value": round(iters / (solve_ms / 1e3), 3), "unit": UNIT, "outer_iterations": iters,
            "total_sweeps": sweeps, "converged": bool(rep.converged[0]), "solve_ms": round(solve_ms, 3),
            "full_match_wall_ms": round(wall_ms, 3), "planted_recovery": float(np.mean(assign[0] == p.perm)),
            "ms_per_sweep": round(solve_ms / max(sweeps, 1), 5)}


def secondary_ga():
    """FastGA at n = 1000 on the GA-scaled c2 recipe (inputs.ga_pair):
    full annealing run (beta 0.5 x 1.075^t <= 10, eps = 1e-4, <= 100 Sinkhorn sweeps) + greedy,
    next to FastPFP's c2 solve (the paper's speed comparison)."""
    import torch

    import paper_1207_1114_b200 as F
    from paper_1207_1114_b200 import inputs
    p = inputs.ga_pair(2, 1000, d=32, lam=1.0, p=0.5, sigma_e=0.05, eps1=1e-4, eps2=1e-4,
                       max_iter1=300, max_iter2=100)
    s = F.Solver(p.n, p.n_prime, p.d)
    stream = torch.cuda.current_stream()
    s.set_option(F.OPT_STREAM, stream.cuda_stream)
    s.set_option(F.OPT_CHECK_EVERY, 8)
    s.set_option(F.OPT_METHOD, F.METHOD_FASTGA)
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    res = []
    for _ in range(3):
        s.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, rep = s.iterate(0.0, p.lam, p.eps1, p.eps2, p.max_iter1, p.max_iter2, want_x=False)
        e1.record(stream)
        torch.cuda.synchronize()
        solve_ms = e0.elapsed_time(e1)
        assign = s.discretize()
        res.append((solve_ms, (time.perf_counter() - t0) * 1e3, rep))
    solve_ms, wall_ms, rep = sorted(res, key=lambda r: r[0])[1]
    s.close()
    return {"workload": "FastGA (Appendix {GAO3} + slack-padded Sinkhorn) on the c2 recipe with GA-scaled "
                        "weights, n=n'=1000, d=32, lambda=1, beta=0.5*1.075^t<=10, eps=1e-4, I1<=100",
            "value": round(rep.iterations / (solve_ms / 1e3), 3), "unit": UNIT,
            "outer_iterations": rep.iterations, "total_sweeps": rep.total_sweeps,
            "solve_ms": round(solve_ms, 3), "full_match_wall_ms": round(wall_ms, 3),
            "ms_per_sweep": round(solve_ms / max(rep.total_sweeps, 1), 5),
            "planted_recovery": float((assign == p.perm).mean())}


C4_N = 128
C4_BATCH = 8192


def c4_roofline(mp, src, pairs, steps, ms, clocks):
    """The batched kernel's products run on the int8 tensor cores (6 MMAs per fp32-accurate product):
    4 n^3 algorithmic flops per pair-iteration against the same derived int8 peak as the c5 GEMM.
    Its sweeps (what bounds it) are reported as `secondary` against the fp32 lanes: per element of a
    sweep P1 is 2 adds, P2 one max, and the row and column sums of the result 2 adds (5 fp32 ops)."""
    gflop = 4.0 * C4_N**3 * pairs * steps / 1e9
    achieved = gflop / (ms / 1e3) / 1e3
    peak, _, note = gemm_peak(mp, src, 3)
    pp = pipe_peak(3, clocks.get("sm_mhz"))
    sweep_ops = 5.0 * C4_N * C4_N * 20 * pairs * steps
    sweep_tops = sweep_ops / (ms / 1e3) / 1e12
    mhz = clocks.get("sm_mhz") or 1965.0
    alu_peak = SMS * 128 * mhz * 1e6 / 1e12
    return {"kernel": "small_solve_tc_kernel (two pairs per CTA: products on tcgen05 kind::i8 + sweeps on chip)",
            "bound": "tensor", "achieved": round(achieved, 2), "peak": round(peak, 1), "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": ncu_traffic("small_solve_tc_kernel"),
            "flops_rule": "4 n^3 per pair-iteration (the two products of P:387), n = 128",
            "peak_source": note,
            "vs_measured_pipe": None if pp is None else {"peak": round(pp, 1), "frac": round(achieved / pp, 4)},
            "note": "the 20 on-chip sweeps per outer iteration (P:388-391) are what bounds the kernel (DESIGN.md §8)",
            "secondary": {"what": "the sweeps: 5 fp32 ops per element (P1 2 adds, P2 1 max, row + column sums 2 adds), "
                                  "20 sweeps of n^2 per pair-iteration, whole kernel time",
                          "bound": "alu", "achieved": round(sweep_tops, 2), "unit": "Tops/s",
                          "peak": round(alu_peak, 1), "frac": round(sweep_tops / alu_peak, 4),
                          "peak_source": f"148 SMs x 128 fp32 lanes x median SM clock {mhz} MHz"}}


def secondary_c4(mp, src, solves=12):
    """BASELINE configs[3]: 8192 pairs of n = 128, fixed 20 outer x 20 sweeps (eps = 0), one pair per
    CTA (batched whole-solve kernel). `solves` back-to-back batch solves in one timed region (enough
    for >= 10 clock samples)."""
    import torch

    import paper_1207_1114_b200 as F
    from paper_1207_1114_b200 import inputs
    probs = inputs.config4(batch=C4_BATCH)
    A, Ap, _, _ = inputs.stack_pairs(probs)
    s = F.BatchedSolver(C4_BATCH, C4_N, C4_N, 0)
    stream = torch.cuda.current_stream()
    s.set_option(F.OPT_STREAM, stream.cuda_stream)
    s.set_graphs(A, Ap)
    s.iterate(0.5, 0.0, 0.0, 0.0, 3, 20, want_x=False)          # warm-up
    torch.cuda.synchronize()
    clk = Clocks(torch.cuda.current_device(), 25)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(solves):
        s.set_x0(None)
        _, rep = s.iterate(0.5, 0.0, 0.0, 0.0, 20, 20, want_x=False)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    assign = s.discretize()
    acc = float(np.mean([np.array_equal(assign[k], probs[k].perm) for k in range(C4_BATCH)]))
    s.close()
    return {"workload": f"c4 (BASELINE configs[3]): {C4_BATCH} pairs n=n'=128, ER p=0.3, noise N(0,0.02^2), "
                        f"lambda=0, fixed 20 outer x 20 sweeps, one pair per CTA",
            "value": round(C4_BATCH * 20 * solves / (ms / 1e3), 1), "unit": "pair_outer_iters/s",
            "solve_ms": round(ms / solves, 3), "solves_timed": solves, "sweeps_per_pair": int(rep.sweeps[0]),
            "planted_recovery_pairs": acc, "roofline": c4_roofline(mp, src, C4_BATCH, 20 * solves, ms, clocks),
            "clocks": clocks}


def run_c4(args):
    """--workload c4 (BASELINE configs[3]): 8192 pairs of n = 128 split evenly over the ranks (pair
    data parallelism, no collective on the path; configs[3] "pairs split evenly over 1/2/4/8 GPUs").
    A step = one outer iteration (20 sweeps) of every pair; value = pairs * steps / max-over-ranks
    time (strong scaling of the fixed batch)."""
    import torch

    import paper_1207_1114_b200 as F
    from paper_1207_1114_b200 import inputs

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    maybe_init_pg(world, "nccl")
    mp, src = load_peaks()
    per = C4_BATCH // world
    first = rank * per
    count = per if rank < world - 1 else C4_BATCH - first
    probs = inputs.config4(batch=C4_BATCH, first=first, count=count)
    A, Ap, _, _ = inputs.stack_pairs(probs)
    s = F.BatchedSolver(count, C4_N, C4_N, 0)
    stream = torch.cuda.current_stream()
    s.set_option(F.OPT_STREAM, stream.cuda_stream)
    s.set_graphs(A, Ap)
    s.iterate(0.5, 0.0, 0.0, 0.0, max(args.warmup, 1), 20, want_x=False)
    s.set_x0(None)
    barrier(world)
    torch.cuda.synchronize()
    clk = Clocks(local, 25)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _, rep = s.iterate(0.5, 0.0, 0.0, 0.0, args.steps, 20, want_x=False)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clocks = clk.stop()
    ms_local = e0.elapsed_time(e1)
    ms = max_over_ranks(ms_local, world)
    st = s.stats()
    assign = s.discretize()
    acc = float(np.mean(np.all(assign == np.stack([p.perm for p in probs]), axis=1)))
    out = {"metric": METRIC, "value": round(C4_BATCH * args.steps / (ms / 1e3), 1), "unit": "pair_outer_iters/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": "c4 (BASELINE configs[3]): 8192 pairs n=n'=128, ER p=0.3, noise N(0,0.02^2), "
                                  "lambda=0, 20 sweeps per outer, one pair per CTA, pairs split evenly over ranks",
                      "parallelism": f"pairs/{world}", "l2": "per-pair working set on chip; inputs 1 GB"},
           "roofline": c4_roofline(mp, src, count, args.steps, ms_local, clocks),
           "clocks": clocks, "gpu_launches": int(st["launches"]), "planted_recovery_pairs_rank0": acc}
    s.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    finish_pg(world)


# ------------------------------------------------------------------------------------------------
# the oracle, timed (cpu_baseline and --impl reference)
# ------------------------------------------------------------------------------------------------
def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count()


def oracle_state(p):
    from oracle import fastpfp as O
    return O.FastPFP(p.A, p.Ap, p.B, p.Bp, p.X0)


def oracle_outer_sample(st, p, inner, sample_sweeps):
    """One oracle outer iteration of problem p at its FULL size (Algorithm 1 lines 3-9 with the
    oracle's own functions), with `sample_sweeps` of the `inner` sweeps actually run and the sweep
    time scaled to `inner` (every sweep of the fixed schedule is the same O(m^2) work).
    Returns (seconds per outer iteration, detail)."""
    from oracle import fastpfp as O
    t0 = time.perf_counter()
    G = O.gradient(st.A, st.Ap, st.K, st.X, p.lam)                       # line 3 (two n^3 products)
    t1 = time.perf_counter()
    st.Y[:p.n, :p.n_prime] = G
    del G
    Y, _, _ = O.project_loop(st.Y, 0.0, sample_sweeps)                  # lines 4-7, sampled
    t2 = time.perf_counter()
    Xt = (1 - p.alpha) * st.X + p.alpha * Y[:p.n, :p.n_prime]           # lines 8-9
    X = Xt / Xt.max()
    t3 = time.perf_counter()
    del Y, Xt, X
    per = (t1 - t0) + (t2 - t1) * inner / sample_sweeps + (t3 - t2)
    return per, {"products_s": round(t1 - t0, 2), "sweep_s": round((t2 - t1) / sample_sweeps, 2),
                 "finalize_s": round(t3 - t2, 2)}


def cpu_baseline(workload, p):
    """The fp64 oracle as it stands on the host cores, at the bench's own problem size: c5 one outer
    iteration at n = 16384 with 2 of the 20 sweeps run (the sweep time scaled by 10); c2 one outer
    iteration at n = 1000 (all 20 sweeps)."""
    inner = p.max_iter2 if workload == "c5" else 20
    sample = 2 if workload == "c5" else inner
    per, detail = oracle_outer_sample(oracle_state(p), p, inner, sample)
    return {"value": round(1.0 / per, 6), "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
            "sample": (f"1 oracle outer iteration of the {workload} workload at its full size (n={p.n}): "
                       f"the two fp64 products, {sample} of the {inner} projection sweeps (time scaled to "
                       f"{inner}) and the blend + rescale"),
            "s_per_outer": round(per, 2), **detail}


def reference_config(workload):
    """The workload description our arm prints in its config, plus what ran."""
    from paper_1207_1114_b200 import inputs
    if workload == "c4":
        cfg = {"workload": ("c4 (BASELINE configs[3]): 8192 pairs n=n'=128, ER p=0.3, noise N(0,0.02^2), "
                            "lambda=0, 20 sweeps per outer, one pair per CTA, pairs split evenly over ranks")}
    elif workload == "c5":
        p = inputs.config5(n=64)   # the recipe's scalars (lambda, alpha, sweeps); sizes are c5's
        cfg = {"workload": workload_desc(p, "c5").replace("n=n'=64", "n=n'=16384"),
               "n": 16384, "n_prime": 16384, "d": p.d, "inner_sweeps": p.max_iter2}
    else:
        p = inputs.config2()
        cfg = {"workload": (f"c2 problem (BASELINE configs[1] recipe: n=n'={p.n}, d={p.d}, ER p=0.5, "
                            f"lambda={p.lam}, alpha={p.alpha}) on c5's fixed schedule: eps = 0, 20 sweeps per "
                            f"outer"),
               "n": p.n, "n_prime": p.n_prime, "d": p.d, "inner_sweeps": 20}
    cfg["reference"] = "fp64 numpy oracle (oracle/) on host cores, bounded sample of the workload"
    return cfg


def run_reference(args):
    """The oracle timed as the reference arm. c5: each step is one full-size (n = 16384) oracle
    outer iteration with 1 of its 20 sweeps run (scaled by 20); warm-up steps run one full-size
    sweep only (the products need no warm-up). c2: full outer iterations (20 sweeps). c4: one outer
    iteration of 64 of the 8192 pairs, scaled to the batch."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import fastpfp as O
    from paper_1207_1114_b200 import inputs
    cores = blas_threads()
    per_step = []
    if args.workload == "c4":
        probs = inputs.config4(first=0, count=64)
        states = [O.FastPFP(q.A, q.Ap) for q in probs]
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            for st in states:
                st.iterate(0.0, 0.5, 0.0, 0.0, 1, 20)
            if k >= args.warmup:
                per_step.append((time.perf_counter() - t0) * C4_BATCH / 64)
        sample = "per step: one oracle outer iteration (20 sweeps) of 64 of the 8192 c4 pairs, scaled to the batch"
        units, unit = C4_BATCH, "pair_outer_iters/s"
    else:
        p = make_problem(args.workload)
        inner = p.max_iter2 if args.workload == "c5" else 20
        sweeps = 1 if args.workload == "c5" else inner
        st = oracle_state(p)
        if args.workload == "c5":
            for _ in range(args.warmup):
                O.sweep(st.Y)
        else:
            for _ in range(args.warmup):
                oracle_outer_sample(st, p, inner, sweeps)
        for _ in range(args.steps):
            per_step.append(oracle_outer_sample(st, p, inner, sweeps)[0])
        sample = (f"per step: one oracle outer iteration of {args.workload} at its full size (n={p.n}): the two fp64 "
                  f"products, {sweeps} of the {inner} sweeps (time scaled to {inner}), blend + rescale")
        units, unit = 1, UNIT
    total = sum(per_step)
    value = units * args.steps / total
    out = {"metric": METRIC, "value": round(value, 6), "unit": unit, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": reference_config(args.workload),
           "cpu_baseline": {"value": round(value, 6), "unit": unit, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": round(value, 6), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------------
# launcher self-test (CPU, gloo, no kernels): the multi-rank plumbing the GPU run uses
# ------------------------------------------------------------------------------------------------
def run_launcher_selftest(args):
    world, rank, _ = dist_env()
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group(backend="gloo")
    barrier(world)
    t = max_over_ranks(float(rank + 1), world)
    if rank == 0:
        print(json.dumps({"selftest": True, "n_gpus": world, "gpus_arg": args.gpus, "max_over_ranks": t}),
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c5", "c2", "c4"])
    ap.add_argument("--precision", type=int, default=None,
                    help="GEMM precision (FASTPFP_OPT_PRECISION); default: the library's (int8 Ozaki)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--launcher-selftest", action="store_true", help=argparse.SUPPRESS)
    # run c5 through the row-sharded handle even on one rank (exercises the multi-GPU code path of
    # this script — shard inputs, e2e, full match — on a single GPU)
    ap.add_argument("--force-shard", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(argv, args.gpus))
    if args.warmup < 3 and args.impl == "ours":
        print("warning: timing rules require >= 3 warm-up steps", file=sys.stderr)
    if args.launcher_selftest:
        run_launcher_selftest(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.workload == "c4":
        run_c4(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
