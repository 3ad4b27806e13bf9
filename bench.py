#!/usr/bin/env python
"""Benchmark of the B200 hot path of the N-D Bartels–Stewart solver (BASELINE.json).

One step = one full solve of the workload's Sylvester equation on the GPU: forward transform
(N mode products with U_j^H), blocked triangular solve, inverse transform (N mode products
with U_j). The host Schur factorisations are setup, computed once and timed separately
(BASELINE.md 2). Metric: unknowns/s = P / step time (P = prod n_j).

  value   device-resident: B already in HBM, K steps timed with CUDA events (max over ranks);
  e2e     through the C-ABI host-buffer call nds_solve_schur (the reference-facing drop-in for
          ndsylv::solve after its Schur step) from pinned host memory: plan creation + singular
          check + H2D(B) + solve + D2H(X) inside the timed region every step;
  roofline  dominant kernel (complex-FP64 DMMA mode-product GEMM), algorithmic FLOPs per launch
          (8 P n_j, one CMAC = 8 real flops) over its CUDA-event launch time, against the FP64
          DMMA peak measured on this pool (profiles/fp64_peaks_r01.json);
  cpu_baseline  the reference CPU solver (oracle/_ref, built from /root/reference sources) on a
          bounded slab sample of the same workload, rank 0 at N=1 only.

--impl reference runs the reference's own CPU solver (oracle/_ref) the same way.
Multi-GPU (torchrun, --gpus N > 1): ONE c3 problem sharded across the ranks by the C-ABI engine
(nds_dist_*; strong scaling, NCCL); --replicas runs independent copies instead (weak scaling).
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

METRIC = "unknowns/s (prod n_j/s), complex128"
DEFAULT_CONFIG = "c1"  # configs[1] of BASELINE.json: N=3, n=256, 16.8M unknowns (fits one GPU)


def fp64_peak():
    path = os.path.join(ROOT, "profiles", "fp64_peaks_r01.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["dmma_tflops_sustained"]), "measured on this pool: DMMA m8n8k4 microbenchmark (" + \
            os.path.relpath(path, ROOT) + ")"
    except Exception:
        return 37.2, "nominal 148 SM x 64 FMA/clk x 2 x 1.965 GHz (no measured file)"


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
    except Exception:
        return 6507.2, "B200_PROFILING.md fallback (no MEASURED_PEAKS.json)"


def ncu_traffic(config):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(config)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[4 + i].lower() == "active"})
        pw = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "power_w_max": max(pw) if pw else None, "samples": len(self.samples)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if os.environ.get("NDS_BENCH_BACKEND", "nccl") == "nccl" else "gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, value, device=None):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def bench_config(config, world, parallelism=None):
    """The `config` object of the JSON line — identical for our arm and the reference arm."""
    from paper_2412_15840_b200 import configs  # the module itself loads no native library
    dims = configs.CONFIGS[config]["dims"]
    return {"workload": config, "dims": list(dims), "P": int(np.prod(dims)),
            "description": configs.DESCRIPTIONS[config],
            "parallelism": parallelism or (f"replicas x{world}" if world > 1 else "1 GPU"),
            "l2": (f"inputs larger than L2 ({16 * int(np.prod(dims)) / 2**20:.0f} MiB per tensor vs 126 MB L2); no flush"
                   if 16 * int(np.prod(dims)) > 126e6 else "inputs fit in L2; no flush (not a headline config)"),
            "schur": "host setup, excluded from the rate (BASELINE.md 2)"}


# Bounded samples of the reference CPU solve for the configs whose full solve takes many minutes
# (c3: ~12 min, c4: ~9 min, c2: ~2 min on 8 cores): the leading planes of the
# workload (same extents in every other mode, same generator).
REF_SAMPLE_DIMS = {"c2": (96, 96, 96, 8), "c3": (128, 128, 128, 2), "c4": (2,) * 23}


class ReferenceStages:
    """The reference's own CPU solve stages (oracle/_ref: the unmodified ndsylv library built from
    /root/reference/proj/src): forward_transform, back_substitute and inverse_transform
    (sylvester.hpp:64-77) with the Schur factors from its own schur() (setup, timed separately,
    like ndsylv::solve's SolveReport::schur_seconds), on the FULL workload for c0 / c1 and on the
    bounded sample REF_SAMPLE_DIMS otherwise. Inputs come from the generator-v1 copy in the
    reference shim, so the product library is never loaded."""

    def __init__(self, config, seed, threads):
        import oracle
        from paper_2412_15840_b200 import configs
        self.ref = oracle.Ref()
        self.ref.set_threads(threads)
        self.sample_dims = REF_SAMPLE_DIMS.get(config)
        self.a, self.b = configs.make_problem(config, seed=seed, dims=self.sample_dims, randn=self.ref.randn)
        self.P = int(self.b.size)
        t0 = time.perf_counter()
        fac = [self.ref.schur(m) for m in self.a]
        self.schur_s = time.perf_counter() - t0
        self.us = [f[0] for f in fac]
        self.ts = [f[1] for f in fac]

    def step(self):
        """One solve (forward, back-substitution, inverse); returns (seconds, stage seconds)."""
        t0 = time.perf_counter()
        c = self.ref.forward_transform(self.us, self.b)
        t1 = time.perf_counter()
        y, _ = self.ref.back_substitute(self.ts, c)
        t2 = time.perf_counter()
        x = self.ref.inverse_transform(self.us, y)
        t3 = time.perf_counter()
        self.x = x
        return t3 - t0, {"transform_seconds": t1 - t0, "backsub_seconds": t2 - t1, "inverse_seconds": t3 - t2}


def reference_sample_text(config, threads):
    d = REF_SAMPLE_DIMS.get(config)
    what = f"the full {config} workload" if d is None else \
        f"a bounded sample of {config}: its leading planes {'x'.join(map(str, d))} (P = {int(np.prod(d))})"
    return (f"reference ndsylv stages (oracle/_ref, unmodified sources, g++ -O3 -fopenmp, no -march; "
            f"OpenMP over {threads} threads in the transforms, back_substitute serial by construction, "
            f"sylvester.cpp:71-108) on {what}; rate = P / (forward + backsub + inverse wall seconds); "
            f"Schur excluded (setup)")


def verify_x(ctx, config, seed, a_list, dims, d_x, d_b):
    """Correctness of the X the timed steps produced: the device relative residual (north_star
    <= 1e-10) and, for seed 0, X at the sampled entries of the reference's X_ref fixture
    (tests/golden/xref_<cfg>.npz, made by the unmodified reference solver; <= 1e-9)."""
    import torch
    out = ctx.dev_residual(a_list, dims, d_x.data_ptr(), d_b.data_ptr())
    out = {k: out[k] for k in ("rel_res_2", "rel_res_max") if k in out}
    path = os.path.join(ROOT, "tests", "golden", f"xref_{config}.npz")
    if seed == 0 and os.path.exists(path):
        fx = np.load(path)
        x_s = d_x[torch.from_numpy(fx["idx"]).to(d_x.device)].cpu().numpy()
        out["xref_rel_max_sampled"] = float(np.max(np.abs(x_s - fx["x"])) / float(fx["xmax"]))
        out["xref_samples"] = int(fx["idx"].size)
    out["ok"] = bool(out.get("rel_res_2", 1.0) <= 1e-10 and out.get("rel_res_max", 1.0) <= 1e-10 and
                     out.get("xref_rel_max_sampled", 0.0) <= 1e-9)
    return out


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    sharded = world > 1 and not args.replicas
    if sharded and "--config" not in sys.argv:
        args.config = "c3"  # the same workload as our arm's sharded default
    threads = os.cpu_count() or 1
    rs = ReferenceStages(args.config, args.seed, threads)
    secs, stages = [], []
    for i in range(args.warmup + args.steps):
        s, st = rs.step()
        if i >= args.warmup:
            secs.append(s)
            stages.append(st)
    mean_s = statistics.mean(secs)
    value = rs.P / mean_s
    line = {"metric": METRIC, "value": value, "unit": "unknowns/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": mean_s * 1e3, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (generator v1, seeded Gaussian)",
            "impl": "reference",
            "config": bench_config(args.config, world,
                                   parallelism=f"sharded x{world} (nds_dist, NCCL)" if sharded else None),
            "cpu_baseline": {"value": value, "unit": "unknowns/s", "cores": threads, "kind": "reference",
                             "sample": reference_sample_text(args.config, threads)},
            "e2e": {"value": value, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "stage_seconds_mean": {k: statistics.mean(st[k] for st in stages) for k in stages[0]},
            "schur_seconds_host": rs.schur_s}
    print(json.dumps(line), flush=True)
    return 0


def run_sharded(args, world, rank, local):
    """ONE problem split across the ranks (strong scaling) through the C-ABI sharded engine
    (nds_dist_*, csrc/sharded.cuh): transforms local in L_N / L_1 with one NCCL
    all-to-all each way, triangular solve pipelined over (rank, block of the last modes) with
    point-to-point forwarding — all on the ranks' own streams, no host sync inside a solve.
    value = P / (max-over-ranks device time per solve). The default for --gpus N > 1 (config c3);
    rank 0 also times the single-GPU plan path on the same config for reference."""
    import torch
    import torch.distributed as dist
    import paper_2412_15840_b200 as nds
    from paper_2412_15840_b200 import configs
    from paper_2412_15840_b200.distributed import Comm, ShardedSolver, plan_layout

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = nds.Context(local)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    a_list, b_host = configs.make_problem(args.config, seed=args.seed)
    dims = tuple(b_host.shape)
    P = int(np.prod(dims))
    t0 = time.perf_counter()
    factors = [ctx.schur(a) for a in a_list]
    schur_s = time.perf_counter() - t0
    us = [f[0] for f in factors]
    ts = [f[1] for f in factors]
    single = None
    if rank == 0 and not args.no_single:  # the 1-GPU plan path on the same workload, for the scaling context
        plan = ctx.plan(us, ts)
        d_b = torch.from_numpy(np.ascontiguousarray(b_host.ravel(order="F"))).to(dev)
        d_x, d_w = torch.empty_like(d_b), torch.empty_like(d_b)
        for _ in range(2):
            plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms1 = e0.elapsed_time(e1) / 3
        single = {"ms_per_solve": ms1, "unknowns_per_s": P / (ms1 * 1e-3)}
        del plan, d_b, d_x, d_w
        torch.cuda.empty_cache()
    comm = Comm.nccl(local) if world > 1 else None
    solver = ShardedSolver(ctx, us, ts, comm)
    off, cnt = solver.slab(rank)
    flat = np.ascontiguousarray(b_host.reshape(-1, order="F")[off:off + cnt])
    del b_host
    d_b = torch.from_numpy(flat).to(dev)
    d_x = torch.empty_like(d_b)
    for _ in range(args.warmup):
        solver.solve(d_b, d_x)
    torch.cuda.synchronize(dev)
    barrier(world)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            solver.solve(d_b, d_x)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    barrier(world)
    ms_step = max_over_ranks(world, e0.elapsed_time(e1), dev) / args.steps
    info = solver.info()
    L = plan_layout(dims, world)
    verify = None
    if not args.no_verify:  # X at the X_ref fixture's samples that fall in this rank's slab
        path = os.path.join(ROOT, "tests", "golden", f"xref_{args.config}.npz")
        if args.seed == 0 and os.path.exists(path):
            fx = np.load(path)
            sel = (fx["idx"] >= off) & (fx["idx"] < off + cnt)
            x_s = d_x[torch.from_numpy(fx["idx"][sel] - off).to(dev)].cpu().numpy()
            err = float(np.max(np.abs(x_s - fx["x"][sel]))) / float(fx["xmax"]) if sel.any() else 0.0
            verify = {"xref_rel_max_sampled": max_over_ranks(world, err, dev), "ok": None}
            verify["ok"] = verify["xref_rel_max_sampled"] <= 1e-9
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": P / (ms_step * 1e-3), "unit": "unknowns/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128 (fp64 DMMA)",
            "data": "synthetic (generator v1, seeded Gaussian)",
            "config": bench_config(args.config, world, parallelism=f"sharded x{world} (nds_dist, NCCL)"),
            "schur_seconds_host": schur_s,
            "sharding": {"head_modes": info["head_modes"], "tail_modes": info["tail_modes"],
                         "pipe_modes": info["pipe_modes"], "pipe_blocks": info["pipe_blocks"],
                         "local_solve_path": nds.Plan.SOLVE_PATHS.get(info["local_solve_path"]),
                         "nvlink_bytes_per_solve_rank0": {"alltoall": L.alltoall_bytes(0),
                                                          "pipeline": L.pipeline_bytes(0)},
                         "nvlink_bytes_per_solve_max_rank": max(L.alltoall_bytes(r) + L.pipeline_bytes(r)
                                                                for r in range(world))},
            "single_gpu_plan_same_config": single,
            "roofline": None, "cpu_baseline": None, "e2e": None,
            "gpu_launches": info["launches"] * args.steps, "launches_per_step": info["launches"],
            "clocks": clk.summary(), "verify": verify}), flush=True)
    solver.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=["c0", "c1", "c2", "c3", "c4"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-verify", action="store_true",
                    help="skip the correctness stamp of the timed X (device residual + X_ref samples)")
    ap.add_argument("--sharded", action="store_true",
                    help="one problem split across the ranks (the default for --gpus N > 1; at N = 1 the same engine "
                         "on one rank)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas of the workload, one per rank (weak scaling)")
    ap.add_argument("--no-single", action="store_true", help="sharded mode: skip the 1-GPU plan reference timing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world, rank, local = dist_init()
    if args.impl == "reference":
        return run_reference(args, world, rank)

    if args.sharded or (world > 1 and not args.replicas):
        if world > 1 and args.config == DEFAULT_CONFIG and "--config" not in sys.argv:
            args.config = "c3"  # the sharded headline (BASELINE.json configs[3]: 1/2/4/8 B200)
        return run_sharded(args, world, rank, local)

    import torch
    import paper_2412_15840_b200 as nds
    from paper_2412_15840_b200 import configs

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = nds.Context(local)
    # A dedicated stream: torch's legacy default stream has handle 0, which the C ABI reads as
    # "use the context's own stream". Kernels and the timing events share this stream.
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    # --- inputs (host, generator v1) and host Schur setup -------------------------------------
    a_list, b_host = configs.make_problem(args.config, seed=args.seed + rank)
    dims = tuple(b_host.shape)
    P = int(np.prod(dims))
    t0 = time.perf_counter()
    factors = [ctx.schur(a) for a in a_list]
    schur_s = time.perf_counter() - t0
    us = [f[0] for f in factors]
    ts = [f[1] for f in factors]
    plan = ctx.plan(us, ts)

    flat = np.ascontiguousarray(b_host.ravel(order="F"))
    pinned_b = torch.from_numpy(flat).pin_memory()
    pinned_x = torch.empty_like(pinned_b).pin_memory()
    d_b = pinned_b.to(dev, non_blocking=True)
    d_x = torch.empty_like(d_b)
    d_w = torch.empty_like(d_b)
    torch.cuda.synchronize(dev)

    # --- device-resident timing ----------------------------------------------------------------
    for _ in range(args.warmup):
        plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
    torch.cuda.synchronize(dev)
    launches_per_step = plan.launches()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize(dev)
    barrier(world)
    ms_total = e0.elapsed_time(e1)
    ms_total = max_over_ranks(world, ms_total, dev)
    ms_step = ms_total / args.steps
    value = world * P / (ms_step * 1e-3)

    # --- per-launch profile of the same workload (separate pass, CUDA events per launch) -----
    plan.profile_begin(2 * (launches_per_step + 4) * args.steps + 8)  # launches + the library's stage markers
    for _ in range(args.steps):
        plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
    recs = plan.profile_end()
    by_kind = {}
    for kind, mode, ms in recs:
        by_kind.setdefault(kind, []).append((mode, ms))
    gemm = by_kind.get("transform_gemm", [])
    passes = by_kind.get("transform_direct", [])
    peak_tf, peak_src = fp64_peak()
    roofline = None
    if gemm:
        flops = [8.0 * P * dims[abs(m) - 1] for m, _ in gemm]
        avg_ms = sum(ms for _, ms in gemm) / len(gemm)
        achieved = sum(flops) / sum(ms for _, ms in gemm) / 1e9  # TFLOP/s (flop/ms / 1e9)
        traffic = ncu_traffic(args.config)
        roofline = {"bound": "tensor", "pipe": "FP64 DMMA (mma.sync.m8n8k4.f64)",
                    "kernel": "zgemm_tma_kernel (modes >= 2, bulk-copy fed) / zgemm_tmap_colm_kernel (mode 1, tensor-map TMA)",
                    "achieved": round(achieved, 3), "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": round(achieved / peak_tf, 4), "traffic": traffic,
                    "flops_per_launch": flops[0], "avg_launch_ms": avg_ms,
                    "peak_source": peak_src,
                    "algorithmic": "8 P n_j real flops per mode pass (1 CMAC = 8 flops)",
                    # the kernel multiplies complex numbers with 3 real products (3M), so it executes
                    # 6 of the 8 algorithmic flops per CMAC: the tensor pipe itself runs at pipe_frac
                    "pipe_frac": round(achieved * 0.75 / peak_tf, 4)}
    elif passes:  # all-binary (c4): the fused binary passes are HBM-bound
        hbm, hbm_src = hbm_peak()
        avg_ms = sum(ms for _, ms in passes) / len(passes)
        achieved = 2.0 * 16 * P / (avg_ms * 1e-3) / 1e9  # GB/s
        roofline = {"bound": "hbm", "kernel": "binary_pass_kernel (fused runs of up to 9 binary modes, unit-diagonal butterflies)",
                    "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                    "traffic": ncu_traffic(args.config), "bytes_per_launch": 2.0 * 16 * P, "avg_launch_ms": avg_ms,
                    "peak_source": hbm_src, "algorithmic": "2 x 16 P bytes per fused pass (read + write once)"}
    step_ms_prof = sum(ms for _, _, ms in recs) / args.steps
    stage_ms = {k: sum(ms for _, ms in v) / args.steps for k, v in by_kind.items()}
    # algorithmic work of the solve: Eq. (9) has sum_j (n_j - 1) / 2 CMACs per entry; on the
    # block-diagonalised route (super-blocks D_j) only the couplings across super-blocks remain,
    # sum_j (n_j - D_j) / 2 per entry (all of it on the FP64 tensor pipe), plus the division
    sb_levels, sb_d = plan.superblocks()
    if sb_d:
        solve_flops = 8.0 * P * sum(n - d for n, d in zip(dims, sb_d)) / 2 + 8.0 * P
    else:
        solve_flops = 8.0 * P * (sum(dims) - len(dims)) / 2 + 8.0 * P
    solve_ms = stage_ms.get("solve_level", 0.0) + stage_ms.get("solve_persistent", 0.0)
    diag_taken, diag_cond = plan.diagonalised()
    kernels = {
        "solve_route": {"diagonalised": diag_taken, "cond_bound": diag_cond, "superblocks": sb_d,
                        "levels": sb_levels or None},
        "transform_gemm_share": stage_ms.get("transform_gemm", 0.0) / step_ms_prof if step_ms_prof else None,
        "stage_ms_per_step": {k: round(v, 4) for k, v in stage_ms.items()},
        "solve_tflops": solve_flops / (solve_ms * 1e-3) / 1e12 if solve_ms else None,
        "solve_frac_fp64": (solve_flops / (solve_ms * 1e-3) / 1e12) / peak_tf if solve_ms else None,
    }
    # every kernel class of the step against its roofline (north_star: "each kernel's achieved
    # HBM GB/s or FP64 FLOP/s as a fraction of B200 peak"), from the per-launch CUDA events
    hbm, hbm_src = hbm_peak()
    per_kernel = []
    if gemm:
        g_ms = sum(ms for _, ms in gemm) / args.steps
        g_fl = sum(8.0 * P * dims[abs(m) - 1] for m, _ in gemm) / args.steps
        per_kernel.append({"kernel": "transform GEMM (zgemm_tma / zgemm_tmap_colm)", "launches_per_step": len(gemm) // args.steps,
                           "ms_per_step": round(g_ms, 4), "achieved": round(g_fl / (g_ms * 1e-3) / 1e12, 3),
                           "unit": "TFLOP/s", "peak": peak_tf, "frac": round(g_fl / (g_ms * 1e-3) / 1e12 / peak_tf, 4),
                           "bound": "FP64 tensor (DMMA)"})
    if passes:
        p_ms = sum(ms for _, ms in passes) / args.steps
        p_by = 32.0 * P * (len(passes) // args.steps)
        per_kernel.append({"kernel": "binary_pass_kernel (fused binary modes)", "launches_per_step": len(passes) // args.steps,
                           "ms_per_step": round(p_ms, 4), "achieved": round(p_by / (p_ms * 1e-3) / 1e9, 1),
                           "unit": "GB/s", "peak": hbm, "frac": round(p_by / (p_ms * 1e-3) / 1e9 / hbm, 4),
                           "bound": "HBM"})
    levels = by_kind.get("solve_level", [])
    if levels and all(n == 2 for n in dims):  # the fused all-binary tile kernel: one read + one write
        f_ms = sum(ms for _, ms in levels) / args.steps
        # algorithmic flops: 24 mode passes of 8 P n_j + the solve's; the kernel executes about half of
        # them (unit-diagonal butterflies: 4 FMAs per output; diagonalised modes: no couplings)
        f_fl = 24 * 16.0 * P + solve_flops
        per_kernel.append({"kernel": "binary_fused_round_kernel (modes 1-12 fwd + tile solve + inv, persistent)",
                           "launches_per_step": len(levels) // args.steps, "ms_per_step": round(f_ms, 4),
                           "achieved": round(32.0 * P / (f_ms * 1e-3) / 1e9, 1), "unit": "GB/s", "peak": hbm,
                           "frac": round(32.0 * P / (f_ms * 1e-3) / 1e9 / hbm, 4), "bound": "FP64 pipe (DFMA) / HBM",
                           "algorithmic_tflops": round(f_fl / (f_ms * 1e-3) / 1e12, 2), "fp64_peak_tflops": peak_tf,
                           "frac_fp64_algorithmic": round(f_fl / (f_ms * 1e-3) / 1e12 / peak_tf, 4)})
    elif solve_ms:
        per_kernel.append({"kernel": "blk_level_kernel (block-diagonalised solve)" if sb_d else
                           "solve (wavefront route: tile_diag_lines + far_group)",
                           "launches_per_step": (len(levels) // args.steps) if levels else None,
                           "ms_per_step": round(solve_ms, 4), "achieved": round(solve_flops / (solve_ms * 1e-3) / 1e12, 3),
                           "unit": "TFLOP/s", "peak": peak_tf,
                           "frac": round(solve_flops / (solve_ms * 1e-3) / 1e12 / peak_tf, 4),
                           "bound": "FP64 tensor (DMMA)"})
    kernels["per_kernel"] = per_kernel

    # --- end to end through the C-ABI host-buffer call -----------------------------------------
    e2e = None
    if not args.no_e2e:
        import ctypes as C
        lib = ctx.lib
        up, ku = nds._ptr_array(us)
        tp, kt = nds._ptr_array(ts)
        dims_c = nds._dims(dims)
        rep = nds._Report()
        sing = nds._Singular()
        def e2e_call(hb, hx):
            rc = lib.nds_solve_schur(ctx.h, len(dims), dims_c, up, tp, hb, hx, 0.0, nds.ALLOW_FAST_PATH,
                                     C.byref(rep), C.byref(sing))
            if rc:
                raise RuntimeError(ctx.last_error())

        def timed(hb, hx):
            for _ in range(2):
                e2e_call(hb, hx)
            barrier(world)
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                e2e_call(hb, hx)
            return max_over_ranks(world, (time.perf_counter() - t0) / args.e2e_steps, dev)

        # the drop-in case: PAGEABLE buffers, as ndsylv::NDTensor's std::vector storage arrives
        # through the adapter (staged by the library through its pinned ring)
        page_b = np.ascontiguousarray(flat)
        page_x = np.empty_like(page_b)
        pg_s = timed(page_b.ctypes.data, page_x.ctypes.data)
        pg_rep = {"h2d_ms": rep.h2d_seconds * 1e3, "d2h_ms": rep.d2h_seconds * 1e3}
        e2e_s = timed(pinned_b.data_ptr(), pinned_x.data_ptr())
        pg_ok = bool(np.array_equal(page_x, pinned_x.numpy()))  # same X bitwise either way
        e2e = {"value": world * P / e2e_s, "unit": "unknowns/s", "h2d_bytes_per_step": 16 * P,
               "d2h_bytes_per_step": 16 * P, "ms_per_step": e2e_s * 1e3, "steps": args.e2e_steps,
               "api": "nds_solve_schur (host buffers, pinned)",
               "h2d_ms": rep.h2d_seconds * 1e3, "d2h_ms": rep.d2h_seconds * 1e3,
               "device_ms": (rep.transform_seconds + rep.backsub_seconds + rep.inverse_seconds) * 1e3,
               "stages_ms": {"h2d_stream": rep.h2d_seconds * 1e3,
                             "forward_incl_h2d": rep.transform_seconds * 1e3,
                             "solve": rep.backsub_seconds * 1e3,
                             "inverse": rep.inverse_seconds * 1e3,
                             "d2h_tail": rep.d2h_seconds * 1e3},
               "pageable": {"value": world * P / pg_s, "ms_per_step": pg_s * 1e3,
                            "api": "nds_solve_schur (host buffers, pageable: std::vector storage of the "
                                   "reference's NDTensor, staged through the library's pinned ring)",
                            "stages_ms": pg_rep, "x_equals_pinned_run": pg_ok}}
        # streamed right-hand sides (nds_plan_execute_host_many): M solves of the same operator
        # through ONE plan whose creation is inside the timed region; the H2D of b[k+1] and the
        # D2H of x[k-1] run under solve k (two pinned B / X buffers alternate, each step copies
        # its full B in and its full X out)
        if world == 1:
            M = max(args.steps, 4)
            pb = [pinned_b, pinned_b.clone().pin_memory()]
            px = [pinned_x.clone().pin_memory(), torch.empty_like(pinned_b).pin_memory()]
            hb = [pb[k % 2].data_ptr() for k in range(M)]
            hx = [px[k % 2].data_ptr() for k in range(M)]
            warm = ctx.plan(us, ts)
            warm.execute_host_many(hb[:4], hx[:4])
            warm.close()
            t0 = time.perf_counter()
            splan = ctx.plan(us, ts)
            t_plan = time.perf_counter() - t0
            _, srep = splan.execute_host_many(hb, hx)
            st_s = (time.perf_counter() - t0) / M
            splan.close()
            x_one = pinned_x.numpy()
            s_rel = float(np.max(np.abs(px[(M - 1) % 2].numpy() - x_one)) / np.max(np.abs(x_one)))
            e2e["streamed"] = {
                "value": P / st_s, "unit": "unknowns/s", "ms_per_step": st_s * 1e3, "steps": M,
                "h2d_bytes_per_step": 16 * P, "d2h_bytes_per_step": 16 * P,
                "api": "nds_plan_create + nds_plan_execute_host_many (pinned host buffers; plan creation "
                       "inside the timed region, amortised over the steps)",
                "plan_create_ms": t_plan * 1e3, "kernel_launches": srep["kernel_launches"],
                "x_rel_vs_one_shot": s_rel}

    # --- correctness stamp of the timed X (outside the timed region) ------------------------------
    verify = None
    if not args.no_verify:
        verify = verify_x(ctx, args.config, args.seed + rank, a_list, dims, d_x, d_b)

    # --- CPU baseline (rank 0, N=1): one full-workload solve of the reference's own stages -------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        try:
            rs = ReferenceStages(args.config, args.seed, threads)
            secs_c, st = rs.step()
            cpu = {"value": rs.P / secs_c, "unit": "unknowns/s", "cores": threads, "kind": "reference",
                   "sample": "one solve: " + reference_sample_text(args.config, threads),
                   "stage_seconds": st, "schur_seconds": rs.schur_s}
            del rs
        except Exception as e:  # the reference build travels with the repo; report if absent
            cpu = {"value": None, "unit": "unknowns/s", "cores": threads, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "unknowns/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128 (fp64 DMMA)", "data": "synthetic (generator v1, seeded Gaussian)",
            "config": bench_config(args.config, world), "schur_seconds_host": schur_s,
            "roofline": roofline, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps, "launches_per_step": launches_per_step,
            "clocks": clk.summary(), "verify": verify,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
