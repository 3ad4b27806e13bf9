"""Measurement for SURVEY 8(f) rows 1-2 (ODE propagator, RK4) on one B200.

Prints one JSON line per workload:
  ode_c1  — OdePropagator::at(t) on config c1's extents/coefficients (N=3, n=256, A_j from generator
            v1, X0 and B seeded complex normal, t = 0.05): device time of nds_ode_at_dev (CUDA
            events, K reps, inputs resident), host-buffer nds_ode_at (D2H included), unknowns/s;
            CPU baseline = the reference's propagate (oracle/_ref, all host threads) on the
            256x256x16 slab, rate = P / (its at() transform + backsub + inverse seconds).
  rk4_c0  — rk4_reference on config c0 (32^3), dt = 1e-4, 2000 steps (CUDA-graph replays), host
            buffers; CPU baseline = the reference's rk4_reference on the same system, 20 steps.
usage: python tools/bench_ode.py [--reps K]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2412_15840_b200 as nds  # noqa: E402
from paper_2412_15840_b200 import configs  # noqa: E402


def rand_c(rng, dims):
    return rng.standard_normal(dims) + 1j * rng.standard_normal(dims)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    import oracle

    ref = oracle.Ref() if os.path.exists(oracle.REF_PATH) else None
    threads = os.cpu_count() or 1
    if ref:
        ref.set_threads(threads)
    ctx = nds.Context(0)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)

    # ---- ode_c1 ------------------------------------------------------------------------------
    a, b = configs.make_problem("c1", seed=0)
    dims = b.shape
    P = int(np.prod(dims))
    x0 = rand_c(np.random.default_rng(1), dims)
    t = 0.05
    t0 = time.perf_counter()
    us, ts = zip(*[ctx.schur(m) for m in a])
    schur_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    ode = ctx.ode(us, ts, b, x0)
    create_s = time.perf_counter() - t0
    d_x = torch.empty(P, dtype=torch.complex128, device="cuda")
    for _ in range(2):
        ode.at_dev(t, d_x.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.reps):
        ode.at_dev(t, d_x.data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / args.reps
    pinned = torch.empty(P, dtype=torch.complex128, pin_memory=True)
    ode.at_ptr(t, pinned.data_ptr())
    t0 = time.perf_counter()
    for _ in range(3):
        rep_h = ode.at_ptr(t, pinned.data_ptr())
    host_ms = (time.perf_counter() - t0) / 3 * 1e3
    cpu = None
    if ref:
        slab = (256, 256, 16)
        sa, sb = configs.make_problem("c1", seed=0, dims=slab)
        sx0 = rand_c(np.random.default_rng(1), slab)
        _, rep = ref.propagate(sa, sb, sx0, t, report=True)
        at_s = rep["transform_seconds"] + rep["backsub_seconds"] + rep["inverse_seconds"]
        cpu = {"value": int(np.prod(slab)) / at_s, "unit": "unknowns/s", "cores": threads, "kind": "reference",
               "sample": f"reference propagate on the {slab} slab of c1, rate = P / at() stage seconds",
               "stage_seconds": {k: rep[k] for k in ("transform_seconds", "backsub_seconds", "inverse_seconds")}}
    print(json.dumps({"workload": "ode_c1", "metric": "unknowns/s per OdePropagator::at(t)", "dims": list(dims),
                      "t": t, "value": P / (dev_ms * 1e-3), "unit": "unknowns/s", "device_ms_per_at": dev_ms,
                      "host_ms_per_at": host_ms, "host_output": "pinned", "report": {k: rep_h[k] for k in (
                          "transform_seconds", "backsub_seconds", "inverse_seconds", "d2h_seconds")},
                      "setup_s": {"schur_host": schur_s, "ode_create": create_s}, "cpu_baseline": cpu,
                      "data": "synthetic (generator v1 coefficients, seeded X0)"}))
    ode.close()

    # ---- rk4_c0 ------------------------------------------------------------------------------
    a0, b0 = configs.make_problem("c0", seed=0)
    dims0 = b0.shape
    P0 = int(np.prod(dims0))
    x00 = rand_c(np.random.default_rng(2), dims0)
    dt, steps = 1e-4, 2000
    ctx.rk4(a0, b0, x00, dt * 10, dt)  # warm-up
    t0 = time.perf_counter()
    ctx.rk4(a0, b0, x00, dt * steps, dt)
    gpu_s = time.perf_counter() - t0
    cpu = None
    if ref:
        cs = 20
        t0 = time.perf_counter()
        ref.rk4(a0, b0, x00, dt * cs, dt)
        c_s = time.perf_counter() - t0
        cpu = {"value": cs / c_s, "unit": "steps/s", "cores": threads, "kind": "reference",
               "sample": f"reference rk4_reference on c0, {cs} steps of dt={dt}"}
    print(json.dumps({"workload": "rk4_c0", "metric": "RK4 steps/s (host buffers in/out)", "dims": list(dims0),
                      "steps": steps, "dt": dt, "value": steps / gpu_s, "unit": "steps/s",
                      "unknown_steps_per_s": steps * P0 / gpu_s, "cpu_baseline": cpu,
                      "data": "synthetic (generator v1 coefficients, seeded X0)"}))


if __name__ == "__main__":
    main()
