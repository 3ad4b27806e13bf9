"""BASELINE.json configs at FULL size on the GPU.

* Parity with the reference's X (north_star: relative max-norm <= 1e-9):
  - c1-c4 against the committed fixtures tests/golden/xref_<cfg>.npz, made by the unmodified
    reference ndsylv::solve (oracle/_ref) on the same generator-v1 inputs
    (tests/golden/make_xref.py): X at 66 K sampled flat indices (plus the first / last 512),
    ||X_ref||_max, and X summed over all modes but the first / the last (every entry enters);
  - c1 and c2 additionally against a fresh full run of the reference on the box's host cores
    (every entry compared; about 1 and 3 minutes of CPU).
* Size-independent properties: relative residual ||sum_j A_j x_j X - B|| / ||B|| <= 1e-10
  (2- and max-norm, on the device) and the forward->inverse round trip (U unitary).
All of them run the production plan path that bench.py times."""
import json
import os

import numpy as np
import pytest

from paper_2412_15840_b200 import configs

from conftest import rel_max

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
EXPECTED_PATH = {"c0": "cubic", "c1": "cubic", "c2": "cubic", "c3": "cubic", "c4": "binary"}


def _device_solve(ctx, name):
    """Generator-v1 inputs of a config, host Schur, one plan execution; returns (a, b, dims, d_b, d_x, plan)."""
    import torch
    a, b = configs.make_problem(name, seed=0)
    dims = b.shape
    us, ts = zip(*[ctx.schur(m) for m in a])
    plan = ctx.plan(list(us), list(ts))
    assert plan.solve_path() == EXPECTED_PATH[name]
    d_b = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).cuda()
    d_x = torch.empty_like(d_b)
    d_w = torch.empty_like(d_b)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
    torch.cuda.synchronize()
    ctx.set_stream(None)
    del d_w
    return a, b, dims, d_b, d_x, plan


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_full_config_against_reference_fixture(ctx, name):
    """X of the full config against the reference's X_ref (sampled entries, max-norm, slice sums)."""
    import torch
    path = os.path.join(GOLDEN, f"xref_{name}.npz")
    fx = np.load(path)
    assert int(fx["seed"]) == 0 and str(fx["generator"]) == configs.GENERATOR_VERSION
    a, b, dims, d_b, d_x, plan = _device_solve(ctx, name)
    del b, d_b
    assert tuple(fx["dims"]) == tuple(dims)
    xmax_ref = float(fx["xmax"])
    idx = torch.from_numpy(fx["idx"]).cuda()
    x_s = d_x[idx].cpu().numpy()
    err = float(np.max(np.abs(x_s - fx["x"]))) / xmax_ref
    xmax = float(d_x.abs().max())
    # column-major flat X: mode 1 is the fastest index, mode N the slowest
    n_all = d_x.numel()
    sum_first = d_x.view(-1, dims[0]).sum(0).cpu().numpy()
    sum_last = d_x.view(dims[-1], -1).sum(1).cpu().numpy()
    meta = json.loads(str(fx["meta"]))
    print(name, {"rel_max_sampled": err, "xmax_rel": abs(xmax - xmax_ref) / xmax_ref,
                 "ref_stage_s": {k: meta["report"][k] for k in ("transform_seconds", "backsub_seconds",
                                                                  "inverse_seconds")}})
    assert err <= 1e-9
    assert abs(xmax - xmax_ref) <= 1e-9 * xmax_ref
    # each slice sum adds n_all / n_j entries whose errors are each <= 1e-9 ||X||_max
    tol_first = 1e-9 * xmax_ref * np.sqrt(n_all / dims[0])
    tol_last = 1e-9 * xmax_ref * np.sqrt(n_all / dims[-1])
    assert np.max(np.abs(sum_first - fx["sum_first"])) <= tol_first
    assert np.max(np.abs(sum_last - fx["sum_last"])) <= tol_last


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_full_config_against_reference_run(ctx, ref, name):
    """The reference ndsylv::solve run on the box's host cores on the same inputs: every entry."""
    a, b, dims, d_b, d_x, plan = _device_solve(ctx, name)
    ref.set_threads(os.cpu_count() or 1)
    x_ref, rep = ref.solve(a, b)
    x_gpu = d_x.cpu().numpy().reshape(dims, order="F")
    err = rel_max(x_gpu, x_ref)
    print(name, {"rel_max": err, "ref_stage_s": {k: rep[k] for k in ("transform_seconds", "backsub_seconds",
                                                                     "inverse_seconds")}})
    assert err <= 1e-9


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "c4"])
def test_full_config_residual(ctx, name):
    import torch
    a, b = configs.make_problem(name, seed=0)
    dims = b.shape
    us, ts = zip(*[ctx.schur(m) for m in a])
    plan = ctx.plan(list(us), list(ts))
    d_b = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).cuda()
    del b
    d_x = torch.empty_like(d_b)
    d_w = torch.empty_like(d_b)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
    torch.cuda.synchronize()
    r = ctx.dev_residual(a, dims, d_x.data_ptr(), d_b.data_ptr())
    assert r["rel_res_2"] <= 1e-10, r
    assert r["rel_res_max"] <= 1e-10, r
    assert np.isfinite(r["res_max"])
    # forward then inverse is the identity up to round-off (test_sylvester.cpp:34-42)
    plan.forward(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
    plan.inverse(d_x.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
    torch.cuda.synchronize()
    err = float((d_x - d_b).abs().max() / d_b.abs().max())
    assert err <= 1e-13
    ctx.set_stream(None)


@pytest.mark.parametrize("name,dims", [("c1", (128, 96, 64)), ("c2", (32, 32, 32, 32)), ("c4", (2,) * 18)])
def test_plan_repeatable(ctx, name, dims):
    """nds_plan_execute gives the bitwise-same X on every call (fixed summation orders, no
    floating-point atomics; test_sylvester.cpp:127-154 pins bitwise reruns), including after a
    buffer change."""
    import torch
    a, b = configs.make_problem(name, seed=3, dims=dims)
    dims = b.shape  # the advection-diffusion generator (c2) uses one extent for every mode
    us, ts = zip(*[ctx.schur(m) for m in a])
    plan = ctx.plan(list(us), list(ts))
    d_b = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).cuda()
    bufs = [(torch.empty_like(d_b), torch.empty_like(d_b)) for _ in range(2)]
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    outs = []
    for k in [0, 0, 0, 1, 1, 0]:
        d_x, d_w = bufs[k]
        d_x.zero_()
        d_w.fill_(float("nan"))
        plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
        torch.cuda.synchronize()
        outs.append(d_x.cpu().numpy().copy())
    ctx.set_stream(None)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    res = ctx.apply_operator(a, np.asfortranarray(outs[0].reshape(dims, order="F")))
    assert np.linalg.norm(res - b) / np.linalg.norm(b) <= 1e-10


def test_plan_on_torch_default_stream(ctx):
    """ctx.set_stream(<torch's default stream, handle 0>) runs the library on the LEGACY default
    stream, so torch work queued right after it (no synchronisation) sees the finished X, and a
    buffer torch frees and reuses is not still being written (ADVICE: a handle of 0 used to fall
    back to the context's own non-blocking stream)."""
    import torch
    a, b = configs.make_problem("c1", seed=4, dims=(128, 128, 128))
    us, ts = zip(*[ctx.schur(m) for m in a])
    plan = ctx.plan(list(us), list(ts))
    d_b = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).cuda()
    ref_x = None
    with torch.cuda.stream(torch.cuda.default_stream()):
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)  # handle 0 -> legacy stream
        assert torch.cuda.current_stream().cuda_stream == 0
        for rep in range(3):
            d_x, d_w = torch.empty_like(d_b), torch.empty_like(d_b)
            d_x.fill_(float("nan"))
            plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
            x_host = d_x.cpu().numpy()  # torch reads on its default stream right away
            del d_x, d_w                # the allocator may hand these to the next iteration
            assert np.all(np.isfinite(x_host))
            if ref_x is None:
                ref_x = x_host
            assert np.array_equal(x_host, ref_x)
        ctx.set_stream(None)
    res = ctx.apply_operator(a, ref_x.reshape(b.shape, order="F"))
    assert np.linalg.norm(res - b) / np.linalg.norm(b) <= 1e-10
