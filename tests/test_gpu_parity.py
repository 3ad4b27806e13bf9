"""GPU parity: the CUDA path through the C ABI against the C oracle / the reference build on
identical inputs. Tolerances follow BASELINE.json north_star: relative max-norm <= 1e-9 for X,
relative residual <= 1e-10; stage kernels are held tighter (1e-12) since only summation order
differs; bitwise where the reference tests pin bitwise behaviour."""
import glob
import os

import numpy as np
import pytest

import oracle
import paper_2412_15840_b200 as nds
from paper_2412_15840_b200 import configs

from conftest import rel_max

pytestmark = pytest.mark.gpu

GOLDEN = sorted(p for p in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))
                if not os.path.basename(p).startswith("xref_"))


def rand_c(rng, shape):
    return np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def rand_factors(rng, dims):
    """Unitary U (QR of a random matrix) and upper-triangular T with well-separated diagonal."""
    us, ts = [], []
    for n in dims:
        q, _ = np.linalg.qr(rand_c(rng, (n, n)))
        t = np.triu(rand_c(rng, (n, n))) / np.sqrt(n)
        t[np.diag_indices(n)] = 2.0 + 0.5 * rng.standard_normal(n) + 0.5j * rng.standard_normal(n)
        us.append(np.asfortranarray(q))
        ts.append(np.asfortranarray(t))
    return us, ts


SHAPES = [(4, 3, 5), (32, 32, 32), (16, 1, 24), (2, 9, 33), (40, 24), (17, 33, 9), (130, 18), (8, 20, 8, 3),
          (2,) * 10, (3, 2, 5, 2, 3), (64, 1), (1, 70), (96, 12, 7)]


@pytest.mark.parametrize("dims", SHAPES, ids=["x".join(map(str, d)) for d in SHAPES])
def test_mode_product_all_modes(ctx, port, dims):
    rng = np.random.default_rng(1)
    x = rand_c(rng, dims)
    for mode in range(1, len(dims) + 1):
        m = rand_c(rng, (dims[mode - 1],) * 2)
        r_gpu = ctx.mode_product(m, mode, x)
        r_ref = port.mode_product(m, mode, x)
        assert rel_max(r_gpu, r_ref) <= 1e-13, mode


@pytest.mark.parametrize("dims", SHAPES, ids=["x".join(map(str, d)) for d in SHAPES])
def test_transforms_and_backsub(ctx, port, dims):
    rng = np.random.default_rng(2)
    us, ts = rand_factors(rng, dims)
    b = rand_c(rng, dims)
    c_gpu = ctx.forward_transform(us, b)
    c_ref = port.forward_transform(us, b)
    assert rel_max(c_gpu, c_ref) <= 1e-13
    x_gpu = ctx.inverse_transform(us, c_ref)
    assert rel_max(x_gpu, port.inverse_transform(us, c_ref)) <= 1e-13
    y_gpu, st = ctx.back_substitute(ts, c_ref)
    y_ref, st_ref = port.back_substitute(ts, c_ref)
    assert rel_max(y_gpu, y_ref) <= 1e-12
    assert st["entries"] == st_ref["entries"] and st["multiplies"] == st_ref["multiplies"]
    assert st["min_abs_denominator"] == pytest.approx(st_ref["min_abs_denominator"], rel=1e-15)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_golden_through_gpu(ctx, path):
    z = np.load(path)
    n = len(z["dims"])
    us = [z[f"u{j}"] for j in range(n)]
    ts = [z[f"t{j}"] for j in range(n)]
    a = [z[f"a{j}"] for j in range(n)]
    assert rel_max(ctx.forward_transform(us, z["b"]), z["c"]) <= 1e-13
    y, st = ctx.back_substitute(ts, z["c"])
    assert rel_max(y, z["y"]) <= 1e-12
    assert st["multiplies"] == int(z["backsub_multiplies"])
    r = ctx.solve_schur(us, ts, z["b"])
    assert rel_max(r.x, z["x"]) <= 1e-9
    # end to end through the GPU path with the product's own host Schur
    r2 = ctx.solve(a, z["b"])
    assert rel_max(r2.x, z["x"]) <= 1e-9
    res = ctx.apply_operator(a, r2.x)
    assert np.max(np.abs(res - z["b"])) <= 1e-10 * (1 + np.max(np.abs(z["b"])))


def test_singular_reports_first_offender(ctx, port):
    # test_sylvester.cpp:110-125
    ts = [np.diag([1.0, -1.0]).astype(complex), np.diag([-1.0, 1.0]).astype(complex)]
    c = np.ones((2, 2), dtype=complex)
    with pytest.raises(nds.SingularOperatorError) as ei:
        ctx.back_substitute(ts, c, 0.0)
    assert ei.value.multi_index == [2, 2]
    assert abs(ei.value.denominator) == 0.0
    # larger: offender set planted at several places; first in descending order wins
    dims = (5, 4, 3)
    rng = np.random.default_rng(5)
    us, ts = rand_factors(rng, dims)
    ts[0][1, 1] = -(ts[1][2, 2] + ts[2][0, 0])  # (2, 3, 1) singular
    ts[0][3, 3] = -(ts[1][0, 0] + ts[2][1, 1])  # (4, 1, 2) singular  (flat larger)
    with pytest.raises(nds.SingularOperatorError) as e_gpu:
        ctx.solve_schur(us, ts, rand_c(rng, dims))
    with pytest.raises(oracle.OracleError) as e_ref:
        port.solve_schur(us, ts, rand_c(rng, dims))
    assert e_gpu.value.multi_index == e_ref.value.bad_index == [4, 1, 2]


def test_identity_n2_bitwise_and_deterministic(ctx):
    # test_sylvester.cpp:127-154
    rng = np.random.default_rng(904)
    b = rand_c(rng, (3, 4))
    r = ctx.solve([np.eye(3), np.eye(4)], b)
    assert r.report["used_normal_fast_path"] == 1
    assert np.array_equal(r.x, b / 2.0)
    b3 = rand_c(rng, (3, 2, 4))
    r3 = ctx.solve([np.eye(3), np.eye(2), np.eye(4)], b3)
    assert np.all(np.abs(r3.x - b3 / 3.0) <= 5e-16 * np.abs(b3))
    assert np.array_equal(ctx.solve([np.eye(3), np.eye(2), np.eye(4)], b3).x, r3.x)


def test_general_route_deterministic(ctx):
    a, b = configs.make_problem("c0", seed=3, dims=(24, 20, 16))
    x1 = ctx.solve(a, b).x
    x2 = ctx.solve(a, b).x
    assert np.array_equal(x1, x2)


def test_fast_path_agrees_with_general(ctx, ref):
    # test_sylvester.cpp:192-211: normal coefficients
    rng = np.random.default_rng(911)
    coeffs = []
    for n in (4, 3):
        q, _ = np.linalg.qr(rand_c(rng, (n, n)))
        d = 1.0 + rng.random(n) + 1j * rng.random(n)
        coeffs.append(q @ np.diag(d) @ q.conj().T)
    b = rand_c(rng, (4, 3))
    fast = ctx.solve(coeffs, b)
    slow = ctx.solve(coeffs, b, allow_fast_path=False)
    assert fast.report["used_normal_fast_path"] == 1 and slow.report["used_normal_fast_path"] == 0
    assert np.max(np.abs(fast.x - slow.x)) <= 1e-10 * (1 + np.max(np.abs(slow.x)))
    x_ref, _ = ref.solve(coeffs, b)
    assert rel_max(fast.x, x_ref) <= 1e-12


def test_real_output(ctx):
    a, b = configs.make_problem("c2", dims=(16, 16, 16, 16))
    r = ctx.solve(a, b, real_output=True)
    assert np.all(r.x.imag == 0)


def test_shape_errors(ctx):
    # test_sylvester.cpp:247-258
    with pytest.raises(ValueError):
        ctx.solve([np.eye(2), np.eye(3)], np.zeros((2, 2)))
    with pytest.raises(ValueError):
        ctx.solve([np.eye(2)], np.zeros((2, 2)))
    with pytest.raises(ValueError):
        ctx.solve([np.eye(4)], np.zeros((4,)))
    with pytest.raises(ValueError):
        ctx.mode_product(np.eye(3), 0, np.zeros((3, 4)))
    with pytest.raises(ValueError):
        ctx.mode_product(np.eye(3), 3, np.zeros((3, 4)))


@pytest.mark.parametrize("dims,seed", [((5, 4, 3), 905), ((2, 9, 33), 42), ((3, 4, 2), 906), ((2,) * 12, 4212),
                                       ((12, 11, 10, 9), 7)])
def test_solve_matches_reference_solver(ctx, ref, dims, seed):
    a, x_true, b = ref.random_problem(list(dims), seed)
    x_ref, rep_ref = ref.solve(a, b)
    r = ctx.solve(a, b)
    assert rel_max(r.x, x_ref) <= 1e-9
    assert np.max(np.abs(r.x - x_true)) <= 1e-9
    assert r.report["backsub_multiplies"] == rep_ref["backsub_multiplies"]
    assert r.report["backsub_entries"] == rep_ref["backsub_entries"]
    assert r.report["used_normal_fast_path"] == rep_ref["used_normal_fast_path"]
    assert r.report["min_abs_denominator"] == pytest.approx(rep_ref["min_abs_denominator"], rel=1e-9)


def test_c0_full_against_reference(ctx, ref):
    a, b = configs.make_problem("c0", seed=0)
    x_ref, _ = ref.solve(a, b)
    r = ctx.solve(a, b)
    assert rel_max(r.x, x_ref) <= 1e-9
    res = ctx.apply_operator(a, r.x)
    assert np.linalg.norm(res - b) / np.linalg.norm(b) <= 1e-10


# Reduced shapes chosen so that the solve runs the PRODUCTION route of each config (16^3 / 8^4
# cubic tiles with >= 3 tile blocks per mode, i.e. DMMA far items, pushed near items and the
# line-owner diagonal kernel; all-binary tiles for c4), with the default environment.
REDUCED = [("c1", (128, 128, 64), "cubic"), ("c2", (32, 32, 32, 32), "cubic"), ("c3", (64, 64, 32, 32), "cubic"),
           ("c3", (32, 32, 32, 32), "cubic"), ("c4", (2,) * 16, "binary"), ("c4", (2,) * 20, "binary")]


@pytest.mark.parametrize("name,dims,path", REDUCED, ids=[f"{n}-{'x'.join(map(str, d))}" for n, d, _ in REDUCED])
def test_configs_reduced_against_reference(ctx, ref, name, dims, path):
    """sylvester.cpp:167-227 on the same inputs: the GPU X (host API and device plan) against the
    reference's X at the north_star tolerance, on the route the full config takes."""
    import torch
    a, b = configs.make_problem(name, seed=1, dims=dims)
    dims = b.shape
    x_ref, rep = ref.solve(a, b)
    r = ctx.solve(a, b)
    assert rel_max(r.x, x_ref) <= 1e-9
    assert r.report["backsub_multiplies"] == rep["backsub_multiplies"]
    us, ts = zip(*[ctx.schur(m) for m in a])
    plan = ctx.plan(list(us), list(ts))
    assert plan.solve_path() == path
    d_b = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).cuda()
    d_x, d_w = torch.empty_like(d_b), torch.empty_like(d_b)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
    torch.cuda.synchronize()
    ctx.set_stream(None)
    x_plan = d_x.cpu().numpy().reshape(dims, order="F")
    assert rel_max(x_plan, x_ref) <= 1e-9


@pytest.mark.parametrize("dims", [(64, 64, 64), (48, 48, 48), (16, 32, 48, 64)],
                         ids=["64x64x64", "48x48x48", "16x32x48x64"])
def test_cubic_solve_stage_against_oracle(ctx, port, dims):
    """The production cubic-tile back-substitution alone (default environment, far items on
    every mode) against the oracle's back_substitute (sylvester.cpp:71-108) on the same C."""
    rng = np.random.default_rng(23)
    us, ts = rand_factors(rng, dims)
    c = rand_c(rng, dims)
    plan = ctx.plan(us, ts, allow_fast_path=False)
    assert plan.solve_path() == "cubic"
    y_gpu = ctx.back_substitute(ts, c)[0]
    y_ref = port.back_substitute(ts, c)[0]
    assert rel_max(y_gpu, y_ref) <= 1e-12


@pytest.mark.parametrize("dims", [(2,) * 20, (48, 40, 64), (16, 16, 16, 32), (40, 3, 1024), (24, 20, 256),
                                  (8, 12, 10, 128)],
                         ids=["bin20", "48x40x64", "16x16x16x32", "40x3x1024", "24x20x256", "8x12x10x128"])
def test_host_path_with_copy_overlap(ctx, port, dims):
    """nds_solve_schur streams B in / X out in chunks of the slowest modes overlapped with the
    per-chunk transform passes; results must equal the unchunked oracle path. The last three
    shapes also split the last pass per chunk (K-split forward accumulation into a third buffer,
    row-block inverse)."""
    rng = np.random.default_rng(17)
    us, ts = rand_factors(rng, dims)
    b = rand_c(rng, dims)
    r = ctx.solve_schur(us, ts, b, allow_fast_path=False)
    x_ref, _ = port.solve_schur(us, ts, b, flags=0)
    assert rel_max(r.x, x_ref) <= 1e-11
    r2 = ctx.solve_schur(us, ts, b, allow_fast_path=False, real_output=True)
    assert np.all(r2.x.imag == 0) and rel_max(r2.x.real, x_ref.real) <= 1e-11


@pytest.mark.parametrize("dims", [(48, 40, 64), (40, 3, 1024), (2,) * 20, (24, 20, 16)],
                         ids=["48x40x64", "40x3x1024", "bin20", "24x20x16"])
def test_host_path_pageable_equals_pinned(ctx, dims):
    """nds_solve_schur from PAGEABLE host buffers (the reference's std::vector storage, staged
    through the library's pinned ring) and from pinned buffers: bitwise the same X."""
    import ctypes as C
    import torch
    rng = np.random.default_rng(29)
    us, ts = rand_factors(rng, dims)
    b = np.asfortranarray(rand_c(rng, dims))
    flat = np.ascontiguousarray(b.reshape(-1, order="F"))
    outs = []
    for pinned in (False, True):
        if pinned:
            hb = torch.from_numpy(flat.copy()).pin_memory()
            hx = torch.empty_like(hb).pin_memory()
            pb, px = hb.data_ptr(), hx.data_ptr()
        else:
            hb, hx = flat.copy(), np.empty_like(flat)
            pb, px = hb.ctypes.data, hx.ctypes.data
        up, ku = nds._ptr_array(us)
        tp, kt = nds._ptr_array(ts)
        rep, sing = nds._Report(), nds._Singular()
        rc = ctx.lib.nds_solve_schur(ctx.h, len(dims), nds._dims(dims), up, tp, pb, px, 0.0, 0, C.byref(rep),
                                     C.byref(sing))
        assert rc == 0, ctx.last_error()
        outs.append(hx.numpy().copy() if pinned else hx.copy())
    assert np.array_equal(outs[0], outs[1])
    x_ref, _ = oracle.Port().solve_schur(us, ts, b, flags=0)
    assert rel_max(outs[0].reshape(dims, order="F"), x_ref) <= 1e-11


@pytest.mark.parametrize("dims,count", [((64, 64, 64), 5), ((16, 16, 16, 32), 3), ((2,) * 18, 4), ((24, 20, 16), 2),
                                        ((48, 40, 64), 1)],
                         ids=["64^3x5", "16x16x16x32x3", "bin18x4", "24x20x16x2", "48x40x64x1"])
def test_execute_host_many(ctx, port, dims, count):
    """nds_plan_execute_host_many: several right-hand sides through one plan, pinned (pipelined:
    H2D of b[k+1] and D2H of x[k-1] under solve k, device buffers double-buffered) and pageable
    (one chunked host solve each). Every x[k] against the oracle on b[k]; pinned and pageable
    runs against each other and against the device-pointer execute of the same plan (bitwise:
    the pipelined path runs the same kernels on whole tensors)."""
    import torch
    rng = np.random.default_rng(41)
    us, ts = rand_factors(rng, dims)
    bs = [np.asfortranarray(rand_c(rng, dims)) for _ in range(count)]
    plan = ctx.plan(us, ts, allow_fast_path=False)
    xs_page, rep = plan.execute_host_many(bs)
    assert rep["kernel_launches"] > 0
    flats = [torch.from_numpy(np.ascontiguousarray(b.reshape(-1, order="F"))).pin_memory() for b in bs]
    outs = [torch.empty_like(f).pin_memory() for f in flats]
    plan.execute_host_many([f.data_ptr() for f in flats], [o.data_ptr() for o in outs])
    dev_b = torch.from_numpy(np.ascontiguousarray(bs[-1].reshape(-1, order="F"))).cuda()
    dev_x = torch.empty_like(dev_b)
    plan.execute(dev_b.data_ptr(), dev_x.data_ptr())
    torch.cuda.synchronize()
    x_dev = dev_x.cpu().numpy()
    for k in range(count):
        x_ref, _ = port.solve_schur(us, ts, bs[k], flags=0)
        x_pin = outs[k].numpy().reshape(dims, order="F")
        assert rel_max(x_pin, x_ref) <= 1e-11
        assert rel_max(xs_page[k], x_ref) <= 1e-11
    if count > 1:
        assert np.array_equal(outs[-1].numpy(), x_dev)
    # in place (x[k] aliases b[k]) gives the same X
    inplace = [f.clone().pin_memory() for f in flats]
    plan.execute_host_many([f.data_ptr() for f in inplace], [f.data_ptr() for f in inplace])
    for k in range(count):
        assert np.array_equal(inplace[k].numpy(), outs[k].numpy()) or count == 1
    plan.close()


@pytest.mark.parametrize("n_modes,seed", [(13, 1), (16, 2), (20, 3)])
def test_binary_diagonalised_route_matches_coupled_solve(ctx, ref, n_modes, seed):
    """All-binary problems with more than 12 modes: a full solve (nds_plan_execute) diagonalises
    the outer modes into the transform passes and solves decoupled tiles; the stage APIs
    (forward, back_substitute, inverse) run the plain coupled solve. Both against the reference."""
    import torch
    a, b = configs.make_problem("c4", seed=seed, dims=(2,) * n_modes)
    x_ref, _ = ref.solve(a, b)
    us, ts = zip(*[ctx.schur(m) for m in a])
    plan = ctx.plan(list(us), list(ts))
    d_b = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).cuda()
    d_x, d_w, d_c = torch.empty_like(d_b), torch.empty_like(d_b), torch.empty_like(d_b)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
    plan.forward(d_b.data_ptr(), d_c.data_ptr(), d_w.data_ptr())
    plan.backsub(d_c.data_ptr())
    plan.inverse(d_c.data_ptr(), d_c.data_ptr(), d_w.data_ptr())
    torch.cuda.synchronize()
    ctx.set_stream(None)
    x_fast = d_x.cpu().numpy().reshape(b.shape, order="F")
    x_stage = d_c.cpu().numpy().reshape(b.shape, order="F")
    assert rel_max(x_fast, x_ref) <= 1e-12
    assert rel_max(x_stage, x_ref) <= 1e-12
    r = ctx.solve(a, b)  # host path (chunked passes) takes the diagonalised route too
    assert rel_max(r.x, x_ref) <= 1e-12


DIAG_CASES = [("c1", (128, 128, 64), True), ("c1", (64, 64, 64), True), ("c3", (64, 64, 32, 32), True),
              ("c3", (32, 32, 32, 32), True), ("c2", (32, 32, 32, 32), True), ("c2", (48, 48, 48, 48), True)]


@pytest.mark.parametrize("name,dims,taken", DIAG_CASES, ids=[f"{n}-{'x'.join(map(str, d))}" for n, d, _ in DIAG_CASES])
def test_cubic_diagonalised_route(ctx, ref, name, dims, taken):
    """Block-diagonalised cubic route (capi.cu plan_cubic_diag): full solves replace T_j by
    W_j^{-1} T_j W_j (W_j = eigenvectors of T_j's diagonal tile blocks), so the diagonal tiles are
    divisions. With the Schur forms reordered (eigenvalues spread over every block) the guard takes
    it for the Gaussian configs (c1, c3) and for the advection-diffusion spectra of c2 (refused in
    the QR iteration's order: clustered neighbours). The route, the wavefront route
    (NO_DIAGONALISE) and the stage APIs (plain factors) all match the reference's X at the
    north_star tolerance."""
    import torch
    a, b = configs.make_problem(name, seed=1, dims=dims)
    x_ref, _ = ref.solve(a, b)
    us, ts = zip(*[ctx.schur(m) for m in a])
    d_b = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).cuda()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    xs = {}
    for diag in (True, False):
        plan = ctx.plan(list(us), list(ts), diagonalise=diag)
        assert plan.solve_path() == "cubic"
        got, cond = plan.diagonalised()
        assert got == (taken and diag)
        if diag and taken:
            assert 1.0 <= cond <= 1e6
        d_x, d_w, d_c = torch.empty_like(d_b), torch.empty_like(d_b), torch.empty_like(d_b)
        plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
        plan.forward(d_b.data_ptr(), d_c.data_ptr(), d_w.data_ptr())
        plan.backsub(d_c.data_ptr())
        plan.inverse(d_c.data_ptr(), d_c.data_ptr(), d_w.data_ptr())
        torch.cuda.synchronize()
        xs[diag] = d_x.cpu().numpy().reshape(b.shape, order="F")
        x_stage = d_c.cpu().numpy().reshape(b.shape, order="F")
        assert rel_max(x_stage, x_ref) <= 1e-11
        plan.close()
    ctx.set_stream(None)
    assert rel_max(xs[True], x_ref) <= 1e-11
    assert rel_max(xs[False], x_ref) <= 1e-11
    r = ctx.solve(a, b)  # host path (chunked passes, split last pass) on the same route
    assert rel_max(r.x, x_ref) <= 1e-11


def test_cubic_diagonalised_superblocks_and_guard(ctx, port):
    """Super-block choice of the block-diagonalised route: every D_j is a multiple of the tile
    edge dividing n_j, the level count is sum_j (n_j / D_j - 1) + 1, and the guard's bound holds.
    The plan reorders the Schur forms so every block holds eigenvalues spread over the spectrum, so
    a repeated eigenvalue still admits the route (the copies land in different blocks), while a mode
    whose eigenvalues are ALL equal (every block repeats one: no eigenvector basis) makes the guard
    refuse it; all plans match the oracle's full solve."""
    import torch
    rng = np.random.default_rng(41)
    dims = (64, 64, 64)
    us, ts = rand_factors(rng, dims)
    b = rand_c(rng, dims)
    x_ref, _ = port.solve_schur(us, ts, b, flags=0)
    ts_rep = [t.copy() for t in ts]
    ts_rep[1][6, 6] = ts_rep[1][5, 5]  # a repeated eigenvalue (same 16-row block before reordering)
    x_rep, _ = port.solve_schur(us, ts_rep, b, flags=0)
    ts_all = [t.copy() for t in ts]
    ts_all[1][np.diag_indices(dims[1])] = 2.5 + 0.25j  # every eigenvalue of mode 2 the same
    x_all, _ = port.solve_schur(us, ts_all, b, flags=0)
    d_b = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).cuda()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    for t_list, x_want, taken in ((ts, x_ref, True), (ts_rep, x_rep, True), (ts_all, x_all, False)):
        plan = ctx.plan(us, t_list, allow_fast_path=False)
        got, cond = plan.diagonalised()
        assert got == taken
        levels, d = plan.superblocks()
        if taken:
            assert cond <= 1e6
            assert all(dj % 16 == 0 and n % dj == 0 for n, dj in zip(dims, d))
            assert levels == sum(n // dj - 1 for n, dj in zip(dims, d)) + 1
        else:
            assert levels == 0 and d is None
        d_x, d_w = torch.empty_like(d_b), torch.empty_like(d_b)
        plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
        torch.cuda.synchronize()
        x = d_x.cpu().numpy().reshape(dims, order="F")
        assert rel_max(x, x_want) <= 1e-11
        plan.close()
    ctx.set_stream(None)


@pytest.mark.parametrize("n_modes,seed", [(16, 5), (24, 6)])
def test_binary_diagonalised_inner_modes(ctx, ref, n_modes, seed):
    """All-binary route: besides the outer modes, inner modes are diagonalised within the guard
    (the fused kernel's tile wavefront shrinks to the coupled inner modes); the full solve through
    the fused kernel (modes 1-12 pass first) matches the reference."""
    import torch
    a, b = configs.make_problem("c4", seed=seed, dims=(2,) * n_modes)
    x_ref, _ = ref.solve(a, b)
    us, ts = zip(*[ctx.schur(m) for m in a])
    plan = ctx.plan(list(us), list(ts))
    got, cond = plan.diagonalised()
    assert got and cond <= 1e6
    d_b = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).cuda()
    d_x, d_w = torch.empty_like(d_b), torch.empty_like(d_b)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
    torch.cuda.synchronize()
    ctx.set_stream(None)
    assert rel_max(d_x.cpu().numpy().reshape(b.shape, order="F"), x_ref) <= 1e-12


def _binary_factors(rng, n_modes, coupled=(), antidiagonal=()):
    """2 x 2 Schur pairs: random unitary U_j and T_j = [[a, b], [0, d]] with separated eigenvalues;
    modes in `coupled` get a repeated eigenvalue (a = d: not diagonalisable, so the route must
    keep their coupling); modes in `antidiagonal` get U_j = [[0, 1], [1, 0]] (zero diagonal: the
    unit-diagonal normalisation of the factors is refused)."""
    us, ts = [], []
    for j in range(n_modes):
        q, _ = np.linalg.qr(rand_c(rng, (2, 2)))
        if j in antidiagonal:
            q = np.array([[0, 1], [1, 0]], dtype=np.complex128)
        a = 2.0 + 0.3 * (rng.standard_normal() + 1j * rng.standard_normal())
        d = a if j in coupled else a + 1.0 + 0.2j * rng.standard_normal()
        t = np.array([[a, 0.5 * (rng.standard_normal() + 1j * rng.standard_normal())], [0, d]], dtype=np.complex128)
        us.append(np.asfortranarray(q))
        ts.append(np.asfortranarray(t))
    return us, ts


@pytest.mark.parametrize("coupled,antidiagonal", [((), ()), ((0, 5, 11), ()), ((1, 2, 3, 4), ()), ((0, 2, 4, 6, 8, 10), ()),
                                                  ((3,), (7,)), ((), (0, 13)), ((0, 1, 2, 3, 4), (12,))])
def test_binary_fused_kernel_variants(ctx, coupled, antidiagonal):
    """The fused all-binary route on hand-built Schur factors, against the C oracle on the same
    factors: up to four coupled inner modes at any tile bits (the solve inside a butterfly round),
    more than four (the popcount-wavefront kernel), and factors with a zero diagonal entry (plain
    instead of unit-diagonal butterflies)."""
    import oracle
    import torch
    rng = np.random.default_rng(1234 + 17 * len(coupled) + len(antidiagonal))
    n_modes = 15
    us, ts = _binary_factors(rng, n_modes, coupled, antidiagonal)
    b = rand_c(rng, (2,) * n_modes)
    b = np.asfortranarray(b)
    x_ref, _ = oracle.Port().solve_schur(us, ts, b)
    plan = ctx.plan(us, ts)
    got, cond = plan.diagonalised()
    assert got and cond <= 1e6
    d_b = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).cuda()
    d_x, d_w = torch.empty_like(d_b), torch.empty_like(d_b)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
    torch.cuda.synchronize()
    ctx.set_stream(None)
    plan.close()
    assert rel_max(d_x.cpu().numpy().reshape(b.shape, order="F"), x_ref) <= 1e-12


def _spectrum_factors(rng, dims, kind):
    """Unitary U and upper-triangular T whose eigenvalues (the diagonal) follow `kind`:
    'spread' (disk of radius 1 around 2), 'clustered' (most of them within 1e-3 of each other),
    'real' (real, graded like a discretised diffusion operator), with O(1/sqrt(n)) coupling."""
    us, ts = [], []
    for n in dims:
        q, _ = np.linalg.qr(rand_c(rng, (n, n)))
        t = np.triu(rand_c(rng, (n, n))) / np.sqrt(n)
        if kind == "spread":
            lam = 2.0 + rng.uniform(0, 1, n) ** 0.5 * np.exp(2j * np.pi * rng.uniform(0, 1, n))
        elif kind == "clustered":
            lam = 2.0 + 1e-3 * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
            lam[: n // 4] += rng.uniform(0.5, 1.5, n // 4)
        else:
            lam = 0.25 + np.sort(rng.uniform(0, 1, n)) ** 2 + 0j
        t[np.diag_indices(n)] = lam
        us.append(np.asfortranarray(q))
        ts.append(np.asfortranarray(t))
    return us, ts


ROUTE_CASES = [((48, 48, 48), "spread"), ((64, 32, 48), "spread"), ((32, 32, 32, 32), "spread"),
               ((48, 48, 48), "clustered"), ((32, 32, 32, 32), "clustered"), ((64, 64, 64), "real"),
               ((32, 48, 32, 16), "real"), ((96, 32, 32), "spread")]


@pytest.mark.parametrize("dims,kind", ROUTE_CASES, ids=[f"{k}-{'x'.join(map(str, d))}" for d, k in ROUTE_CASES])
def test_diagonalised_route_guard_random_spectra(ctx, port, dims, kind):
    """The guard on random spectra: whenever the plan takes the block-diagonalised route its bound
    is <= 1e6 and X matches the oracle at the north_star tolerance; clustered spectra (no
    well-conditioned eigenvector basis for the blocks) must either be refused (wavefront route)
    or still land within tolerance. Both routes of the same plan are checked."""
    import torch
    import zlib
    rng = np.random.default_rng(zlib.crc32(f"{kind}{dims}".encode()))
    us, ts = _spectrum_factors(rng, dims, kind)
    b = rand_c(rng, dims)
    x_ref, _ = port.solve_schur(us, ts, b, flags=0)
    d_b = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).cuda()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    for diag in (True, False):
        plan = ctx.plan(us, ts, allow_fast_path=False, diagonalise=diag)
        taken, cond = plan.diagonalised()
        d_x, d_w = torch.empty_like(d_b), torch.empty_like(d_b)
        plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
        torch.cuda.synchronize()
        err = rel_max(d_x.cpu().numpy().reshape(dims, order="F"), x_ref)
        if taken:
            assert cond <= 1e6
            assert err <= 1e-9, (kind, dims, cond, err)
        else:
            assert err <= 1e-11, (kind, dims, err)
        plan.close()
    ctx.set_stream(None)
    r = ctx.solve_schur(us, ts, b, allow_fast_path=False)  # one-shot route choice
    assert rel_max(r.x, x_ref) <= 1e-9
