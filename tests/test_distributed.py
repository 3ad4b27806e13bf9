"""Multi-GPU sharded solve.

CPU (gloo, world 2-4): the engine's schedule (layouts, all-to-all re-shards, pipelined solve with
head couplings over the Kronecker sum T_H, pipe couplings, extent-1 folding) run by
HostShardedSolver with numpy mode products and the C oracle's back_substitute, against the
single-process oracle — including all-binary problems sharded over hypercube super-modes.

GPU: the C-ABI engine (nds_dist_*) with P ranks as host threads sharing the one GPU through the
loopback transport (correctness of the stream-ordered orchestration, not a performance claim),
with a real NCCL communicator at world 1, and nds_solve_multi."""
import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2412_15840_b200.distributed import HostShardedSolver, block_partition, gather_LN, plan_layout, scatter_LN


def _mode_product_np(x, dims, m, mode):
    X = x.numpy().reshape(dims, order="F")
    R = np.moveaxis(np.tensordot(m, X, axes=([1], [mode - 1])), 0, mode - 1)
    return torch.from_numpy(np.asfortranarray(R).reshape(-1, order="F").copy())


class CpuOps:
    """Test-only local compute: numpy mode products and the C oracle's back_substitute."""

    def __init__(self):
        self.port = oracle.Port()

    def mode_product(self, dims, m, mode, x):
        return _mode_product_np(x, dims, m, mode)

    def back_substitute(self, ts, dims, c, tol):
        y, _ = self.port.back_substitute(ts, c.numpy().reshape(dims, order="F"), tol)
        c.copy_(torch.from_numpy(y.reshape(-1, order="F").copy()))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(dims, seed):
    rng = np.random.default_rng(seed)
    us, ts = [], []
    for n in dims:
        q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        t = np.triu(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
        t[np.diag_indices(n)] = 2.0 + 0.3 * rng.standard_normal(n) + 0.3j * rng.standard_normal(n)
        us.append(np.asfortranarray(q))
        ts.append(np.asfortranarray(t))
    b = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    return us, ts, b


def _worker(rank, world, port, dims, seed, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    us, ts, b = _problem(dims, seed)
    slabs = scatter_LN(b, world)
    solver = HostShardedSolver(dims, us, ts, CpuOps())
    x_local = solver.solve(torch.from_numpy(slabs[rank]))
    np.save(os.path.join(out_dir, f"x{rank}.npy"), x_local.numpy())
    dist.destroy_process_group()


CASES = [(2, (6, 5, 8)), (3, (7, 4, 9)), (2, (4, 3, 2, 5)), (3, (5, 6)), (4, (8, 6, 16)), (4, (16, 3, 5, 8)),
         (2, (2,) * 8), (4, (2,) * 9), (4, (2,) * 5)]


@pytest.mark.parametrize("world,dims", CASES, ids=[f"w{w}-{'x'.join(map(str, d))}" for w, d in CASES])
def test_sharded_schedule_matches_oracle(tmp_path, world, dims):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, dims, 123, str(tmp_path)), nprocs=world, join=True)
    us, ts, b = _problem(dims, 123)
    x = gather_LN([np.load(tmp_path / f"x{r}.npy") for r in range(world)], dims)
    x_ref, _ = oracle.Port().solve_schur(us, ts, b, flags=0)
    assert np.max(np.abs(x - x_ref)) / np.max(np.abs(x_ref)) <= 1e-12


def test_block_partition():
    assert block_partition(8, 3) == ([0, 3, 6], [3, 3, 2])
    assert block_partition(4, 4) == ([0, 1, 2, 3], [1, 1, 1, 1])
    s, m = block_partition(256, 8)
    assert sum(m) == 256 and all(v == 32 for v in m)


def test_layouts_of_the_sharded_configs():
    """c3 keeps its local solves on the cubic 8^4 route (blocks of 16 x 128 x 128 x 8); c4 shards
    over hypercube super-modes (3 head / 3 tail binary modes at P = 8, 16 pipe blocks)."""
    for P in (2, 4, 8):
        L = plan_layout((128,) * 4, P)
        assert (L.h, L.g, L.gp) == (1, 1, 1)
        assert all(m % 8 == 0 for m in L.mH) and all(m % 8 == 0 for m in L.mK)
        assert len(L.sK) >= 2 * P
        L = plan_layout((2,) * 29, P)
        k = P.bit_length() - 1
        assert (L.h, L.g) == (k, k) and L.mH == [1] * P and len(L.sK) == 2 ** L.gp >= 2 * P
        # every lower rank's inbound couplings come from hypercube neighbours only
        assert all(sum(L.couples(q, qp) for qp in range(P)) == k - bin(q).count("1") for q in range(P))
    L = plan_layout((256,) * 3, 8)
    assert all(m % 16 == 0 for m in L.mH) and all(m % 16 == 0 for m in L.mK)
    with pytest.raises(ValueError):
        plan_layout((2,) * 29, 6)
    with pytest.raises(ValueError):
        plan_layout((4, 8, 3), 4)
    # L_N slabs tile the tensor in order
    L = plan_layout((6, 5, 8), 3)
    assert [L.slab(r) for r in range(3)] == [(0, 90), (90, 90), (180, 60)]
    # NVLink bytes per solve: c3 at P = 8
    L = plan_layout((128,) * 4, 8)
    assert L.alltoall_bytes(0) == 2 * 7 * 16 * 16 * 128 * 128 * 16
    assert L.pipeline_bytes(7) == 7 * 16 * 16 * 128 * 128 * 128


# ---- the C-ABI engine on the GPU ------------------------------------------------------------------

def _engine_run(dims, P, seed=7):
    """P loopback ranks (host threads, one context each, one GPU): returns X and the infos."""
    import paper_2412_15840_b200 as nds
    from paper_2412_15840_b200.distributed import Comm, ShardedSolver
    us, ts, b = _problem(dims, seed)
    comms = Comm.loopback(P) if P > 1 else [None]
    slabs = scatter_LN(b, P)
    out, infos, errs = [None] * P, [None] * P, []

    def rank_main(r):
        try:
            ctx = nds.Context(0)
            solver = ShardedSolver(ctx, us, ts, comms[r])
            off, cnt = solver.slab(r)
            assert cnt == slabs[r].size
            db = torch.from_numpy(slabs[r]).cuda()
            dx = torch.empty_like(db)
            for _ in range(2):  # twice: buffers and events are reused
                solver.solve(db, dx)
            torch.cuda.synchronize()
            out[r] = dx.cpu().numpy()
            infos[r] = solver.info()
            solver.close()
            ctx.close()
        except Exception as e:  # surfaced below
            errs.append(repr(e))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in comms:
        if c is not None:
            c.close()
    assert not errs, errs
    return us, ts, b, gather_LN(out, dims), infos


ENGINE = [((24, 16, 32), 1), ((24, 16, 32), 2), ((32, 16, 16, 32), 4), ((48, 32, 64), 2), ((64, 32, 64), 4),
          ((2,) * 14, 2), ((2,) * 15, 4), ((40, 24, 16), 3)]


@pytest.mark.gpu
@pytest.mark.parametrize("dims,P", ENGINE, ids=[f"P{p}-{'x'.join(map(str, d))}" for d, p in ENGINE])
def test_engine_loopback_matches_oracle(dims, P):
    us, ts, b, x, infos = _engine_run(dims, P)
    x_ref, _ = oracle.Port().solve_schur(us, ts, b, flags=0)
    assert np.max(np.abs(x - x_ref)) / np.max(np.abs(x_ref)) <= 1e-12
    L = plan_layout(dims, P)
    for r, i in enumerate(infos):
        assert (i["ranks"], i["rank"]) == (P, r)
        assert (i["head_modes"], i["tail_modes"], i["pipe_modes"], i["pipe_blocks"]) == (L.h, L.g, L.gp, len(L.sK))
        assert i["alltoall_bytes"] == L.alltoall_bytes(r) and i["pipeline_bytes"] == L.pipeline_bytes(r)
    if dims == (64, 32, 64):  # 16^3-tile blocks: the local solves stay on the cubic route
        assert all(i["local_solve_path"] == 2 for i in infos)
    if all(d == 2 for d in dims):
        assert all(i["local_solve_path"] == 3 for i in infos)


@pytest.mark.gpu
def test_engine_singular_is_global():
    """Every rank raises the same global first offender before any exchange (no hang)."""
    import paper_2412_15840_b200 as nds
    from paper_2412_15840_b200.distributed import Comm, ShardedSolver
    dims = (8, 4, 8)
    us, ts, _ = _problem(dims, 3)
    ts[0][5, 5] = -(ts[1][2, 2] + ts[2][6, 6])
    comms = Comm.loopback(2)
    seen = []

    def rank_main(r):
        ctx = nds.Context(0)
        try:
            ShardedSolver(ctx, us, ts, comms[r])
        except nds.SingularOperatorError as e:
            seen.append(tuple(e.multi_index))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert seen == [(6, 3, 7), (6, 3, 7)]


@pytest.mark.gpu
def test_engine_nccl_world1_and_solve_multi(ctx):
    """A real NCCL communicator (world 1, unique id through a torch.distributed group) and the
    single-process multi-device entry on the one GPU."""
    import paper_2412_15840_b200 as nds
    from paper_2412_15840_b200.distributed import Comm, ShardedSolver
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("gloo", rank=0, world_size=1)
    dims = (32, 16, 48)
    us, ts, b = _problem(dims, 9)
    x_ref, _ = oracle.Port().solve_schur(us, ts, b, flags=0)
    comm = Comm.nccl(0)
    solver = ShardedSolver(ctx, us, ts, comm)
    db = torch.from_numpy(np.asfortranarray(b).reshape(-1, order="F").copy()).cuda()
    dx = torch.empty_like(db)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    solver.solve(db, dx)
    torch.cuda.synchronize()
    ctx.set_stream(None)
    x = dx.cpu().numpy().reshape(dims, order="F")
    assert np.max(np.abs(x - x_ref)) / np.max(np.abs(x_ref)) <= 1e-12
    solver.close()
    comm.close()
    x2 = nds.solve_multi([0], us, ts, b)
    assert np.max(np.abs(x2 - x_ref)) / np.max(np.abs(x_ref)) <= 1e-12


@pytest.mark.gpu
def test_rectangular_update_kernels(ctx):
    """nds_dev_mode_update (GEMM and direct variants, incl. K = 8 GEMMs) against numpy."""
    rng = np.random.default_rng(5)
    for shape, mode, rows in [((40, 20, 3), 1, 7), ((6, 40, 5), 2, 33), ((3, 5, 64), 3, 17), ((2, 3, 4), 2, 2),
                              ((16, 16, 8), 3, 40), ((8, 8, 8), 1, 64)]:
        x0 = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        m = rng.standard_normal((rows, shape[mode - 1])) + 1j * rng.standard_normal((rows, shape[mode - 1]))
        out_shape = list(shape)
        out_shape[mode - 1] = rows
        acc0 = rng.standard_normal(out_shape) + 1j * rng.standard_normal(out_shape)
        dx = torch.from_numpy(x0.reshape(-1, order="F").copy()).cuda()
        dacc = torch.from_numpy(acc0.reshape(-1, order="F").copy()).cuda()
        ctx.dev_mode_update(shape, mode, m, dx.data_ptr(), dacc.data_ptr())
        torch.cuda.synchronize()
        got = dacc.cpu().numpy().reshape(out_shape, order="F")
        want = acc0 + np.moveaxis(np.tensordot(m, x0, axes=([1], [mode - 1])), 0, mode - 1)
        assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
