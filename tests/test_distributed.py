"""Multi-rank orchestration of the sharded solver (paper_2412_15840_b200/distributed.py) on CPU
with the gloo backend: L_N / L_1 re-shards (uneven all-to-all), slab-pipelined triangular solve
with rectangular cross-slab updates, and the distributed result against the single-process C
oracle. The per-rank compute uses a CPU LocalOps built on the oracle (test-only); on GPUs the
same orchestration runs CudaLocalOps (C ABI kernels) with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2412_15840_b200.distributed import ShardedSolver, block_partition, gather_LN, scatter_LN


def _mode_product_np(x, dims, m, mode):
    X = x.numpy().reshape(dims, order="F")
    R = np.moveaxis(np.tensordot(m, X, axes=([1], [mode - 1])), 0, mode - 1)
    return torch.from_numpy(np.asfortranarray(R).reshape(-1, order="F").copy())


class CpuOps:
    """Test-only LocalOps: numpy mode products and the C oracle's back_substitute."""

    def __init__(self):
        self.port = oracle.Port()

    def mode_product(self, dims, m, mode, x):
        return _mode_product_np(x, dims, m, mode)

    def mode_update(self, dims_x, mode, m, x, acc):
        acc += _mode_product_np(x, dims_x, m, mode)

    def back_substitute(self, ts, dims, c, tol):
        y, _ = self.port.back_substitute(ts, c.numpy().reshape(dims, order="F"), tol)
        c.copy_(torch.from_numpy(y.reshape(-1, order="F").copy()))

    def synchronize(self):
        pass


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dims, seed, out_dir, sub_blocks=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(seed)
    us, ts = [], []
    for n in dims:
        q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        t = np.triu(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
        t[np.diag_indices(n)] = 2.0 + 0.3 * rng.standard_normal(n) + 0.3j * rng.standard_normal(n)
        us.append(q)
        ts.append(t)
    b = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    slabs = scatter_LN(b, world)
    solver = ShardedSolver(dims, us, ts, CpuOps(), sub_blocks=sub_blocks)
    x_local = solver.solve(torch.from_numpy(slabs[rank]))
    np.save(os.path.join(out_dir, f"x{rank}.npy"), x_local.numpy())
    if rank == 0:
        np.savez(os.path.join(out_dir, "problem.npz"), b=b, **{f"u{j}": u for j, u in enumerate(us)},
                 **{f"t{j}": t for j, t in enumerate(ts)})
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,sub_blocks", [(2, (6, 5, 8), None), (3, (7, 4, 5), None), (2, (4, 3, 2, 5), None),
                                                  (3, (5, 6), None), (2, (6, 5, 8), 1), (3, (7, 4, 9), 9),
                                                  (2, (5, 3, 7), 3)])
def test_sharded_solve_matches_oracle(tmp_path, world, dims, sub_blocks):
    # sub_blocks: pipeline depth along mode N (None = 4 per rank, 1 = serial slabs, n_N = one
    # mode-N index per block)
    port = _free_port()
    mp.spawn(_worker, args=(world, port, dims, 123, str(tmp_path), sub_blocks), nprocs=world, join=True)
    z = np.load(tmp_path / "problem.npz")
    n = len(dims)
    us = [z[f"u{j}"] for j in range(n)]
    ts = [z[f"t{j}"] for j in range(n)]
    x = gather_LN([np.load(tmp_path / f"x{r}.npy") for r in range(world)], dims)
    x_ref, _ = oracle.Port().solve_schur(us, ts, z["b"], flags=0)
    assert np.max(np.abs(x - x_ref)) / np.max(np.abs(x_ref)) <= 1e-12


def test_block_partition():
    assert block_partition(8, 3) == ([0, 3, 6], [3, 3, 2])
    assert block_partition(4, 4) == ([0, 1, 2, 3], [1, 1, 1, 1])
    s, m = block_partition(256, 8)
    assert sum(m) == 256 and all(v == 32 for v in m)


@pytest.mark.gpu
def test_cuda_local_ops_single_rank(ctx):
    """The GPU LocalOps (C ABI device kernels) under the same orchestration, 1 rank, NCCL."""
    from paper_2412_15840_b200.distributed import CudaLocalOps
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1)
    rng = np.random.default_rng(5)
    dims = (24, 20, 32)
    us, ts = [], []
    for n in dims:
        q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        t = np.triu(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
        t[np.diag_indices(n)] = 2.0 + 0.3 * rng.standard_normal(n)
        us.append(np.asfortranarray(q))
        ts.append(np.asfortranarray(t))
    b = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    x_ref, _ = oracle.Port().solve_schur(us, ts, b, flags=0)
    for k in (1, 5):  # whole slab, and 5 mode-N sub-blocks (device mode-N coupling updates)
        solver = ShardedSolver(dims, us, ts, CudaLocalOps(ctx), sub_blocks=k)
        x = solver.solve(torch.from_numpy(scatter_LN(b, 1)[0]).cuda()).cpu().numpy().reshape(dims, order="F")
        assert np.max(np.abs(x - x_ref)) / np.max(np.abs(x_ref)) <= 1e-12
    # rectangular update kernel (GEMM and direct variants) against numpy
    for shape, mode, rows in [((40, 20, 3), 1, 7), ((6, 40, 5), 2, 33), ((3, 5, 64), 3, 17), ((2, 3, 4), 2, 2)]:
        x0 = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        m = rng.standard_normal((rows, shape[mode - 1])) + 1j * rng.standard_normal((rows, shape[mode - 1]))
        out_shape = list(shape)
        out_shape[mode - 1] = rows
        acc0 = rng.standard_normal(out_shape) + 1j * rng.standard_normal(out_shape)
        dx = torch.from_numpy(x0.reshape(-1, order="F").copy()).cuda()
        dacc = torch.from_numpy(acc0.reshape(-1, order="F").copy()).cuda()
        ctx.dev_mode_update(shape, mode, m, dx.data_ptr(), dacc.data_ptr())
        got = dacc.cpu().numpy().reshape(out_shape, order="F")
        want = acc0 + np.moveaxis(np.tensordot(m, x0, axes=([1], [mode - 1])), 0, mode - 1)
        assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
