"""Multi-GPU sharded solve: one rank per GPU.

The product path is the C-ABI engine (`nds_dist_*`, csrc/sharded.cuh): per rank, the
transforms in layout L_N / L_1 with one all-to-all each way, and the triangular solve pipelined
over (rank, block of the last modes) with point-to-point forwarding of solved blocks — NCCL P2P
on the rank's communication stream, stream-ordered against its compute stream (no host sync).
`ShardedSolver` drives it from Python (torchrun: one process per GPU; the NCCL unique id is
broadcast through the torch.distributed group).

`plan_layout` mirrors the engine's mode groups and partitions (checked against `nds_dist_info`
by the GPU tests), and `HostShardedSolver` runs the SAME schedule with host tensors over any
torch.distributed backend — the gloo tests (tests/test_distributed.py) cover the multi-rank
orchestration on CPU with it.

Layouts (column-major complex128 slabs):
  L_N: rank r owns tail super-indices [sG_r, sG_r + mG_r) of the last g modes (g = 1: a block of
       mode N; all-binary problems: g = log2 P modes, one index each) — a contiguous range of the
       full tensor;
  L_1: rank q owns head super-indices [sH_q, sH_q + mH_q) of the first h modes (h = g).
Solve (B and X in L_N): forward modes outside the tail group (local) -> all-to-all L_N -> L_1 ->
forward tail modes (local) -> pipelined triangular solve -> inverse modes outside the head group
(local) -> all-to-all L_1 -> L_N -> inverse head modes (local).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist


def block_partition(n: int, parts: int):
    """Contiguous block split of range(n): (starts, sizes), earlier parts one larger."""
    base, extra = divmod(n, parts)
    sizes = [base + (1 if r < extra else 0) for r in range(parts)]
    starts = [sum(sizes[:r]) for r in range(parts)]
    return starts, sizes


@dataclass
class Layout:
    """Mode groups and partitions of the sharded solve (mirror of choose_groups, sharded.cuh)."""
    dims: tuple
    P: int
    h: int = 1
    g: int = 1
    gp: int = 1
    sH: list = field(default_factory=list)
    mH: list = field(default_factory=list)
    sG: list = field(default_factory=list)
    mG: list = field(default_factory=list)
    sK: list = field(default_factory=list)
    mK: list = field(default_factory=list)

    @property
    def N(self):
        return len(self.dims)

    def couples(self, lo, hi):
        """Rank `lo` needs rank `hi`'s solved blocks (structural nonzero of T_H[lo, hi])."""
        if hi <= lo:
            return False
        if self.h == 1:
            return self.mH[lo] > 0 and self.mH[hi] > 0
        a, b = self.sH[lo], self.sH[hi]
        return bin(a ^ b).count("1") == 1 and (b & ~a) != 0

    def ln_dims(self, r):
        N = self.N
        return tuple(self.dims[j] if j < N - self.g else (self.mG[r] if self.g == 1 else 1) for j in range(N))

    def l1_dims(self, q):
        return tuple(self.dims[j] if j >= self.h else (self.mH[q] if self.h == 1 else 1) for j in range(self.N))

    def slab(self, r):
        """(flat offset, count) of rank r's L_N slab in the full column-major tensor."""
        head = int(np.prod(self.dims[:self.N - self.g]))
        return self.sG[r] * head, self.mG[r] * head

    def mid(self, hi):
        return int(np.prod(self.dims[self.h:hi], dtype=np.int64)) if hi > self.h else 1

    def alltoall_bytes(self, q):
        Mg = self.mid(self.N - self.g)
        return sum(16 * (self.mH[r] * Mg * self.mG[q] + self.mH[q] * Mg * self.mG[r]) for r in range(self.P) if r != q)

    def pipeline_bytes(self, q):
        Mp = self.mid(self.N - self.gp)
        nK = int(np.prod(self.dims[self.N - self.gp:]))
        return 16 * self.mH[q] * Mp * nK * sum(self.couples(qq, q) for qq in range(q))


def plan_layout(dims, P) -> Layout:
    dims = tuple(int(d) for d in dims)
    N = len(dims)
    L = Layout(dims, P)
    binary = all(d == 2 for d in dims)
    if P > 64:
        raise ValueError("at most 64 ranks")
    if P > 1 and binary:
        k = P.bit_length() - 1
        if 1 << k != P:
            raise ValueError("all-binary problems shard over a power-of-two rank count")
        if 2 * k > N - 1:
            raise ValueError("too few binary modes for this rank count")
        L.h = L.g = k
        L.gp = max(1, min(k + 1, N - k - 1))
    elif P > 1 and (dims[0] < P or dims[-1] < P):
        raise ValueError("the first and last extents must be at least the number of ranks")
    nH = int(np.prod(dims[:L.h]))
    nG = int(np.prod(dims[N - L.g:]))
    nK = int(np.prod(dims[N - L.gp:]))
    L.sH, L.mH = block_partition(nH, P)
    L.sG, L.mG = block_partition(nG, P)
    K = 1
    if P > 1:
        if binary:
            K = nK
        else:
            edge = 16 if N == 3 else 8
            K = next((c for c in range(min(4 * P, nK), 1, -1) if nK % c == 0 and (nK // c) % edge == 0), 1)
            if K == 1:  # no whole-tile blocking: pipeline anyway
                K = min(2 * P, nK)
    L.sK, L.mK = block_partition(nK, K)
    return L


def kron_sum(ts, dims):
    """Kronecker sum of the T_j of consecutive modes on their column-major super-index."""
    n = int(np.prod(dims))
    out = np.zeros((n, n), dtype=np.complex128)
    acc = 1
    for t, d in zip(ts, dims):
        left = np.eye(acc)
        right = np.eye(n // (acc * d))
        out += np.kron(right, np.kron(t, left))  # column-major: earlier modes vary fastest
        acc *= d
    return out


# ---- the C-ABI engine (product path on GPUs) ----------------------------------------------------

class Comm:
    """An nds_comm handle: NCCL (one rank per GPU) or the in-process loopback (tests)."""

    def __init__(self, lib, handle):
        self.lib, self.h = lib, handle

    @staticmethod
    def nccl(device: int, group=None):
        """NCCL communicator over the ranks of a torch.distributed group (unique id broadcast)."""
        from . import load_library
        lib = load_library()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        buf = (C.c_uint8 * 128)()
        if rank == 0 and lib.nds_comm_unique_id(buf) != 0:
            raise RuntimeError(lib.nds_last_error(None).decode())
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        if lib.nds_comm_create_nccl(C.byref(h), int(device), rank, world, uid) != 0:
            raise RuntimeError(lib.nds_last_error(None).decode())
        return Comm(lib, h)

    @staticmethod
    def loopback(world: int):
        from . import load_library
        lib = load_library()
        arr = (C.c_void_p * world)()
        if lib.nds_comm_create_loopback(int(world), arr) != 0:
            raise RuntimeError(lib.nds_last_error(None).decode())
        return [Comm(lib, C.c_void_p(arr[r])) for r in range(world)]

    def close(self):
        if self.h:
            self.lib.nds_comm_destroy(self.h)
            self.h = None


class ShardedSolver:
    """One rank of the sharded solve on its GPU (nds_dist_*): `solve(d_b, d_x)` with this rank's
    L_N slabs as device pointers (or torch tensors), asynchronous on the context stream."""

    def __init__(self, ctx, us, ts, comm: Comm | None = None, singular_tol=0.0):
        from . import _dims, _ptr_array, _Singular, SingularOperatorError, NdsError, ERR_SINGULAR
        self.ctx = ctx
        self.dims = tuple(int(u.shape[0]) for u in us)
        up, self._ku = _ptr_array(us)
        tp, self._kt = _ptr_array(ts)
        self.comm = comm
        h = C.c_void_p()
        sing = _Singular()
        rc = ctx.lib.nds_dist_create(ctx.h, comm.h if comm else None, len(self.dims), _dims(self.dims), up, tp,
                                     float(singular_tol), C.byref(h), C.byref(sing))
        if rc == ERR_SINGULAR:
            raise SingularOperatorError(ctx.last_error(), sing.multi_index[:sing.n_modes],
                                        complex(sing.den_re, sing.den_im))
        if rc:
            raise NdsError(rc, ctx.last_error())
        self.h = h

    def slab(self, rank: int):
        off, cnt = C.c_int64(), C.c_int64()
        self.ctx.lib.nds_dist_slab(self.h, int(rank), C.byref(off), C.byref(cnt))
        return off.value, cnt.value

    def info(self) -> dict:
        from . import _DistInfo
        i = _DistInfo()
        self.ctx.lib.nds_dist_info(self.h, C.byref(i))
        return {k: getattr(i, k) for k, _ in _DistInfo._fields_}

    def solve(self, d_b, d_x):
        from . import NdsError
        pb = d_b.data_ptr() if hasattr(d_b, "data_ptr") else int(d_b)
        px = d_x.data_ptr() if hasattr(d_x, "data_ptr") else int(d_x)
        rc = self.ctx.lib.nds_dist_solve(self.h, pb, px)
        if rc:
            raise NdsError(rc, self.ctx.last_error())

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.nds_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- host mirror of the engine's schedule (gloo tests) ------------------------------------------

class HostShardedSolver:
    """The engine's schedule (sharded.cuh dist_solve_impl) on host tensors over torch.distributed,
    with the per-rank compute supplied by `ops` (mode_product(dims, m, mode, x),
    back_substitute(ts, dims, c, tol)). Same layout, couplings, folding and block order."""

    def __init__(self, dims, us, ts, ops, group=None, singular_tol=0.0):
        self.dims = tuple(int(d) for d in dims)
        self.N = len(self.dims)
        if self.N < 2:
            raise ValueError("problem order must be at least 2")
        self.us = [np.asarray(u, dtype=np.complex128) for u in us]
        self.ts = [np.asarray(t, dtype=np.complex128) for t in ts]
        self.uhs = [u.conj().T.copy() for u in self.us]
        self.ops, self.group = ops, group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.L = plan_layout(self.dims, self.P)
        self.tol = singular_tol if singular_tol > 0 else np.finfo(float).eps * sum(np.linalg.norm(t) for t in self.ts)
        L, N = self.L, self.N
        self.TH = kron_sum(self.ts[:L.h], self.dims[:L.h])
        self.TK = kron_sum(self.ts[N - L.gp:], self.dims[N - L.gp:])

    def _g(self, q):
        return q if self.group is None else dist.get_global_rank(self.group, q)

    def _apply(self, d, lo, hi, adjoint, x):
        for j in range(lo, hi + 1):
            x = self.ops.mode_product(d, self.uhs[j - 1] if adjoint else self.us[j - 1], j, x)
        return x

    def _exchange(self, send, recv):
        """send/recv: per peer flat complex tensors (views into contiguous buffers)."""
        ops = []
        for r in range(self.P):
            if r == self.rank:
                continue
            if send[r].numel():
                ops.append(dist.P2POp(dist.isend, torch.view_as_real(send[r]).contiguous(), self._g(r), self.group))
            if recv[r].numel():
                ops.append(dist.P2POp(dist.irecv, recv[r], self._g(r), self.group))
        bufs = [op.tensor for op in ops if op.op is dist.irecv]
        for w in dist.batch_isend_irecv(ops) if ops else []:
            w.wait()
        return bufs

    def solve(self, b_local):
        L, q, N, P = self.L, self.rank, self.N, self.P
        lnd, l1d = L.ln_dims(q), L.l1_dims(q)
        Mg, Mp = L.mid(N - L.g), L.mid(N - L.gp)
        x = self._apply(lnd, 1, N - L.g, True, b_local)
        # L_N -> L_1: pack rows [sH_r, sH_r + mH_r) of the head index for rank r
        nH = int(np.prod(self.dims[:L.h]))
        rows = x.reshape(-1, nH)
        send = [rows[:, L.sH[r]:L.sH[r] + L.mH[r]].reshape(-1).contiguous() for r in range(P)]
        l1 = torch.empty(int(np.prod(l1d)), dtype=torch.complex128)
        plane_g = L.mH[q] * Mg
        recv = [torch.empty(2 * L.mH[q] * Mg * L.mG[r], dtype=torch.float64) for r in range(P)]
        self._exchange(send, recv)
        for r in range(P):
            piece = send[q] if r == q else torch.view_as_complex(recv[r].reshape(-1, 2))
            l1[L.sG[r] * plane_g:(L.sG[r] + L.mG[r]) * plane_g] = piece
        c = self._apply(l1d, N - L.g + 1, N, True, l1)
        self._pipelined_backsub(c, Mp)
        y = self._apply(l1d, L.h + 1, N, False, c)
        # L_1 -> L_N
        send = [y[L.sG[r] * plane_g:(L.sG[r] + L.mG[r]) * plane_g].contiguous() for r in range(P)]
        recv = [torch.empty(2 * L.mH[r] * Mg * L.mG[q], dtype=torch.float64) for r in range(P)]
        self._exchange(send, recv)
        out = torch.empty(int(np.prod(lnd)), dtype=torch.complex128)
        o_rows = out.reshape(-1, nH)
        for r in range(P):
            piece = send[q] if r == q else torch.view_as_complex(recv[r].reshape(-1, 2))
            o_rows[:, L.sH[r]:L.sH[r] + L.mH[r]] = piece.reshape(-1, L.mH[r])
        return self._apply(lnd, 1, L.h, False, out)

    def _local_ts(self, k):
        """T blocks of block k's local solve, extent-1 modes folded into the first other mode."""
        L, q, N = self.L, self.rank, self.N
        ext, tb = [], []
        for j in range(N):
            n, s0, m = self.dims[j], 0, self.dims[j]
            if j < L.h:
                s0, m = (L.sH[q], L.mH[q]) if L.h == 1 else ((L.sH[q] // int(np.prod(self.dims[:j]))) % n, 1)
            elif j >= N - L.gp:
                s0, m = (L.sK[k], L.mK[k]) if L.gp == 1 else \
                    ((L.sK[k] // int(np.prod(self.dims[N - L.gp:j]))) % n, 1)
            ext.append(m)
            tb.append(self.ts[j][s0:s0 + m, s0:s0 + m])
        keep = [j for j in range(N) if ext[j] > 1]
        fold = sum(tb[j][0, 0] for j in range(N) if ext[j] == 1)
        if not keep:
            return (1,), [np.array([[fold]])]
        lt = [np.array(tb[j], dtype=np.complex128) for j in keep]
        lt[0] = lt[0] + fold * np.eye(ext[keep[0]])
        return tuple(ext[j] for j in keep), lt

    def _pipelined_backsub(self, c, Mp):
        L, q, P = self.L, self.rank, self.P
        plane = L.mH[q] * Mp
        higher = [qp for qp in range(P - 1, q, -1) if L.couples(q, qp)]
        lower = [qq for qq in range(q - 1, -1, -1) if L.couples(qq, q)]
        K = len(L.sK)
        for k in reversed(range(K)):
            blk = c[L.sK[k] * plane:(L.sK[k] + L.mK[k]) * plane]
            recv = []
            for qp in higher:
                t = torch.empty(2 * L.mH[qp] * Mp * L.mK[k], dtype=torch.float64)
                recv.append(dist.P2POp(dist.irecv, t, self._g(qp), self.group))
            for w in dist.batch_isend_irecv(recv) if recv else []:
                w.wait()
            for qp, op in zip(higher, recv):
                y = torch.view_as_complex(op.tensor.reshape(-1, 2))
                m = -self.TH[L.sH[q]:L.sH[q] + L.mH[q], L.sH[qp]:L.sH[qp] + L.mH[qp]]
                blk += self.ops.mode_product((L.mH[qp], Mp * L.mK[k]), m, 1, y)
            ldims, lts = self._local_ts(k)
            self.ops.back_substitute(lts, ldims, blk, self.tol)
            sends = [dist.P2POp(dist.isend, torch.view_as_real(blk).contiguous(), self._g(qq), self.group)
                     for qq in lower]
            for w in dist.batch_isend_irecv(sends) if sends else []:
                w.wait()
            if k > 0:  # pipe couplings into the lower blocks of this rank
                m = -self.TK[:L.sK[k], L.sK[k]:L.sK[k] + L.mK[k]]
                c[:L.sK[k] * plane] += self.ops.mode_product((plane, L.mK[k]), m, 2, blk)


def scatter_LN(b, P):
    """Split a full column-major tensor (numpy, shape dims) into the L_N slabs (host helper)."""
    L = plan_layout(b.shape, P)
    flat = np.asfortranarray(b).reshape(-1, order="F")
    return [flat[o:o + n].copy() for o, n in (L.slab(r) for r in range(P))]


def gather_LN(slabs, dims):
    return np.concatenate([np.asarray(s) for s in slabs]).reshape(dims, order="F")
