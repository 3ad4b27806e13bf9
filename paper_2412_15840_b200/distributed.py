"""Multi-GPU solve: one process per GPU, torch.distributed (NCCL over NVLink) for the exchanges.

SURVEY.md 8(e). The transforms shard naturally; the triangular solve does not.

Layouts (every local tensor is column-major complex128, flattened):
  L_N: rank r owns the slab of mode N  [sN_r, sN_r + mN_r)   -> local dims (n_1, ..., n_{N-1}, mN_r)
  L_1: rank q owns the slab of mode 1  [s1_q, s1_q + m1_q)   -> local dims (m1_q, n_2, ..., n_N)

solve(B in L_N):
  1. forward, modes 1..N-1: local (each mode product is independent across mode-N slabs);
  2. all-to-all re-shard L_N -> L_1 (the only exchange of the transform);
  3. forward, mode N: local in L_1;
  4. triangular solve, pipelined over (rank, sub-block): each rank's L_1 slab is cut into K
     contiguous sub-blocks along mode N (the slowest index). Block (q, k) needs
       - the mode-1 couplings  C_q[k] -= T_1[q rows, q' cols] x_1 Y_q'[k]  from every q' > q
         (T_1 is dense upper triangular, so rank q needs every higher rank, not only q + 1),
         received point-to-point as soon as rank q' has solved its block k;
       - the mode-N couplings from its own blocks k' > k, applied by rank q right after solving
         k':  C_q[:s_k'] -= T_N[:s_k', k' cols] x_N Y_q[k']  (one rectangular update);
     then the local solve with T_1 and T_N restricted to their diagonal blocks. Blocks form a
     wavefront over (P-1-q) + (K-1-k): P + K - 1 waves instead of P serial slab solves;
  5. inverse, modes 2..N: local in L_1;
  6. all-to-all re-shard L_1 -> L_N;
  7. inverse, mode 1: local in L_N.  X is returned in the input layout L_N.

The per-rank compute goes through `LocalOps`; `CudaLocalOps` calls the C ABI kernels on the
rank's GPU. Tests substitute a CPU implementation to exercise the orchestration with gloo.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def block_partition(n: int, parts: int):
    """Contiguous block split of range(n): (starts, sizes), earlier parts one larger."""
    base, extra = divmod(n, parts)
    sizes = [base + (1 if r < extra else 0) for r in range(parts)]
    starts = [sum(sizes[:r]) for r in range(parts)]
    return starts, sizes


class CudaLocalOps:
    """Local compute on this rank's GPU through the ndsylv_b200 C ABI (device pointers)."""

    def __init__(self, ctx):
        self.ctx = ctx
        # one stream for the C ABI kernels and torch/NCCL: received blocks are read in stream order
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)

    def zeros(self, count, like):
        return torch.zeros(count, dtype=torch.complex128, device=like.device)

    def mode_product(self, dims, m, mode, x):
        out = torch.empty(int(np.prod(dims)), dtype=torch.complex128, device=x.device)
        self.ctx.dev_mode_apply(dims, mode, m, x.data_ptr(), out.data_ptr())
        return out

    def mode_update(self, dims_x, mode, m, x, acc):
        """acc += m x_mode x (m rectangular, host)."""
        self.ctx.dev_mode_update(dims_x, mode, m, x.data_ptr(), acc.data_ptr())

    def back_substitute(self, ts, dims, c, tol):
        self.ctx.dev_back_substitute(ts, dims, c.data_ptr(), tol)

    def synchronize(self):
        torch.cuda.synchronize()


def _exchange(send_blocks, recv_sizes, group):
    """Uneven all-to-all of complex128 blocks (sent as float64 pairs)."""
    send = torch.cat([b.reshape(-1) for b in send_blocks]) if send_blocks else torch.empty(0, dtype=torch.complex128)
    send_r = torch.view_as_real(send.contiguous()).reshape(-1)
    recv_r = torch.empty(2 * sum(recv_sizes), dtype=torch.float64, device=send_r.device)
    dist.all_to_all_single(recv_r, send_r, [2 * s for s in recv_sizes], [2 * b.numel() for b in send_blocks],
                           group=group)
    recv = torch.view_as_complex(recv_r.reshape(-1, 2))
    out, off = [], 0
    for s in recv_sizes:
        out.append(recv[off:off + s])
        off += s
    return out


class ShardedSolver:
    """Distributed solve of sum_j A_j x_j X = B from host Schur factors (same on every rank)."""

    def __init__(self, dims, us, ts, ops, group=None, singular_tol=0.0, sub_blocks=None):
        self.dims = tuple(int(d) for d in dims)
        self.N = len(self.dims)
        if self.N < 2:
            raise ValueError("problem order must be at least 2")
        self.us = [np.asfortranarray(u, dtype=np.complex128) for u in us]
        self.ts = [np.asfortranarray(t, dtype=np.complex128) for t in ts]
        self.uhs = [np.asfortranarray(u.conj().T) for u in self.us]
        self.ops = ops
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        n1, nN = self.dims[0], self.dims[-1]
        if n1 < self.P or nN < self.P:
            raise ValueError("n_1 and n_N must be >= the number of ranks")
        self.s1, self.m1 = block_partition(n1, self.P)
        self.sN, self.mN = block_partition(nN, self.P)
        # pipeline depth along mode N (K sub-blocks per rank)
        k = sub_blocks if sub_blocks is not None else 4 * self.P if self.P > 1 else 1
        self.sK, self.mK = block_partition(nN, max(1, min(int(k), nN)))
        # sylvester.cpp:29-33 — the tolerance of the WHOLE operator, not of a slab
        self.tol = singular_tol if singular_tol > 0 else np.finfo(float).eps * sum(np.linalg.norm(t) for t in self.ts)

    # local dims
    def dims_LN(self, r):
        return self.dims[:-1] + (self.mN[r],)

    def dims_L1(self, q):
        return (self.m1[q],) + self.dims[1:]

    def reshard_N_to_1(self, x):
        """x: this rank's L_N slab -> this rank's L_1 slab."""
        r, n1 = self.rank, self.dims[0]
        rows = x.reshape(-1, n1)  # column-major: mode 1 fastest
        send = [rows[:, self.s1[q]:self.s1[q] + self.m1[q]].contiguous() for q in range(self.P)]
        rest = int(np.prod(self.dims[1:-1]))
        recv_sizes = [self.m1[r] * rest * self.mN[src] for src in range(self.P)]
        blocks = _exchange(send, recv_sizes, self.group)
        return torch.cat(blocks)  # mode N is the slowest index: source slabs concatenate in order

    def reshard_1_to_N(self, y):
        """y: this rank's L_1 slab -> this rank's L_N slab."""
        r, nN = self.rank, self.dims[-1]
        planes = y.reshape(nN, -1)  # column-major: mode N slowest
        send = [planes[self.sN[q]:self.sN[q] + self.mN[q]].contiguous() for q in range(self.P)]
        rest = int(np.prod(self.dims[1:-1]))
        recv_sizes = [self.m1[src] * rest * self.mN[r] for src in range(self.P)]
        blocks = _exchange(send, recv_sizes, self.group)
        n1 = self.dims[0]
        out = torch.empty(n1 * rest * self.mN[r], dtype=y.dtype, device=y.device)
        o_rows = out.reshape(-1, n1)
        for src, blk in enumerate(blocks):
            o_rows[:, self.s1[src]:self.s1[src] + self.m1[src]] = blk.reshape(-1, self.m1[src])
        return out

    def solve(self, b_local):
        """b_local: this rank's L_N slab of B. Returns this rank's L_N slab of X."""
        ops, r, N = self.ops, self.rank, self.N
        # 1. forward, modes 1..N-1 (local in L_N)
        x = b_local
        for j in range(1, N):
            x = ops.mode_product(self.dims_LN(r), self.uhs[j - 1], j, x)
        # 2. re-shard, 3. mode N (local in L_1)
        c = self.reshard_N_to_1(x)
        c = ops.mode_product(self.dims_L1(r), self.uhs[N - 1], N, c)
        # 4. triangular solve pipelined over (rank, mode-N sub-block)
        self.pipelined_backsub(c)
        # 5. inverse, modes 2..N (local in L_1), 6. re-shard, 7. mode 1 (local in L_N)
        y = c
        for j in range(2, N + 1):
            y = ops.mode_product(self.dims_L1(r), self.us[j - 1], j, y)
        x = self.reshard_1_to_N(y)
        return ops.mode_product(self.dims_LN(r), self.us[0], 1, x)

    def _global(self, q):
        return q if self.group is None else dist.get_global_rank(self.group, q)

    def pipelined_backsub(self, c):
        """Step 4 in place on this rank's L_1 slab c (see the module docstring)."""
        ops, r, N, P = self.ops, self.rank, self.N, self.P
        t1, tN = self.ts[0], self.ts[-1]
        s1, m1 = self.s1[r], self.m1[r]
        mid = int(np.prod(self.dims[1:-1]))
        plane = m1 * mid  # entries per mode-N index in this rank's slab
        pending = []  # (work, tensor): sends stay alive until the end
        for k in reversed(range(len(self.mK))):
            sk, mk = self.sK[k], self.mK[k]
            blk = c[sk * plane:(sk + mk) * plane]
            # mode-1 couplings from every higher rank's block k
            for q in range(P - 1, r, -1):
                yq = torch.empty(self.m1[q] * mid * mk, dtype=c.dtype, device=c.device)
                yr = torch.view_as_real(yq)
                dist.recv(yr, src=self._global(q), group=self.group)
                m = -np.asfortranarray(t1[s1:s1 + m1, self.s1[q]:self.s1[q] + self.m1[q]])
                ops.mode_update((self.m1[q],) + self.dims[1:-1] + (mk,), 1, m, yq, blk)
            # local solve: T_1 and T_N restricted to their diagonal blocks
            ts_local = [np.asfortranarray(t1[s1:s1 + m1, s1:s1 + m1])] + self.ts[1:-1] + \
                       [np.asfortranarray(tN[sk:sk + mk, sk:sk + mk])]
            ops.back_substitute(ts_local, (m1,) + self.dims[1:-1] + (mk,), blk, self.tol)
            # forward the solved block to every lower rank (point-to-point, non-blocking)
            if r > 0:
                ops.synchronize()
                br = torch.view_as_real(blk)
                for q in range(r - 1, -1, -1):
                    pending.append((dist.isend(br, dst=self._global(q), group=self.group), br))
            # mode-N couplings of this block into the lower sub-blocks of this rank
            if sk > 0:
                m = -np.asfortranarray(tN[:sk, sk:sk + mk])
                ops.mode_update((m1,) + self.dims[1:-1] + (mk,), N, m, blk, c[:sk * plane])
        for w, _ in pending:
            w.wait()


def scatter_LN(b, P):
    """Split a full column-major tensor (numpy, shape dims) into the L_N slabs (host helper)."""
    nN = b.shape[-1]
    s, m = block_partition(nN, P)
    flat = np.asfortranarray(b).reshape(-1, order="F")
    plane = int(np.prod(b.shape[:-1]))
    return [flat[s[r] * plane:(s[r] + m[r]) * plane].copy() for r in range(P)]


def gather_LN(slabs, dims):
    return np.concatenate([np.asarray(s) for s in slabs]).reshape(dims, order="F")
