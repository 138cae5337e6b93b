"""Slab mode: one 3-D field sharded along axis 0 over R ranks.

The reference has no distributed path: this runs its decompose / recompose
(transform.hpp:485-530) for a field whose axis-0 planes are split into R
slabs, one per GPU, with the exchange steps the level passes need:

* the plane passes read a halo of fine planes (two on the left, one on the
  right) around a rank's slab (`Exchange.halo`);
* the axis-0 Thomas solve (batched_solve, transform.hpp:116-130) needs whole
  axis-0 columns, so the fp64 load-vector volume G of the level is
  transposed (all-to-all: each rank gets every plane of 1/R of the columns),
  solved, and transposed back (`Exchange.transpose`, `.transpose_back`);
  the correction is then applied to the rank's coarse planes;
* recompose's interpolation reads the right neighbour's first corrected
  coarse plane (`Exchange.halo`, right side only);
* below the slab levels the coarse block is gathered (`Exchange.gather`) and
  the remaining levels run on every rank (they are small).

Slab boundaries sit at multiples of 2^S fine planes (S slab levels), so they
stay on nodal planes of every slab level.  Every per-rank buffer is
full-size and globally indexed; a rank writes its own planes only.  The
level passes are the C-ABI's mgrx_gpu_slab_* entry points (sm_100a
kernels); the results are bit-identical to the single-GPU decompose /
recompose (the same per-element arithmetic; tests/test_slab.py).

Two exchanges: `TorchExchange` (torch.distributed: NCCL between GPUs, or
gloo for the CPU tests of the data movement) with one local rank per
process, and `LocalExchange`, which runs all R ranks in one process (on one
GPU) with device copies — the emulation the single-GPU tests use.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

from . import GridHierarchy, MultilevelCoefficients, SolverWorkspace, _check, _dims_arr, _dtype_code, decompose, \
    recompose
from ._lib import lib


# --------------------------------------------------------------- partition

def slab_bounds(n0: int, ranks: int, slab_levels: int) -> List[int]:
    """Fine-plane boundaries P_0 = 0 < ... < P_R = n0 - 1 at the finest level,
    multiples of 2^slab_levels (rank r owns planes [P_r, P_{r+1}), the last
    rank also plane n0 - 1)."""
    unit = 1 << slab_levels
    if (n0 - 1) % unit:
        raise ValueError(f"n0 - 1 = {n0 - 1} is not a multiple of 2^{slab_levels}")
    units = (n0 - 1) // unit
    if units < ranks:
        raise ValueError(f"{units} slab units for {ranks} ranks")
    return [(r * units // ranks) * unit for r in range(ranks)] + [n0 - 1]


def shell_plane_range(p: int, info) -> tuple:
    """[start, end) of fine plane p's shell entries in the level-centric
    buffer (pack_level_centric, reorder.hpp:180-215: reordered planes in
    order, an even plane's nodal rows omitted): one contiguous run."""
    n0, n1, n2, m0, m1, m2, _, off = info[:8]
    full, short = n1 * n2, n1 * n2 - m1 * m2
    r0 = p // 2 if p % 2 == 0 else m0 + p // 2
    start = r0 * short if r0 < m0 else m0 * short + (r0 - m0) * full
    return off + start, off + start + (short if r0 < m0 else full)


def column_bounds(ncols: int, ranks: int) -> List[int]:
    return [r * ncols // ranks for r in range(ranks + 1)]


def max_slab_levels(h: GridHierarchy, ranks: int, min_planes: int = 8) -> int:
    """Slab levels S: the finest levels while every rank keeps at least
    `min_planes` coarse planes and 2^S divides n0 - 1."""
    L = h.num_levels()
    n0 = h.level_dims(L)[0]
    S = 0
    while S < L and (n0 - 1) % (1 << (S + 1)) == 0 and ((n0 - 1) >> (S + 1)) >= ranks * min_planes:
        S += 1
    return S


# ---------------------------------------------------------------- exchanges

class LocalExchange:
    """All R ranks in this process (one GPU): exchanges are device copies."""

    def __init__(self, ranks: int):
        self.world = ranks
        self.local = list(range(ranks))

    def halo(self, bufs, plane, bounds, left: int, right: int):
        """bufs[r] (planes, plane elements): rank r receives planes
        [bounds[r] - left, bounds[r]) from rank r - 1 and
        [bounds[r+1], bounds[r+1] + right) from rank r + 1."""
        R = self.world
        for r in range(R):
            if r > 0 and left:
                b = bounds[r]
                bufs[r][b - left:b] = bufs[r - 1][b - left:b]
            if r + 1 < R and right:
                b = bounds[r + 1]
                bufs[r][b:b + right] = bufs[r + 1][b:b + right]

    def halo_ranges(self, bufs, left, right):
        """1-D bufs: rank r receives the element ranges left(r) from rank
        r - 1 and right(r) from rank r + 1 (lists of (start, end))."""
        R = self.world
        for r in range(R):
            if r > 0:
                for a, b in left(r):
                    bufs[r][a:b] = bufs[r - 1][a:b]
            if r + 1 < R:
                for a, b in right(r):
                    bufs[r][a:b] = bufs[r + 1][a:b]

    def transpose(self, G, K, Cb):
        """G[r]: (m0, ncols) with rank r's planes [K[r], K[r+1]) set ->
        Gt[r]: (m0, Cb[r+1] - Cb[r]) full axis-0 columns of rank r."""
        import torch

        R = self.world
        return [torch.cat([G[q][K[q]:K[q + 1], Cb[r]:Cb[r + 1]] for q in range(R)]).contiguous() for r in range(R)]

    def transpose_back(self, Gt, K, Cb):
        """Gt[r] (m0, W_r) -> z[r]: (K[r+1] - K[r], ncols), rank r's planes."""
        import torch

        R = self.world
        return [torch.cat([Gt[q][K[r]:K[r + 1]] for q in range(R)], dim=1).contiguous() for r in range(R)]

    def gather(self, bufs, bounds):
        """Every rank gets every rank's planes [bounds[q], bounds[q+1])."""
        R = self.world
        for r in range(R):
            for q in range(R):
                if q != r:
                    bufs[r][bounds[q]:bounds[q + 1]] = bufs[q][bounds[q]:bounds[q + 1]]


class TorchExchange:
    """One rank per process over torch.distributed (NCCL between GPUs; gloo
    for CPU tensors in the tests).  Same semantics as LocalExchange with the
    lists holding this rank's buffer only."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.local = [self.rank]

    def halo(self, bufs, plane, bounds, left: int, right: int):
        dist, r, R = self.dist, self.rank, self.world
        buf = bufs[0]
        ops = []
        # to the right neighbour: my last `left` planes; to the left: my first `right`
        if r + 1 < R and left:
            b = bounds[r + 1]
            ops.append(dist.P2POp(dist.isend, buf[b - left:b].contiguous(), r + 1, self.group))
        if r > 0 and right:
            b = bounds[r]
            ops.append(dist.P2POp(dist.isend, buf[b:b + right].contiguous(), r - 1, self.group))
        recv = []
        if r > 0 and left:
            b = bounds[r]
            t = buf.new_empty(buf[b - left:b].shape)
            ops.append(dist.P2POp(dist.irecv, t, r - 1, self.group))
            recv.append((slice(b - left, b), t))
        if r + 1 < R and right:
            b = bounds[r + 1]
            t = buf.new_empty(buf[b:b + right].shape)
            ops.append(dist.P2POp(dist.irecv, t, r + 1, self.group))
            recv.append((slice(b, b + right), t))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for sl, t in recv:
            buf[sl] = t

    def halo_ranges(self, bufs, left, right):
        import torch

        dist, r, R = self.dist, self.rank, self.world
        buf = bufs[0]
        ops, recv = [], []
        if r + 1 < R:  # what rank r + 1 wants from its left neighbour
            ops.append(dist.P2POp(dist.isend, torch.cat([buf[a:b] for a, b in left(r + 1)]), r + 1, self.group))
        if r > 0:  # what rank r - 1 wants from its right neighbour
            ops.append(dist.P2POp(dist.isend, torch.cat([buf[a:b] for a, b in right(r - 1)]), r - 1, self.group))
        if r > 0:
            rl = left(r)
            t = buf.new_empty(sum(b - a for a, b in rl))
            ops.append(dist.P2POp(dist.irecv, t, r - 1, self.group))
            recv.append((rl, t))
        if r + 1 < R:
            rr = right(r)
            t = buf.new_empty(sum(b - a for a, b in rr))
            ops.append(dist.P2POp(dist.irecv, t, r + 1, self.group))
            recv.append((rr, t))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for rng, t in recv:
            o = 0
            for a, b in rng:
                buf[a:b] = t[o:o + b - a]
                o += b - a

    def transpose(self, G, K, Cb):
        import torch

        dist, r, R = self.dist, self.rank, self.world
        g = G[0]
        send = torch.cat([g[K[r]:K[r + 1], Cb[q]:Cb[q + 1]].reshape(-1) for q in range(R)])
        W = Cb[r + 1] - Cb[r]
        out = g.new_empty((K[R] - K[0]) * W)
        # output splits: K_q rows x my width from each q; input: my rows x W_q to each q
        dist.all_to_all_single(out, send, [(K[q + 1] - K[q]) * W for q in range(R)],
                               [(K[r + 1] - K[r]) * (Cb[q + 1] - Cb[q]) for q in range(R)], group=self.group)
        return [out.view(K[R] - K[0], W)]

    def transpose_back(self, Gt, K, Cb):
        import torch

        dist, r, R = self.dist, self.rank, self.world
        gt = Gt[0]
        send = torch.cat([gt[K[q]:K[q + 1]].reshape(-1) for q in range(R)])
        rows = K[r + 1] - K[r]
        out = gt.new_empty(rows * Cb[R])
        dist.all_to_all_single(out, send, [rows * (Cb[q + 1] - Cb[q]) for q in range(R)],
                               [(K[q + 1] - K[q]) * (Cb[r + 1] - Cb[r]) for q in range(R)], group=self.group)
        parts, o = [], 0
        for q in range(R):
            w = Cb[q + 1] - Cb[q]
            parts.append(out[o:o + rows * w].view(rows, w))
            o += rows * w
        return [torch.cat(parts, dim=1).contiguous()]

    def gather(self, bufs, bounds):
        dist, R = self.dist, self.world
        buf = bufs[0]
        sizes = [bounds[q + 1] - bounds[q] for q in range(R)]
        mx = max(sizes)
        mine = buf[bounds[self.rank]:bounds[self.rank + 1]]
        pad = buf.new_zeros((mx,) + tuple(buf.shape[1:]))
        pad[:mine.shape[0]] = mine
        got = [buf.new_empty(pad.shape) for _ in range(R)]
        dist.all_gather(got, pad, group=self.group)
        for q in range(R):
            if q != self.rank:
                buf[bounds[q]:bounds[q + 1]] = got[q][:sizes[q]]


# ------------------------------------------------------------------ passes

def _level_info(ws, code, dims, L, level):
    info = (C.c_int64 * 9)()
    _check(lib.mgrx_gpu_slab_level(ws.handle, code, len(dims), _dims_arr(dims), L, level, info), ws.handle)
    return [int(x) for x in info]


def _fused_depth(ws, code, dims, L, limit):
    """Consecutive levels from the finest that run on the fused 3-D path."""
    d = 0
    while d < limit and _level_info(ws, code, dims, L, L - d)[6]:
        d += 1
    return d


def _ptr(t, offset_elems: int = 0):
    return C.c_void_p(t.data_ptr() + offset_elems * t.element_size())


def slab_decompose(fields: Sequence, hierarchy: GridHierarchy, exch, workspaces: Sequence[SolverWorkspace],
                   slab_levels: Optional[int] = None):
    """decompose of a slab-sharded field.  fields[i]: full-size CUDA tensor
    of local rank exch.local[i] holding (at least) its planes
    [P_r, P_{r+1}).  Returns the level-centric buffers (one per local rank):
    each holds the coarse levels (replicated) and its own planes' shells."""
    import torch

    R = exch.world
    h = hierarchy
    L = h.num_levels()
    dims = h.level_dims(L)
    code = _dtype_code(fields[0])
    S = max_slab_levels(h, R) if slab_levels is None else slab_levels
    S = _fused_depth(workspaces[0], code, dims, L, S)
    P = slab_bounds(dims[0], R, S)
    dt, dev = fields[0].dtype, fields[0].device
    # NaN where a rank writes nothing (its buffer then merges by isnan)
    outs = [torch.full((h.total_count(),), float("nan"), dtype=dt, device=dev) for _ in exch.local]
    blk = [f.reshape(f.shape[0], -1) for f in fields]
    for ws in workspaces:
        ws._bind_stream()
    for j in range(S):
        l = L - j
        info = _level_info(workspaces[0], code, dims, L, l)
        n0, m0, m1, m2 = info[0], info[3], info[4], info[5]
        if not info[6]:
            raise ValueError(f"level {l} is not on the fused 3-D path")
        Pf = [p >> j for p in P]
        Pf[R] = n0
        K = [p >> (j + 1) for p in P]
        K[R] = m0
        exch.halo(blk, None, Pf, 2, 1)
        G = [torch.empty((m0, m1 * m2), dtype=torch.float64, device=dev) for _ in exch.local]
        coarse = [torch.empty((m0, m1 * m2), dtype=dt, device=dev) for _ in exch.local]
        for i, r in enumerate(exch.local):
            ws = workspaces[i]
            _check(lib.mgrx_gpu_slab_dec_plane(ws.handle, code, 3, _dims_arr(dims), L, l, K[r], K[r + 1],
                                               _ptr(blk[i]), _ptr(outs[i]), _ptr(coarse[i]), _ptr(G[i])), ws.handle)
            _check(lib.mgrx_gpu_slab_inplane(ws.handle, code, 3, _dims_arr(dims), L, l, K[r], K[r + 1], _ptr(G[i])),
                   ws.handle)
        Cb = column_bounds(m1 * m2, R)
        Gt = exch.transpose(G, K, Cb)
        for i, r in enumerate(exch.local):
            ws = workspaces[i]
            _check(lib.mgrx_gpu_slab_axis0(ws.handle, code, 3, _dims_arr(dims), L, l, Cb[r + 1] - Cb[r], _ptr(Gt[i])),
                   ws.handle)
        z = exch.transpose_back(Gt, K, Cb)
        for i, r in enumerate(exch.local):
            ws = workspaces[i]
            _check(lib.mgrx_gpu_slab_apply(ws.handle, code, _ptr(coarse[i], K[r] * m1 * m2), _ptr(z[i]),
                                           (K[r + 1] - K[r]) * m1 * m2, 1.0), ws.handle)
        blk = coarse
    # the remaining levels: gather the coarse block, decompose it on every rank
    Lc = L - S
    Kc = [p >> S for p in P]
    Kc[R] = h.level_dims(Lc)[0]
    exch.gather(blk, Kc)
    dims_c = h.level_dims(Lc)
    hc = GridHierarchy.create(dims_c, Lc)
    for i in range(len(exch.local)):
        mc = decompose(blk[i].reshape(dims_c), hc, 0, workspaces[i])
        outs[i][:hc.total_count()] = mc.buffer
    return outs


def slab_recompose(coeffs: Sequence, hierarchy: GridHierarchy, exch, workspaces: Sequence[SolverWorkspace],
                   slab_levels: Optional[int] = None):
    """recompose into a slab-sharded field.  coeffs[i]: the level-centric
    buffer on local rank exch.local[i] holding the coarse levels and the
    shells of its own planes (what slab_decompose returns); the shells of
    the halo planes are exchanged here (the buffers are updated in place).  Returns full-size fields (one per
    local rank) holding its planes [P_r, P_{r+1}) (the last rank also n0 - 1)."""
    import torch

    R = exch.world
    h = hierarchy
    L = h.num_levels()
    dims = h.level_dims(L)
    code = _dtype_code(coeffs[0])
    S = max_slab_levels(h, R) if slab_levels is None else slab_levels
    S = _fused_depth(workspaces[0], code, dims, L, S)
    P = slab_bounds(dims[0], R, S)
    dt, dev = coeffs[0].dtype, coeffs[0].device
    for ws in workspaces:
        ws._bind_stream()
    Lc = L - S
    dims_c = h.level_dims(Lc)
    hc = GridHierarchy.create(dims_c, Lc)
    cur = []
    for i in range(len(exch.local)):
        f = recompose(MultilevelCoefficients(coeffs[i][:hc.total_count()], hc, 0), workspaces[i])
        cur.append(f.reshape(dims_c[0], -1))
    for j in reversed(range(S)):
        l = L - j
        info = _level_info(workspaces[0], code, dims, L, l)
        n0, n1, n2, m0, m1, m2 = info[:6]
        if not info[6]:
            raise ValueError(f"level {l} is not on the fused 3-D path")
        Pf = [p >> j for p in P]
        Pf[R] = n0
        K = [p >> (j + 1) for p in P]
        K[R] = m0
        # the plane pass reads the shells of fine planes [2 K_r - 2, 2 K_{r+1}]
        exch.halo_ranges(coeffs, lambda r: [shell_plane_range(p, info) for p in (Pf[r] - 2, Pf[r] - 1)],
                         lambda r: [shell_plane_range(Pf[r + 1], info)])
        G = [torch.empty((m0, m1 * m2), dtype=torch.float64, device=dev) for _ in exch.local]
        for i, r in enumerate(exch.local):
            ws = workspaces[i]
            _check(lib.mgrx_gpu_slab_rec_plane(ws.handle, code, 3, _dims_arr(dims), L, l, K[r], K[r + 1],
                                               _ptr(coeffs[i]), _ptr(G[i])), ws.handle)
            _check(lib.mgrx_gpu_slab_inplane(ws.handle, code, 3, _dims_arr(dims), L, l, K[r], K[r + 1], _ptr(G[i])),
                   ws.handle)
        Cb = column_bounds(m1 * m2, R)
        Gt = exch.transpose(G, K, Cb)
        for i, r in enumerate(exch.local):
            ws = workspaces[i]
            _check(lib.mgrx_gpu_slab_axis0(ws.handle, code, 3, _dims_arr(dims), L, l, Cb[r + 1] - Cb[r], _ptr(Gt[i])),
                   ws.handle)
        z = exch.transpose_back(Gt, K, Cb)
        for i, r in enumerate(exch.local):
            ws = workspaces[i]
            _check(lib.mgrx_gpu_slab_apply(ws.handle, code, _ptr(cur[i], K[r] * m1 * m2), _ptr(z[i]),
                                           (K[r + 1] - K[r]) * m1 * m2, -1.0), ws.handle)
        # the interpolation reads the right neighbour's first corrected plane
        exch.halo(cur, None, K, 0, 1)
        fine = [torch.empty((n0, n1 * n2), dtype=dt, device=dev) for _ in exch.local]
        for i, r in enumerate(exch.local):
            ws = workspaces[i]
            _check(lib.mgrx_gpu_slab_interp(ws.handle, code, 3, _dims_arr(dims), L, l, Pf[r], Pf[r + 1],
                                            _ptr(coeffs[i]), _ptr(cur[i]), _ptr(fine[i])), ws.handle)
        cur = fine
    return [c.reshape(dims) for c in cur]
