"""Slab mode: one 3-D field sharded along axis 0 over R ranks.

The reference has no distributed path: this runs its decompose / recompose
(transform.hpp:485-530) for a field whose axis-0 planes are split into R
slabs, one per GPU, with the exchange steps the level passes need:

* the plane passes read a halo of fine planes (two on the left, one on the
  right) around a rank's slab (`Exchange.halo`);
* the axis-0 Thomas solve (batched_solve, transform.hpp:116-130) needs whole
  axis-0 columns, so the fp64 load-vector volume G of the level is
  transposed (all-to-all: each rank gets every plane of 1/R of the columns),
  solved, and transposed back (`Exchange.transpose`, `.transpose_back`; the
  send / receive blocks are packed by the K-pack kernel
  mgrx_gpu_slab_pack / _unpack); the correction is then applied to the
  rank's coarse planes;
* recompose's plane pass reads the shells of the halo planes, and its
  interpolation the right neighbour's first corrected coarse plane;
* below the slab levels the coarse block is gathered (`Exchange.gather`) and
  the remaining levels run on every rank (they are small).

Every per-rank buffer is sized to the rank's slab plus its halo:
`PlaneSlab` holds planes [lo, hi) of a level volume, `ShellSlab` the shell
entries (level-centric layout, pack_level_centric reorder.hpp:162-217) of
fine planes [plo, phi] as two runs, the even planes' and the odd planes'.
The C-ABI's mgrx_gpu_slab_* passes index globally: they get base pointers
shifted back by the global offset of the slab's first element (only the
slab's planes are touched) and, for the shells, the distance between the
two runs (odd_shift).  Slab boundaries sit at multiples of 2^S fine planes
(S slab levels), so they stay on nodal planes of every slab level.  The
results are bit-identical to the single-GPU decompose / recompose (the same
per-element arithmetic; tests/test_slab.py).

Two exchanges: `TorchExchange` (torch.distributed: NCCL between GPUs, or
gloo for the CPU tests of the data movement) with one local rank per
process, and `LocalExchange`, which runs all R ranks in one process (on one
GPU) with device copies — the emulation the single-GPU tests use.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence

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


def owned_planes(P: Sequence[int], r: int, n: int) -> tuple:
    """[lo, hi) of the planes rank r owns out of n (the last rank also n - 1)."""
    return P[r], (P[r + 1] if r + 1 < len(P) - 1 else n)


# ------------------------------------------------------------ local buffers

class PlaneSlab:
    """Planes [lo, hi) of a level volume (`elems` values per plane), held
    locally and addressed by global plane index."""

    def __init__(self, lo: int, hi: int, elems: int, dtype, device, fill=None):
        import torch

        self.lo, self.hi, self.elems = lo, hi, elems
        shape = (max(hi - lo, 0), elems)
        self.t = torch.full(shape, fill, dtype=dtype, device=device) if fill is not None else \
            torch.empty(shape, dtype=dtype, device=device)

    def planes(self, a: int, b: int):
        a, b = max(a, self.lo), min(b, self.hi)
        return self.t[a - self.lo:max(b, a) - self.lo]

    def vptr(self):
        """Base pointer of the global indexing (plane p at p * elems)."""
        return C.c_void_p(self.t.data_ptr() - self.lo * self.elems * self.t.element_size())

    def nbytes(self) -> int:
        return self.t.numel() * self.t.element_size()


class ShellSlab:
    """Shell entries of fine planes [plo, phi] of one level: the even planes'
    run [E0, E1) and the odd planes' run [O0, O1) of the level's shell
    (positions relative to the shell start node_count(l - 1)), stored back to
    back."""

    def __init__(self, info, plo: int, phi: int, dtype, device, fill=float("nan")):
        import torch

        self.info = info
        self.off = info[7]
        plo, phi = max(plo, 0), min(phi, info[0] - 1)
        ev = [p for p in range(plo, phi + 1) if p % 2 == 0]
        od = [p for p in range(plo, phi + 1) if p % 2 == 1]
        rel = lambda p: [x - self.off for x in shell_plane_range(p, info)]  # noqa: E731
        self.E0, self.E1 = (rel(ev[0])[0], rel(ev[-1])[1]) if ev else (0, 0)
        self.O0, self.O1 = (rel(od[0])[0], rel(od[-1])[1]) if od else (0, 0)
        self.plo, self.phi = plo, phi
        self.t = torch.full((self.E1 - self.E0 + self.O1 - self.O0,), fill, dtype=dtype, device=device)

    def run(self, p: int):
        """This slab's storage of fine plane p's shell run."""
        a, b = [x - self.off for x in shell_plane_range(p, self.info)]
        if p % 2 == 0:
            return self.t[a - self.E0:b - self.E0]
        base = self.E1 - self.E0
        return self.t[base + a - self.O0:base + b - self.O0]

    def vptr(self):
        """d_out / d_coeffs of the C-ABI (level-centric base; the entry point
        adds node_count(l - 1))."""
        return C.c_void_p(self.t.data_ptr() - (self.off + self.E0) * self.t.element_size())

    def odd_shift(self) -> int:
        return self.E1 - self.O0

    def nbytes(self) -> int:
        return self.t.numel() * self.t.element_size()


class SlabCoefficients:
    """One rank's share of a slab-sharded decomposition: the coarse levels
    below the slab levels (replicated, level-centric, `coarse`) and per slab
    level l the shells of its fine planes plus their halo (`shells[l]`)."""

    def __init__(self, coarse, shells: Dict[int, ShellSlab], bounds: List[int], slab_levels: int):
        self.coarse = coarse
        self.shells = shells
        self.bounds = bounds
        self.slab_levels = slab_levels

    def nbytes(self) -> int:
        return self.coarse.numel() * self.coarse.element_size() + sum(s.nbytes() for s in self.shells.values())


# ------------------------------------------------------------------ K-pack

def _torch_pack(src, cb):
    import torch

    return torch.cat([src[:, cb[q]:cb[q + 1]].reshape(-1) for q in range(len(cb) - 1)])


def _torch_unpack(src, rows, cb):
    import torch

    parts, o = [], 0
    for q in range(len(cb) - 1):
        w = cb[q + 1] - cb[q]
        parts.append(src[o:o + rows * w].view(rows, w))
        o += rows * w
    return torch.cat(parts, dim=1).contiguous()


class KPack:
    """Packs the column blocks of a rows x ncols fp64 array back to back
    (the all-to-all send buffer) and unpacks the inverse, with the library's
    K-pack kernel on CUDA tensors (torch ops on CPU tensors, for the gloo
    tests)."""

    def __init__(self, ws: Optional[SolverWorkspace] = None):
        self.ws = ws

    def pack(self, src, cb):
        if not src.is_cuda or self.ws is None:
            return _torch_pack(src, cb)
        import torch

        rows, pitch = src.shape
        out = torch.empty(rows * (cb[-1] - cb[0]), dtype=src.dtype, device=src.device)
        arr = (C.c_uint64 * len(cb))(*cb)
        self.ws._bind_stream()
        _check(lib.mgrx_gpu_slab_pack(self.ws.handle, C.c_void_p(src.data_ptr()), rows, pitch, arr, len(cb) - 1,
                                      C.c_void_p(out.data_ptr())), self.ws.handle)
        return out

    def unpack(self, src, rows, cb):
        if not src.is_cuda or self.ws is None:
            return _torch_unpack(src, rows, cb)
        import torch

        out = torch.empty((rows, cb[-1] - cb[0]), dtype=src.dtype, device=src.device)
        arr = (C.c_uint64 * len(cb))(*cb)
        self.ws._bind_stream()
        _check(lib.mgrx_gpu_slab_unpack(self.ws.handle, C.c_void_p(src.data_ptr()), rows, cb[-1] - cb[0], arr,
                                        len(cb) - 1, C.c_void_p(out.data_ptr())), self.ws.handle)
        return out


# ---------------------------------------------------------------- exchanges

class LocalExchange:
    """All R ranks in this process (one GPU): exchanges are device copies."""

    def __init__(self, ranks: int, kpack: Optional[KPack] = None):
        self.world = ranks
        self.local = list(range(ranks))
        self.kp = kpack or KPack()

    def halo(self, slabs: Sequence[PlaneSlab], bounds, left: int, right: int):
        """slabs[r] receives planes [bounds[r] - left, bounds[r]) from rank
        r - 1 and [bounds[r+1], bounds[r+1] + right) from rank r + 1 (as far
        as both slabs hold them)."""
        R = self.world
        for r in range(R):
            if r > 0 and left:
                a, b = bounds[r] - left, bounds[r]
                dst, src = slabs[r].planes(a, b), slabs[r - 1].planes(a, b)
                if dst.shape[0]:
                    dst.copy_(src)
            if r + 1 < R and right:
                a, b = bounds[r + 1], bounds[r + 1] + right
                dst, src = slabs[r].planes(a, b), slabs[r + 1].planes(a, b)
                if dst.shape[0]:
                    dst.copy_(src)

    def halo_shells(self, shells: Sequence[ShellSlab], left, right):
        """shells[r] receives the shell runs of planes left(r) from rank r - 1
        and right(r) from rank r + 1."""
        R = self.world
        for r in range(R):
            if r > 0:
                for p in left(r):
                    shells[r].run(p).copy_(shells[r - 1].run(p))
            if r + 1 < R:
                for p in right(r):
                    shells[r].run(p).copy_(shells[r + 1].run(p))

    def transpose(self, G, K, Cb):
        """G[r]: (K[r+1] - K[r], ncols), rank r's planes -> Gt[r]: (m0,
        Cb[r+1] - Cb[r]), full axis-0 columns of rank r."""
        import torch

        R = self.world
        sends = [self.kp.pack(G[q], Cb) for q in range(R)]
        out = []
        for r in range(R):
            parts = []
            for q in range(R):
                rows = K[q + 1] - K[q]
                parts.append(sends[q][rows * Cb[r]:rows * Cb[r + 1]].view(rows, Cb[r + 1] - Cb[r]))
            out.append(torch.cat(parts).contiguous())
        return out

    def transpose_back(self, Gt, K, Cb):
        """Gt[r] (m0, W_r) -> z[r]: (K[r+1] - K[r], ncols), rank r's planes."""
        import torch

        R = self.world
        out = []
        for r in range(R):
            rows = K[r + 1] - K[r]
            recv = torch.cat([Gt[q][K[r]:K[r + 1]].reshape(-1) for q in range(R)])
            out.append(self.kp.unpack(recv, rows, Cb))
        return out

    def gather(self, slabs: Sequence[PlaneSlab], bounds, n: int):
        """Every rank gets the full volume (n planes) from the ranks' own
        planes [bounds[q], bounds[q+1]) (the last rank's up to n)."""
        import torch

        R = self.world
        full = torch.cat([slabs[q].planes(*owned_planes(bounds, q, n)) for q in range(R)])
        return [full.clone() for _ in range(R)]


class TorchExchange:
    """One rank per process over torch.distributed (NCCL between GPUs; gloo
    for CPU tensors in the tests).  Same semantics as LocalExchange with the
    lists holding this rank's buffer only."""

    def __init__(self, group=None, kpack: Optional[KPack] = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.local = [self.rank]
        self.kp = kpack or KPack()

    def _p2p(self, sends, recvs):
        dist = self.dist
        ops = [dist.P2POp(dist.isend, t, peer, self.group) for peer, t in sends] + \
              [dist.P2POp(dist.irecv, t, peer, self.group) for peer, t in recvs]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def halo(self, slabs, bounds, left: int, right: int):
        r, R = self.rank, self.world
        s = slabs[0]
        sends, recvs, back = [], [], []
        # what rank r + 1 wants (its left halo) / rank r - 1 wants (its right halo)
        if r + 1 < R and left:
            sends.append((r + 1, s.planes(bounds[r + 1] - left, bounds[r + 1]).contiguous()))
        if r > 0 and right:
            sends.append((r - 1, s.planes(bounds[r], bounds[r] + right).contiguous()))
        if r > 0 and left:
            dst = s.planes(bounds[r] - left, bounds[r])
            t = dst.new_empty(dst.shape)
            recvs.append((r - 1, t))
            back.append((dst, t))
        if r + 1 < R and right:
            dst = s.planes(bounds[r + 1], bounds[r + 1] + right)
            t = dst.new_empty(dst.shape)
            recvs.append((r + 1, t))
            back.append((dst, t))
        self._p2p(sends, recvs)
        for dst, t in back:
            dst.copy_(t)

    def halo_shells(self, shells, left, right):
        import torch

        r, R = self.rank, self.world
        s = shells[0]
        sends, recvs, back = [], [], []
        if r + 1 < R:
            sends.append((r + 1, torch.cat([s.run(p) for p in left(r + 1)])))
        if r > 0:
            sends.append((r - 1, torch.cat([s.run(p) for p in right(r - 1)])))
        if r > 0:
            runs = [s.run(p) for p in left(r)]
            t = s.t.new_empty(sum(x.numel() for x in runs))
            recvs.append((r - 1, t))
            back.append((runs, t))
        if r + 1 < R:
            runs = [s.run(p) for p in right(r)]
            t = s.t.new_empty(sum(x.numel() for x in runs))
            recvs.append((r + 1, t))
            back.append((runs, t))
        self._p2p(sends, recvs)
        for runs, t in back:
            o = 0
            for x in runs:
                x.copy_(t[o:o + x.numel()])
                o += x.numel()

    def transpose(self, G, K, Cb):
        dist, r, R = self.dist, self.rank, self.world
        send = self.kp.pack(G[0], Cb)
        W = Cb[r + 1] - Cb[r]
        out = send.new_empty((K[R] - K[0]) * W)
        # output splits: K_q rows x my width from each q; input: my rows x W_q to each q
        dist.all_to_all_single(out, send, [(K[q + 1] - K[q]) * W for q in range(R)],
                               [(K[r + 1] - K[r]) * (Cb[q + 1] - Cb[q]) for q in range(R)], group=self.group)
        return [out.view(K[R] - K[0], W)]

    def transpose_back(self, Gt, K, Cb):
        dist, r, R = self.dist, self.rank, self.world
        gt = Gt[0]
        send = gt.reshape(-1)  # rows [K_q, K_{q+1}) for q in order are contiguous
        rows = K[r + 1] - K[r]
        out = gt.new_empty(rows * Cb[R])
        dist.all_to_all_single(out, send, [rows * (Cb[q + 1] - Cb[q]) for q in range(R)],
                               [(K[q + 1] - K[q]) * (Cb[r + 1] - Cb[r]) for q in range(R)], group=self.group)
        return [self.kp.unpack(out, rows, Cb)]

    def gather(self, slabs, bounds, n: int):
        dist, R = self.dist, self.world
        s = slabs[0]
        sizes = [owned_planes(bounds, q, n)[1] - owned_planes(bounds, q, n)[0] for q in range(R)]
        mx = max(sizes)
        mine = s.planes(*owned_planes(bounds, self.rank, n))
        pad = s.t.new_zeros((mx, s.elems))
        pad[:mine.shape[0]] = mine
        got = [s.t.new_empty(pad.shape) for _ in range(R)]
        dist.all_gather(got, pad, group=self.group)
        import torch

        return [torch.cat([got[q][:sizes[q]] for q in range(R)])]


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


def _vp(t, offset_elems: int = 0):
    return C.c_void_p(t.data_ptr() + offset_elems * t.element_size())


def _levels(h, R, ws, code, slab_levels):
    L = h.num_levels()
    dims = h.level_dims(L)
    S = max_slab_levels(h, R) if slab_levels is None else slab_levels
    S = _fused_depth(ws, code, dims, L, S)
    return L, dims, S, slab_bounds(dims[0], R, S)


def _bounds(P, j, n0, m0):
    """Fine (Pf) and coarse (K) plane bounds of slab level j."""
    R = len(P) - 1
    Pf = [p >> j for p in P]
    Pf[R] = n0
    K = [p >> (j + 1) for p in P]
    K[R] = m0
    return Pf, K


def _axis0(exch, workspaces, G, K, Cb, code, dims, L, l):
    """Transpose G, axis-0 solve of every rank's column block, transpose back."""
    Gt = exch.transpose(G, K, Cb)
    for i, r in enumerate(exch.local):
        ws = workspaces[i]
        _check(lib.mgrx_gpu_slab_axis0(ws.handle, code, 3, _dims_arr(dims), L, l, Cb[r + 1] - Cb[r], _vp(Gt[i])),
               ws.handle)
    return exch.transpose_back(Gt, K, Cb)


def slab_decompose(fields: Sequence, hierarchy: GridHierarchy, exch, workspaces: Sequence[SolverWorkspace],
                   slab_levels: Optional[int] = None) -> List[SlabCoefficients]:
    """decompose of a slab-sharded field.  fields[i]: the slab of local rank
    exch.local[i] — a PlaneSlab of the finest level (or a full-size tensor,
    of which only the rank's planes are read).  Returns one
    SlabCoefficients per local rank: its planes' shells and the replicated
    coarse levels."""
    import torch

    R = exch.world
    h = hierarchy
    code = _dtype_code(fields[0].t if isinstance(fields[0], PlaneSlab) else fields[0])
    L, dims, S, P = _levels(h, R, workspaces[0], code, slab_levels)
    n0f = dims[0]
    plane_f = dims[1] * dims[2]
    for ws in workspaces:
        ws._bind_stream()
    if exch.kp.ws is None:  # the K-pack kernel on this rank's context
        exch.kp.ws = workspaces[0]
    # the finest level's input slabs with their halo (two planes left, one right)
    blk = []
    for i, r in enumerate(exch.local):
        f = fields[i]
        lo, hi = owned_planes(P, r, n0f)
        s = PlaneSlab(max(0, lo - 2), min(n0f, hi + 1), plane_f, f.t.dtype if isinstance(f, PlaneSlab) else f.dtype,
                      f.t.device if isinstance(f, PlaneSlab) else f.device)
        src = f.planes(lo, hi) if isinstance(f, PlaneSlab) else f.reshape(n0f, -1)[lo:hi]
        s.planes(lo, hi).copy_(src)
        blk.append(s)
    shells: List[Dict[int, ShellSlab]] = [dict() for _ in exch.local]
    dt, dev = blk[0].t.dtype, blk[0].t.device
    for j in range(S):
        l = L - j
        info = _level_info(workspaces[0], code, dims, L, l)
        n0, m0, m1, m2 = info[0], info[3], info[4], info[5]
        if not info[6]:
            raise ValueError(f"level {l} is not on the fused 3-D path")
        Pf, K = _bounds(P, j, n0, m0)
        exch.halo(blk, Pf, 2, 1)
        G, coarse = [], []
        for i, r in enumerate(exch.local):
            ws = workspaces[i]
            plo, phi = owned_planes(Pf, r, n0)
            sh = ShellSlab(info, plo - 2, phi, dt, dev)  # own planes + the recompose halo
            shells[i][l] = sh
            g = PlaneSlab(K[r], K[r + 1], m1 * m2, torch.float64, dev)
            cs = PlaneSlab(max(0, K[r] - 2), min(m0, K[r + 1] + 1), m1 * m2, dt, dev)
            _check(lib.mgrx_gpu_slab_dec_plane(ws.handle, code, 3, _dims_arr(dims), L, l, K[r], K[r + 1],
                                               blk[i].vptr(), sh.vptr(), cs.vptr(), g.vptr(), sh.odd_shift()),
                   ws.handle)
            _check(lib.mgrx_gpu_slab_inplane(ws.handle, code, 3, _dims_arr(dims), L, l, K[r], K[r + 1], g.vptr()),
                   ws.handle)
            G.append(g.t)
            coarse.append(cs)
        Cb = column_bounds(m1 * m2, R)
        z = _axis0(exch, workspaces, G, K, Cb, code, dims, L, l)
        for i, r in enumerate(exch.local):
            ws = workspaces[i]
            cp = coarse[i].planes(K[r], K[r + 1])
            _check(lib.mgrx_gpu_slab_apply(ws.handle, code, _vp(cp), _vp(z[i]), cp.numel(), 1.0), ws.handle)
        blk = coarse
    # the remaining levels: gather the coarse block, decompose it on every rank
    Lc = L - S
    dims_c = h.level_dims(Lc)
    Kc = [p >> S for p in P]
    Kc[R] = dims_c[0]
    full = exch.gather(blk, Kc, dims_c[0])
    hc = GridHierarchy.create(dims_c, Lc)
    out = []
    for i in range(len(exch.local)):
        mc = decompose(full[i].reshape(dims_c), hc, 0, workspaces[i])
        out.append(SlabCoefficients(mc.buffer, shells[i], P, S))
    return out


def slab_recompose(coeffs: Sequence[SlabCoefficients], hierarchy: GridHierarchy, exch,
                   workspaces: Sequence[SolverWorkspace]) -> List[PlaneSlab]:
    """recompose into a slab-sharded field.  coeffs[i]: what slab_decompose
    returned on local rank exch.local[i] (the halo planes' shells are
    exchanged here, in place).  Returns per local rank a PlaneSlab of the
    finest level holding (at least) its planes [P_r, P_{r+1}) (the last rank
    also n0 - 1)."""
    R = exch.world
    h = hierarchy
    code = _dtype_code(coeffs[0].coarse)
    L = h.num_levels()
    dims = h.level_dims(L)
    S, P = coeffs[0].slab_levels, coeffs[0].bounds
    dt, dev = coeffs[0].coarse.dtype, coeffs[0].coarse.device
    for ws in workspaces:
        ws._bind_stream()
    if exch.kp.ws is None:
        exch.kp.ws = workspaces[0]
    Lc = L - S
    dims_c = h.level_dims(Lc)
    hc = GridHierarchy.create(dims_c, Lc)
    Kc = [p >> S for p in P]
    Kc[R] = dims_c[0]
    cur = []  # corrected coarse planes of the next level: [K_r, K_{r+1} + 1)
    for i, r in enumerate(exch.local):
        f = recompose(MultilevelCoefficients(coeffs[i].coarse, hc, 0), workspaces[i]).reshape(dims_c[0], -1)
        lo, hi = owned_planes(Kc, r, dims_c[0])
        s = PlaneSlab(lo, min(dims_c[0], hi + 1), f.shape[1], dt, dev)
        s.t.copy_(f[s.lo:s.hi])
        cur.append(s)
    for j in reversed(range(S)):
        l = L - j
        info = _level_info(workspaces[0], code, dims, L, l)
        n0, n1, n2, m0, m1, m2 = info[:6]
        Pf, K = _bounds(P, j, n0, m0)
        sh = [coeffs[i].shells[l] for i in range(len(exch.local))]
        # the plane pass reads the shells of fine planes [2 K_r - 2, 2 K_{r+1}]
        exch.halo_shells(sh, lambda r: [p for p in (Pf[r] - 2, Pf[r] - 1) if p >= 0],
                         lambda r: [Pf[r + 1]])
        G = []
        for i, r in enumerate(exch.local):
            ws = workspaces[i]
            g = PlaneSlab(K[r], K[r + 1], m1 * m2, __import__("torch").float64, dev)
            _check(lib.mgrx_gpu_slab_rec_plane(ws.handle, code, 3, _dims_arr(dims), L, l, K[r], K[r + 1],
                                               sh[i].vptr(), g.vptr(), sh[i].odd_shift()), ws.handle)
            _check(lib.mgrx_gpu_slab_inplane(ws.handle, code, 3, _dims_arr(dims), L, l, K[r], K[r + 1], g.vptr()),
                   ws.handle)
            G.append(g.t)
        Cb = column_bounds(m1 * m2, R)
        z = _axis0(exch, workspaces, G, K, Cb, code, dims, L, l)
        for i, r in enumerate(exch.local):
            ws = workspaces[i]
            cp = cur[i].planes(K[r], K[r + 1])
            _check(lib.mgrx_gpu_slab_apply(ws.handle, code, _vp(cp), _vp(z[i]), cp.numel(), -1.0), ws.handle)
        # the interpolation reads the right neighbour's first corrected plane
        exch.halo(cur, K, 0, 1)
        fine = []
        for i, r in enumerate(exch.local):
            ws = workspaces[i]
            lo, hi = owned_planes(Pf, r, n0)
            fs = PlaneSlab(lo, min(n0, hi + 1), n1 * n2, dt, dev)
            _check(lib.mgrx_gpu_slab_interp(ws.handle, code, 3, _dims_arr(dims), L, l, lo, hi, sh[i].vptr(),
                                            cur[i].vptr(), fs.vptr(), sh[i].odd_shift()), ws.handle)
            fine.append(fs)
        cur = fine
    return cur


def assemble_coefficients(parts: Sequence[SlabCoefficients], hierarchy: GridHierarchy):
    """The global level-centric buffer from every rank's SlabCoefficients
    (tests): the replicated coarse levels, then each rank's own planes'
    shells."""
    import torch

    h = hierarchy
    L = h.num_levels()
    dims = h.level_dims(L)
    p0 = parts[0]
    R = len(parts)
    out = torch.full((h.total_count(),), float("nan"), dtype=p0.coarse.dtype, device=p0.coarse.device)
    out[:p0.coarse.numel()] = p0.coarse
    for j in range(p0.slab_levels):
        l = L - j
        for r, part in enumerate(parts):
            sh = part.shells[l]
            n0 = sh.info[0]
            Pf = [p >> j for p in part.bounds]
            Pf[R] = n0
            lo, hi = owned_planes(Pf, r, n0)
            for p in range(lo, hi):
                a, b = shell_plane_range(p, sh.info)
                out[a:b] = sh.run(p)
    return out
