"""Slab mode: a field split into axis-0 slabs over R ranks.

* GPU: all R ranks emulated in one process (LocalExchange, device copies)
  must reproduce the single-GPU decompose / recompose bit for bit; the
  planes a rank does not own are NaN-poisoned, so a missing halo or
  transpose block shows up.
* CPU (gloo, world size 2): TorchExchange's halo / transpose / gather data
  movement equals LocalExchange's on the same buffers.
"""
import os

import pytest

from paper_2010_05872_b200.slab import LocalExchange, TorchExchange, column_bounds, max_slab_levels, \
    shell_plane_range, slab_bounds


def test_shell_plane_ranges_tile_the_level():
    # level 9 of 513^3: fine 513^3, coarse 257^3, shell offset 257^3
    info = [513, 513, 513, 257, 257, 257, 1, 257 ** 3]
    rngs = sorted(shell_plane_range(p, info) for p in range(513))
    assert rngs[0][0] == 257 ** 3 and rngs[-1][1] == 513 ** 3
    assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))


def test_bounds():
    assert slab_bounds(1025, 8, 7) == [0, 128, 256, 384, 512, 640, 768, 896, 1024]
    assert slab_bounds(513, 3, 2) == [0, 168, 340, 512]
    assert all(b % 4 == 0 for b in slab_bounds(513, 3, 2))
    assert column_bounds(10, 3) == [0, 3, 6, 10]
    with pytest.raises(ValueError):
        slab_bounds(100, 2, 3)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,dtype,ranks", [((129, 129, 129), "f64", 2), ((257, 129, 65), "f32", 3),
                                               ((513, 513, 513), "f32", 4)])
def test_slab_emulated_matches_single_gpu(shape, dtype, ranks):
    _slab_case(shape, dtype, ranks)


@pytest.mark.gpu
@pytest.mark.slow
def test_slab_1025_eight_ranks_slab_sized_buffers():
    """Config 5b's field over 8 emulated ranks: bit-identical to one GPU,
    every rank holding about 1/8 of the field plus halos."""
    _slab_case((1025, 1025, 1025), "f32", 8, check_memory=True)


@pytest.mark.gpu
def test_kpack_kernel_matches_torch():
    """mgrx_gpu_slab_pack / _unpack (the all-to-all K-pack) against the torch
    reference packing, on uneven column blocks."""
    import torch

    import paper_2010_05872_b200 as mg
    from paper_2010_05872_b200.slab import KPack, _torch_pack, _torch_unpack

    g = torch.Generator(device="cuda").manual_seed(5)
    src = torch.randn(37, 1001, generator=g, dtype=torch.float64, device="cuda")
    kp = KPack(mg.SolverWorkspace())
    for cb in ([0, 1001], [0, 300, 301, 700, 1001], column_bounds(1001, 8)):
        packed = kp.pack(src, cb)
        torch.cuda.synchronize()
        assert torch.equal(packed, _torch_pack(src, cb))
        back = kp.unpack(packed, 37, cb)
        assert torch.equal(back, _torch_unpack(packed, 37, cb)) and torch.equal(back, src)


def _slab_case(shape, dtype, ranks, check_memory=False):
    import torch

    import paper_2010_05872_b200 as mg
    from synthetic_fields import config2_field
    from paper_2010_05872_b200.slab import PlaneSlab, _fused_depth, assemble_coefficients, owned_planes, \
        slab_decompose, slab_recompose

    dt = torch.float64 if dtype == "f64" else torch.float32
    f = config2_field(shape, seed=3, device="cuda").to(dt)
    h = mg.GridHierarchy.create(shape)
    ws1 = mg.SolverWorkspace()
    want = mg.decompose(f, h, 0, ws1).buffer
    back_want = mg.recompose(mg.MultilevelCoefficients(want, h, 0), ws1)
    S = max_slab_levels(h, ranks)
    assert S >= 1
    S = _fused_depth(ws1, 1 if dtype == "f64" else 0, shape, h.num_levels(), S)
    assert S >= 1
    P = slab_bounds(shape[0], ranks, S)
    plane = shape[1] * shape[2]
    fields = []
    for r in range(ranks):  # each rank holds only its own planes (slab-sized)
        lo, hi = owned_planes(P, r, shape[0])
        s = PlaneSlab(lo, hi, plane, dt, f.device)
        s.t.copy_(f.reshape(shape[0], -1)[lo:hi])
        fields.append(s)
    ex = LocalExchange(ranks)
    wss = [mg.SolverWorkspace() for _ in range(ranks)]
    outs = slab_decompose(fields, h, ex, wss, S)
    got = assemble_coefficients(outs, h)
    torch.cuda.synchronize()
    assert not torch.isnan(got).any()
    assert torch.equal(got, want)
    if check_memory:  # per-rank coefficient storage ~ 1/R of the buffer
        for o in outs:
            assert o.nbytes() < 1.5 * want.numel() * want.element_size() / ranks, o.nbytes()
    del want
    # recompose from each rank's own coefficients (its shells + the coarse
    # levels; the halo planes' shells are exchanged inside)
    backs = slab_recompose(outs, h, ex, wss)
    bw = back_want.reshape(shape[0], -1)
    for r in range(ranks):
        lo, hi = owned_planes(P, r, shape[0])
        assert torch.equal(backs[r].planes(lo, hi), bw[lo:hi]), r
    torch.cuda.synchronize()


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2010_05872_b200.slab import PlaneSlab, ShellSlab

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        m0, ncols = 12, 10
        base = torch.randn(m0, ncols, generator=g, dtype=torch.float64)
        K = [0, 5, 12]
        Cb = column_bounds(ncols, world)
        loc = LocalExchange(world)
        te = TorchExchange()

        def slab(r, fill_own=True):  # rank r's planes with a 2-left / 1-right halo, halo NaN
            lo, hi = K[r], K[r + 1]
            s = PlaneSlab(max(0, lo - 2), min(m0, hi + 1), ncols, torch.float64, "cpu", fill=float("nan"))
            s.planes(lo, hi).copy_(base[lo:hi])
            return s

        # plane halo
        L_s = [slab(r) for r in range(world)]
        loc.halo(L_s, K, 2, 1)
        T_s = [slab(rank)]
        te.halo(T_s, K, 2, 1)
        ok = torch.equal(T_s[0].t.nan_to_num(-1), L_s[rank].t.nan_to_num(-1))
        ok &= not bool(torch.isnan(L_s[rank].t).any())
        # shell halo (level 12 x 10 x 10 -> shells of planes around the slab)
        info = [12, 10, 10, 6, 5, 5, 1, 0, 1200]
        Pf = [0, 6, 12]

        def shells(r):
            s = ShellSlab(info, Pf[r] - 2, Pf[r + 1], torch.float64, "cpu")
            for p in range(Pf[r], min(Pf[r + 1], 12)):
                x = s.run(p)
                x.copy_(torch.arange(x.numel(), dtype=torch.float64) + 1000 * p)
            return s

        left = lambda r: [p for p in (Pf[r] - 2, Pf[r] - 1) if p >= 0]  # noqa: E731
        right = lambda r: [Pf[r + 1]]  # noqa: E731
        L_sh = [shells(r) for r in range(world)]
        loc.halo_shells(L_sh, left, right)
        T_sh = [shells(rank)]
        te.halo_shells(T_sh, left, right)
        ok &= torch.equal(T_sh[0].t.nan_to_num(-1), L_sh[rank].t.nan_to_num(-1))
        # transposes (the torch K-pack on CPU tensors)
        G = [base[K[r]:K[r + 1]].contiguous() for r in range(world)]
        Gt_l = loc.transpose(G, K, Cb)
        Gt_t = te.transpose([G[rank]], K, Cb)
        ok &= torch.equal(Gt_t[0], Gt_l[rank])
        ok &= torch.equal(Gt_l[rank], base[:, Cb[rank]:Cb[rank + 1]])
        z_l = loc.transpose_back(Gt_l, K, Cb)
        z_t = te.transpose_back(Gt_t, K, Cb)
        ok &= torch.equal(z_t[0], z_l[rank])
        ok &= torch.equal(z_l[rank], base[K[rank]:K[rank + 1]])
        # gather
        G_l = loc.gather([slab(r) for r in range(world)], K, m0)
        G_t = te.gather([slab(rank)], K, m0)
        ok &= torch.equal(G_t[0], G_l[rank]) and torch.equal(G_l[rank], base)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_torch_exchange_matches_local_gloo():
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
