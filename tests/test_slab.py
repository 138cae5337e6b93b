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
    import torch

    import paper_2010_05872_b200 as mg
    from synthetic_fields import config2_field
    from paper_2010_05872_b200.slab import _fused_depth, slab_decompose, slab_recompose

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
    fields = []
    for r in range(ranks):
        x = torch.full_like(f, float("nan"))
        hi = P[r + 1] if r + 1 < ranks else shape[0]
        x[P[r]:hi] = f[P[r]:hi]
        fields.append(x)
    ex = LocalExchange(ranks)
    wss = [mg.SolverWorkspace() for _ in range(ranks)]
    outs = slab_decompose(fields, h, ex, wss, S)
    got = outs[0].clone()
    for o in outs[1:]:
        got = torch.where(torch.isnan(got), o, got)
    torch.cuda.synchronize()
    assert not torch.isnan(got).any()
    assert torch.equal(got, want)
    # recompose from each rank's own coefficients (its shells + the coarse
    # levels; the halo planes' shells are exchanged inside)
    backs = slab_recompose(outs, h, ex, wss, S)
    back = torch.empty_like(f)
    for r in range(ranks):
        hi = P[r + 1] if r + 1 < ranks else shape[0]
        back[P[r]:hi] = backs[r][P[r]:hi]
    torch.cuda.synchronize()
    assert torch.equal(back, back_want)


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        m0, ncols = 12, 10
        base = [torch.randn(m0, ncols, generator=g, dtype=torch.float64) for _ in range(world)]
        K = [0, 5, 12]
        Cb = column_bounds(ncols, world)
        loc = LocalExchange(world)
        te = TorchExchange()
        # halo
        L_bufs = [b.clone() for b in base]
        loc.halo(L_bufs, None, K, 2, 1)
        T_buf = [base[rank].clone()]
        te.halo(T_buf, None, K, 2, 1)
        ok = torch.equal(T_buf[0], L_bufs[rank])
        # halo of element ranges
        flat = [b.reshape(-1).clone() for b in base]
        left = lambda r: [(r * 7, r * 7 + 3), (40, 42)]  # noqa: E731
        right = lambda r: [(100 + r, 103 + r)]  # noqa: E731
        L_fl = [f.clone() for f in flat]
        loc.halo_ranges(L_fl, left, right)
        T_fl = [flat[rank].clone()]
        te.halo_ranges(T_fl, left, right)
        ok &= torch.equal(T_fl[0], L_fl[rank])
        # transposes
        Gt_l = loc.transpose(base, K, Cb)
        Gt_t = te.transpose([base[rank]], K, Cb)
        ok &= torch.equal(Gt_t[0], Gt_l[rank])
        z_l = loc.transpose_back(Gt_l, K, Cb)
        z_t = te.transpose_back(Gt_t, K, Cb)
        ok &= torch.equal(z_t[0], z_l[rank])
        ok &= torch.equal(z_l[rank], base[rank][K[rank]:K[rank + 1]])
        # gather
        G_l = [b.clone() for b in base]
        loc.gather(G_l, K)
        G_t = [base[rank].clone()]
        te.gather(G_t, K)
        ok &= torch.equal(G_t[0], G_l[rank])
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
