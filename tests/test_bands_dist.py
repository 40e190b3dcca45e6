"""Row-band decomposition host logic on CPU: the band plan, and the one-round
halo exchange between ranks over torch.distributed (gloo, world_size 2 and 3)
reproducing exactly the extended crops sliced from the full frame."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_08642_b200 import bands


def test_plan_properties():
    for H, L, k, G in [(4320, 4, 7, 8), (1080, 3, 5, 4), (2160, 4, 7, 2), (777, 3, 5, 3)]:
        pl = bands.plan(H, L, k, G)
        align = 1 << (L - 1)
        assert pl[0].own[0] == 0 and pl[-1].own[1] == H
        for a, b in zip(pl, pl[1:]):
            assert a.own[1] == b.own[0] and a.own[1] % align == 0
        halo = bands.halo_rows(L, k)
        assert halo % align == 0 and halo >= sum((k // 2 + 1) << l for l in range(L))
        for b in pl:
            assert b.ext[0] == max(0, b.own[0] - halo) and b.ext[1] == min(H, b.own[1] + halo)
            assert b.ext[0] % align == 0
    with pytest.raises(ValueError):
        bands.plan(100, 4, 7, 8)


def _frame(H, W, L, k, seed=0):
    g = torch.Generator().manual_seed(seed)
    noisy = torch.rand(1, 3, H, W, generator=g)
    demod = torch.rand(1, 3, H, W, generator=g)
    shapes = [(H, W)]
    while len(shapes) < L:
        shapes.append(((shapes[-1][0] + 1) // 2, (shapes[-1][1] + 1) // 2))
    logits = [torch.randn(1, k * k + (4 if l < L - 1 else 0), h, w, generator=g)
              for l, (h, w) in enumerate(shapes)]
    return noisy, demod, logits


def _worker(rank, world, port, H, W, L, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        noisy, demod, logits = _frame(H, W, L, k)
        pl = bands.plan(H, L, k, world)
        b = pl[rank]
        own = lambda t, l: t[:, :, slice(*bands.level_rows(b.own, l, H))].contiguous()  # noqa: E731
        n, d, lg = bands.exchange_band_inputs(dist, rank, world, pl, H, own(noisy, 0), own(demod, 0),
                                              [own(z, l) for l, z in enumerate(logits)])
        rn, rd, rl = bands.crop_inputs(noisy, demod, logits, b, H)
        ok = torch.equal(n, rn) and torch.equal(d, rd) and all(torch.equal(a, c) for a, c in zip(lg, rl))
        q.put((rank, ok, tuple(n.shape)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,H,W,L,k", [(2, 200, 24, 3, 5), (3, 300, 20, 4, 7)])
def test_halo_exchange_gloo(world, H, W, L, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, L, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
