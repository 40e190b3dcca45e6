"""Row-band protocol on CPU: the band plan, and
the exchange protocol of paper_2602_08642_b200/bands.py -- round A (Rh rows of
each pooled level, level 0 noisy + demod; no logits), rounds B_l (one Lhat row
per level) -- between one process per band over torch.distributed (gloo,
world 2 and 3), with the oracle's level arithmetic: the stitched output equals
the same arithmetic run on the unsplit frame bit for bit (and oracle.forward
to 1e-13).  The same protocol runs on the
GPU with the library's level kernels (tests/test_gpu_bands.py)."""
import os
import socket

import numpy as np
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
        rh = bands.halo(k)
        assert rh % 2 == 0 and rh >= k // 2
        for b in pl:
            for l in range(L):
                a, e = bands.level_rows(b.own, l, H)
                assert e - a >= rh
    with pytest.raises(ValueError):
        bands.plan(100, 4, 7, 8)
    # ~1.1 MB per boundary and direction at 8K k7 fp32 (SURVEY.md 8(e) variant 1)
    assert 1.0e6 < bands.halo_bytes(7680, 4, 7) < 1.3e6


def _frame(H, W, L, k, seed=0):
    rng = np.random.default_rng(seed)
    noisy = rng.lognormal(-1.0, 1.5, (H, W, 3))
    demod = rng.uniform(0.0005, 1.0, (H, W, 3))
    from oracle import pyramid as op
    logits = op.random_logits(H, W, L, k, rng, temporal=False)
    return noisy, demod, logits


def _t(a):  # HWC numpy -> (1, C, H, W) torch float64
    return torch.from_numpy(np.ascontiguousarray(a.transpose(2, 0, 1)))[None]


def _worker(rank, world, port, H, W, L, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests._band_cpu import OracleCompute
        noisy, demod, logits = _frame(H, W, L, k)
        pl = bands.plan(H, L, k, world)
        e = bands.BandForward(pl, rank, H, W, L, k, OracleCompute(k), dtype=torch.float64, device="cpu")
        a, b = pl[rank].own
        e.noisy_own.copy_(_t(noisy)[:, :, a:b])
        e.demod_own.copy_(_t(demod)[:, :, a:b])
        for l, z in enumerate(logits):
            la, lb = bands.level_rows(pl[rank].own, l, H)
            e.logits_own[l].copy_(_t(z)[:, :, la:lb])
        out = e.run(bands.GlooTransport(dist))
        q.put((rank, a, b, out[0].permute(1, 2, 0).numpy().copy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,H,W,L,k", [(2, 72, 24, 3, 5), (3, 120, 20, 4, 7), (2, 45, 18, 3, 3)])
def test_band_protocol_gloo_bitwise(world, H, W, L, k):
    from oracle import pyramid as op
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, L, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    noisy, demod, logits = _frame(H, W, L, k)
    ref = _single_band(noisy, demod, logits, k)
    got = np.zeros_like(ref)
    for _, a, b, o in res:
        got[a:b] = o
    np.testing.assert_array_equal(got, ref)
    # and the one-band pipeline is the oracle's forward (to rounding)
    full, _ = op.forward(noisy, logits, None, demod, k=k)
    np.testing.assert_allclose(ref, full, rtol=1e-13, atol=1e-13 * np.abs(full).max())


def _single_band(noisy, demod, logits, k):
    """The same compute without any band split (the full-frame reference
    whose per-pixel arithmetic the bands must reproduce bit for bit)."""
    from tests._band_cpu import OracleCompute
    out = bands.forward_emulated(_t(noisy), [_t(z) for z in logits], _t(demod), ksize=k, bands=1,
                                 compute=OracleCompute(k))
    return out[0].permute(1, 2, 0).numpy()


def test_band_protocol_local_lockstep_bitwise():
    """All bands in one process (LocalTransport, the GPU emulation's driver)
    with the oracle arithmetic: bitwise equal to oracle.forward, 4 bands."""
    from oracle import pyramid as op
    from tests._band_cpu import OracleCompute
    H, W, L, k = 96, 16, 3, 5
    noisy, demod, logits = _frame(H, W, L, k, seed=3)
    out = bands.forward_emulated(_t(noisy), [_t(z) for z in logits], _t(demod), ksize=k, bands=4,
                                 compute=OracleCompute(k))
    np.testing.assert_array_equal(out[0].permute(1, 2, 0).numpy(), _single_band(noisy, demod, logits, k))
    full, _ = op.forward(noisy, logits, None, demod, k=k)
    np.testing.assert_allclose(out[0].permute(1, 2, 0).numpy(), full, rtol=1e-13, atol=1e-13 * np.abs(full).max())
