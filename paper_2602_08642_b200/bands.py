"""Row-band decomposition of one frame across GPUs.

A frame too large for one GPU's step (8K, 4-level 7x7) is split into G row
bands.  Each band owns rows [y0, y1) whose boundaries are multiples of
2^(L-1), so the count-correct pooling is band-local at every level.  The
pyramid forward of an output row depends on a finite cone of input rows:
the k x k gather reaches r level-l rows (= r * 2^l fine rows) and the
upsample one coarse parent row, at every level, so

    halo(L, k) = align_up(sum_{l<L} (r + 2) * 2^l, 2^(L-1))

input rows above and below suffice for the band's rows to be exact.  Each
band receives those halo rows of its inputs (noisy, demod, logits of every
level) from its neighbours in ONE exchange round -- peer-to-peer over NVLink
(torch.distributed point-to-point between the one-process-per-GPU ranks; no
collective), or device-to-device copies when bands are emulated on one GPU --
then runs the unmodified single-GPU forward on its extended crop and keeps
its own rows.  Because every output pixel's arithmetic is independent of
where the crop starts, the stitched output equals the single-GPU full-frame
output bit for bit (tests/test_gpu_bands.py).

Alternative designs (exchanging pooled levels and Lhat rows per level,
SURVEY.md 8(e) variant 1) move less data but need one round per level; with
NVLink at ~770 GB/s the single input round costs ~(2 halo x W x 300 B) /
770 GB/s ~ 0.1 ms at 8K k7, overlappable with the band interior.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops


@dataclass(frozen=True)
class Band:
    index: int
    own: tuple[int, int]   # rows this band outputs
    ext: tuple[int, int]   # rows of input it needs (own + halo, clipped to the frame)


def halo_rows(levels: int, ksize: int) -> int:
    r = ksize // 2
    align = 1 << (levels - 1)
    cone = sum((r + 2) << l for l in range(levels))
    return -(-cone // align) * align


def plan(height: int, levels: int, ksize: int, bands: int) -> list[Band]:
    """Split `height` rows into `bands` aligned bands (as equal as alignment allows)."""
    align = 1 << (levels - 1)
    units = -(-height // align)
    if bands < 1 or bands > units:
        raise ValueError(f"cannot split {height} rows into {bands} bands of >= {align} rows")
    halo = halo_rows(levels, ksize)
    out, start = [], 0
    for g in range(bands):
        n = units // bands + (1 if g < units % bands else 0)
        y0, y1 = start * align, min((start + n) * align, height)
        out.append(Band(g, (y0, y1), (max(0, y0 - halo), min(height, y1 + halo))))
        start += n
    if bands > 1 and min(b.own[1] - b.own[0] for b in out) < halo:
        raise ValueError(f"bands of {height // bands} rows are thinner than the {halo}-row halo; "
                         "use fewer bands")
    return out


def level_rows(rows: tuple[int, int], level: int, height: int) -> tuple[int, int]:
    """Rows of level `level` covering fine rows [a, b) (a aligned)."""
    a, b = rows
    hl = -(-height // (1 << level))
    return a >> level, min(-(-b // (1 << level)), hl)


def crop_inputs(noisy, demod, logits, band: Band, height: int):
    """Slice a band's extended crop out of full-frame tensors (emulation and tests)."""
    e0, e1 = band.ext
    cl = []
    for l, z in enumerate(logits):
        a, b = level_rows((e0, e1), l, height)
        cl.append(z[:, :, a:b].contiguous())
    return (noisy[:, :, e0:e1].contiguous(),
            demod[:, :, e0:e1].contiguous() if demod is not None else None, cl)


def forward_emulated(noisy, logits, demod=None, *, ksize, bands: int):
    """All bands on the tensors' device, one after another (correctness
    reference for the distributed path; the exchange is a D2D slice)."""
    H = noisy.shape[2]
    out = torch.empty_like(noisy)
    for band in plan(H, len(logits), ksize, bands):
        n, d, lg = crop_inputs(noisy, demod, logits, band, H)
        o, _ = ops.pyramid_forward(n, lg, d, ksize=ksize)
        y0, y1 = band.own
        e0 = band.ext[0]
        out[:, :, y0:y1] = o[:, :, y0 - e0:y1 - e0]
    return out


# ---------------------------------------------------------------------------
# distributed: one process per GPU, each holding its own band's rows


def _exchange_rows(dist, rank, world, own_t, rows_own, rows_ext, halo_up_rows, halo_dn_rows):
    """Assemble the extended crop of one tensor (rows along dim 2) from the
    own rows plus halo rows received from rank-1 (above) and rank+1 (below).

    own_t: this rank's own rows [o0, o1); rows_ext: [e0, e1).  The neighbour
    above sends its last (o0 - e0) rows, the one below its first (e1 - o1)."""
    o0, o1 = rows_own
    e0, e1 = rows_ext
    shape = list(own_t.shape)
    shape[2] = e1 - e0
    ext = torch.empty(shape, dtype=own_t.dtype, device=own_t.device)
    ext[:, :, o0 - e0:o1 - e0] = own_t
    reqs = []
    if rank > 0:
        n_up = halo_up_rows  # rows this rank must send up = what rank-1 needs below
        if n_up > 0:
            reqs.append(dist.isend(own_t[:, :, :n_up].contiguous(), rank - 1))
        if o0 - e0 > 0:
            buf_up = torch.empty_like(ext[:, :, :o0 - e0])
            reqs.append(("recv", dist.irecv(buf_up, rank - 1), buf_up, 0))
    if rank < world - 1:
        n_dn = halo_dn_rows
        if n_dn > 0:
            reqs.append(dist.isend(own_t[:, :, own_t.shape[2] - n_dn:].contiguous(), rank + 1))
        if e1 - o1 > 0:
            buf_dn = torch.empty_like(ext[:, :, o1 - e0:])
            reqs.append(("recv", dist.irecv(buf_dn, rank + 1), buf_dn, o1 - e0))
    for r in reqs:
        if isinstance(r, tuple):
            _, req, buf, at = r
            req.wait()
            ext[:, :, at:at + buf.shape[2]] = buf
        else:
            r.wait()
    return ext


def exchange_band_inputs(dist, rank, world, band_list, height, noisy_own, demod_own, logits_own):
    """One exchange round: every input's halo rows from the neighbours.
    Returns the extended-crop tensors (noisy, demod, logits)."""
    b = band_list[rank]
    up = band_list[rank - 1] if rank > 0 else None
    dn = band_list[rank + 1] if rank < world - 1 else None

    def rows_for(level):
        own = level_rows(b.own, level, height)
        ext = level_rows(b.ext, level, height)
        # rows the neighbour above needs from us (its ext end beyond its own end)
        send_up = 0
        if up is not None:
            up_ext_end = level_rows(up.ext, level, height)[1]
            send_up = max(0, up_ext_end - own[0])
        send_dn = 0
        if dn is not None:
            dn_ext_start = level_rows(dn.ext, level, height)[0]
            send_dn = max(0, own[1] - dn_ext_start)
        return own, ext, send_up, send_dn

    own, ext, su, sd = rows_for(0)
    n = _exchange_rows(dist, rank, world, noisy_own, own, ext, su, sd)
    d = _exchange_rows(dist, rank, world, demod_own, own, ext, su, sd) if demod_own is not None else None
    lg = []
    for l, z in enumerate(logits_own):
        own_l, ext_l, su_l, sd_l = rows_for(l)
        lg.append(_exchange_rows(dist, rank, world, z, own_l, ext_l, su_l, sd_l))
    return n, d, lg


def forward_distributed(dist, rank, world, height, noisy_own, logits_own, demod_own=None, *,
                        ksize):
    """This rank's band of the frame: exchange halos, run the single-GPU
    forward on the extended crop, return the band's own output rows."""
    levels = len(logits_own)
    band_list = plan(height, levels, ksize, world)
    n, d, lg = exchange_band_inputs(dist, rank, world, band_list, height, noisy_own, demod_own,
                                    logits_own)
    out, _ = ops.pyramid_forward(n, lg, d, ksize=ksize)
    b = band_list[rank]
    return out[:, :, b.own[0] - b.ext[0]:b.own[1] - b.ext[0]]
