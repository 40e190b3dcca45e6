"""Row-band decomposition of one frame across GPUs.

A frame too large for one GPU's step (8K, 4-level 7x7) is split into G row
bands, one per GPU.  Band boundaries are multiples of 2^(L-1) rows, so the
count-correct pooling is band-local at every level, and every band owns its
rows of every level: its inputs (noisy, demod, the logits of each level) and
its outputs.  Only the data the survey's "variant 1" names crosses a
boundary (no logits ever do):

* round A, once: the Rh = even(r) nearest rows of each pooled level L^l
  (level 0: noisy and demod) to each neighbour -- the k x k gather of the
  band's edge rows reaches r rows into the neighbour;
* round B_l, once per level l >= 1 during the coarse-to-fine sweep: the
  band's first Lhat^l row to the neighbour above -- the parent
  floor((y + 1) / 2) of that neighbour's last fine row (pyramid.py:227).

That is ~1.1 MB per boundary and direction at 8K k7 fp32 (level 0: 4 rows x
7680 x 24 B), against ~1.3 GB of HBM traffic per band.  Transfers are posted
coarse levels first and level 0 last, and each is waited on only right
before the level that reads it, so the large level-0 halo moves while the
coarse levels compute.

Layout per band and level l (H_l own rows): row-extended buffers of
H_l + 2 Rh rows -- the image (halo rows received, or at the frame's top and
bottom edge replicas of the edge row, which is exactly the reference's
clamp), the logits (halo rows zero: their outputs are never used), the
output Lhat^l, and for l >= 1 the parent buffer P^l = Lhat^l rows
[-Rh/2, H_l + Rh/2) with row H_l + Rh/2 received from the neighbour below
(or a replica of the last row at the frame bottom), so that fine extended
row q has parent (q + i) / 2 in P^l exactly as in the full frame.  Every
level runs the library's own fused level kernel (ssb_pyr_forward_level) on
these buffers, so each output pixel's arithmetic is the full-frame call's:
the stitched output is bitwise equal (tests/test_gpu_bands.py).

Transports (same protocol, same tags):
* LocalTransport  -- all bands in one process (emulation / tests);
* GlooTransport   -- one process per band over torch.distributed point to
  point (the CPU protocol test, tests/test_bands_dist.py);
* PeerTransport   -- one process per GPU: the neighbours' receive buffers are
  mapped through CUDA IPC at setup, and each transfer is one P2P-store
  kernel plus a system-scope generation flag (ssb_halo_put), waited on by
  the consumer's stream (ssb_flag_wait): no NCCL, no host round trip.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Band:
    index: int
    own: tuple[int, int]  # level-0 rows this band owns (and outputs)


def halo(ksize: int) -> int:
    """Rows exchanged per level: the gather radius, rounded up to even (the
    parent buffers start Rh/2 coarse rows above the band)."""
    r = ksize // 2
    return r + (r & 1)


def level_rows(rows: tuple[int, int], level: int, height: int) -> tuple[int, int]:
    """Rows of level `level` owned by level-0 rows [a, b) (a aligned)."""
    a, b = rows
    hl = -(-height // (1 << level))
    return a >> level, min(-(-b // (1 << level)), hl)


def plan(height: int, levels: int, ksize: int, bands: int) -> list[Band]:
    """Split `height` rows into `bands` bands aligned to 2^(L-1) (as equal as
    alignment allows); every band needs >= Rh rows at every level."""
    align = 1 << (levels - 1)
    units = -(-height // align)
    if bands < 1 or bands > units:
        raise ValueError(f"cannot split {height} rows into {bands} bands of >= {align} rows")
    out, start = [], 0
    for g in range(bands):
        n = units // bands + (1 if g < units % bands else 0)
        out.append(Band(g, (start * align, min((start + n) * align, height))))
        start += n
    rh = halo(ksize)
    for b in out:
        for l in range(levels):
            a, e = level_rows(b.own, l, height)
            if bands > 1 and e - a < rh:
                raise ValueError(f"band {b.index} has {e - a} rows at level {l} (< the {rh}-row halo); "
                                 "use fewer bands")
    return out


def halo_bytes(width: int, levels: int, ksize: int, channels: int = 3, esz: int = 4) -> int:
    """Bytes one band sends to one neighbour per frame (round A + rounds B)."""
    rh = halo(ksize)
    total = 0
    for l in range(levels):
        wl = -(-width // (1 << l))
        total += rh * wl * channels * esz * (2 if l == 0 else 1)
        if l >= 1:
            total += wl * channels * esz
    return total


# ---------------------------------------------------------------------------
# compute back ends


class CudaCompute:
    """The library's kernels (the product path)."""

    def __init__(self, ksize: int, blend: str = "native"):
        from . import ops
        self.ops, self.k, self.blend = ops, ksize, blend

    def pool(self, src, dst, demod=None):
        self.ops.pool2_into(src, dst, demod)

    def forward_level(self, img, logits, demod, parent, out):
        self.ops.pyramid_forward_level(img, logits, ksize=self.k, demod=demod, coarse=parent, out=out,
                                       blend=self.blend)


# ---------------------------------------------------------------------------
# one band


class BandForward:
    """Buffers and protocol of one band.  Write the band's inputs into
    `noisy_own`, `demod_own`, `logits_own[l]` (views of the extended
    buffers), then drive `steps(transport)` (a generator: one yield between
    posting a round's sends and consuming its receives, so emulated bands can
    run in lockstep); the output rows are `out_own`."""

    def __init__(self, bands: list[Band], index: int, height: int, width: int, levels: int, ksize: int,
                 compute, *, channels: int = 3, batch: int = 1, dtype=torch.float32, logit_dtype=None,
                 device="cuda", demod: bool = True, blend: str = "native", alloc=None):
        self.bands, self.index, self.band = bands, index, bands[index]
        self.H, self.W, self.L, self.k = height, width, levels, ksize
        self.compute, self.rh = compute, halo(ksize)
        self.up = index - 1 if index > 0 else None
        self.dn = index + 1 if index < len(bands) - 1 else None
        alloc = alloc or (lambda shape, dt: torch.empty(shape, dtype=dt, device=device))
        ldt = logit_dtype or dtype
        rh = self.rh
        self.rows = [level_rows(self.band.own, l, height) for l in range(levels)]
        self.hl = [b - a for a, b in self.rows]
        self.wl = [-(-width // (1 << l)) for l in range(levels)]
        ncl = lambda l: ksize * ksize + ((4 if blend == "native" else 1) if l < levels - 1 else 0)  # noqa: E731
        self.img = [alloc((batch, channels, self.hl[l] + 2 * rh, self.wl[l]), dtype) for l in range(levels)]
        self.dem = alloc((batch, channels, self.hl[0] + 2 * rh, self.wl[0]), dtype) if demod else None
        self.logit = [alloc((batch, ncl(l), self.hl[l] + 2 * rh, self.wl[l]), ldt) for l in range(levels)]
        for z in self.logit:  # halo rows: zero logits (their outputs are discarded)
            z[:, :, :rh].zero_()
            z[:, :, rh + z.shape[2] - 2 * rh:].zero_()
        self.out = [alloc((batch, channels, self.hl[l] + 2 * rh, self.wl[l]), dtype) for l in range(levels)]
        self.par = [None] + [alloc((batch, channels, self.hl[l] + rh + 1, self.wl[l]), dtype)
                             for l in range(1, levels)]
        self.noisy_own = self.img[0][:, :, rh:rh + self.hl[0]]
        self.demod_own = self.dem[:, :, rh:rh + self.hl[0]] if demod else None
        self.logits_own = [z[:, :, rh:rh + self.hl[l]] for l, z in enumerate(self.logit)]
        self.out_own = self.out[0][:, :, rh:rh + self.hl[0]]

    # -- receive targets of this band (tags are the same on both sides)
    def recv_view(self, tag):
        kind, l, side = tag
        rh, h = self.rh, self.hl[l]
        if kind in ("img", "dem"):
            buf = self.img[l] if kind == "img" else self.dem
            return buf[:, :, :rh] if side == "top" else buf[:, :, rh + h:]
        if kind == "par":  # the parent row below the band's own coarse rows
            return self.par[l][:, :, rh // 2 + h:rh // 2 + h + 1]
        raise KeyError(tag)

    def send_view(self, tag):
        """The rows this band sends for `tag` (named by the RECEIVER's slot):
        ("img", l, "bottom") goes to the band above (its bottom halo) = this
        band's first Rh own rows; ("img", l, "top") to the band below = its
        last Rh own rows; ("par", l, -) to the band above = own Lhat^l row 0."""
        kind, l, side = tag
        rh, h = self.rh, self.hl[l]
        if kind in ("img", "dem"):
            buf = self.img[l] if kind == "img" else self.dem
            return buf[:, :, rh:2 * rh] if side == "bottom" else buf[:, :, h:h + rh]
        if kind == "par":
            return self.out[l][:, :, rh:rh + 1]
        raise KeyError(tag)

    def _edge_fill(self):
        """Frame top / bottom: replicate the edge row into the halo (= the
        reference's clamp-to-edge, pyramid.py:173-182)."""
        rh = self.rh
        bufs = [(l, b) for l, b in enumerate(self.img)] + ([(0, self.dem)] if self.dem is not None else [])
        for l, b in bufs:
            h = self.hl[l]
            if self.up is None:
                b[:, :, :rh].copy_(b[:, :, rh:rh + 1].expand(-1, -1, rh, -1))
            if self.dn is None:
                b[:, :, rh + h:].copy_(b[:, :, rh + h - 1:rh + h].expand(-1, -1, rh, -1))

    def _image_tags(self, l):
        kinds = ["img", "dem"] if (l == 0 and self.dem is not None) else ["img"]
        return [(kd, l) for kd in kinds]

    def steps(self, tr):
        """The protocol (generator).  `tr` is this band's transport."""
        rh, L = self.rh, self.L
        tr.begin_frame()
        # pooled levels of the own rows (band-local: boundaries are aligned)
        for l in range(1, L):
            src = self.img[l - 1][:, :, rh:rh + self.hl[l - 1]]
            dst = self.img[l][:, :, rh:rh + self.hl[l]]
            dm = self.dem[:, :, rh:rh + self.hl[0]] if (l == 1 and self.dem is not None) else None
            self.compute.pool(src, dst, dm)
        self._edge_fill()
        # round A: coarse levels first, level 0 (the big one) last
        for l in range(L - 1, -1, -1):
            for kd, _ in self._image_tags(l):
                if self.up is not None:
                    tr.send(self.up, (kd, l, "bottom"), self.send_view((kd, l, "bottom")))
                if self.dn is not None:
                    tr.send(self.dn, (kd, l, "top"), self.send_view((kd, l, "top")))
        yield "A"
        for l in range(L - 1, -1, -1):
            for kd, _ in self._image_tags(l):
                if self.up is not None:
                    tr.recv(self.up, (kd, l, "top"), self.recv_view((kd, l, "top")))
                if self.dn is not None:
                    tr.recv(self.dn, (kd, l, "bottom"), self.recv_view((kd, l, "bottom")))
            parent = self.par[l + 1] if l < L - 1 else None
            self.compute.forward_level(self.img[l], self.logit[l], self.dem if l == 0 else None, parent,
                                       self.out[l])
            if l >= 1:
                h = self.hl[l]
                # P^l = Lhat^l rows [-Rh/2, H_l + Rh/2): own rows + the halo
                # rows' parents (values unused), then the boundary row
                self.par[l][:, :, :rh // 2 + h].copy_(self.out[l][:, :, rh - rh // 2:rh + h])
                if self.up is not None:
                    tr.send(self.up, ("par", l, "-"), self.send_view(("par", l, "-")))
                yield f"B{l}"
                if self.dn is not None:
                    tr.recv(self.dn, ("par", l, "-"), self.recv_view(("par", l, "-")))
                else:  # frame bottom: the clamp onto the last coarse row
                    self.par[l][:, :, rh // 2 + h:].copy_(
                        self.out[l][:, :, rh + h - 1:rh + h].expand(-1, -1, rh // 2 + 1, -1))
                if self.dn is not None and rh // 2 > 0:
                    # rows past the received one: only parents of halo rows
                    self.par[l][:, :, rh // 2 + h + 1:].copy_(
                        self.par[l][:, :, rh // 2 + h:rh // 2 + h + 1].expand(-1, -1, rh // 2, -1))
        tr.end_frame()
        yield "done"

    def run(self, tr):
        for _ in self.steps(tr):
            pass
        return self.out_own


# ---------------------------------------------------------------------------
# transports


class LocalTransport:
    """All bands in one process: a send hands the source view to a mailbox;
    the matching receive copies it (bands advance in lockstep, so every
    send of a round precedes its receives)."""

    def __init__(self, mailbox: dict, me: int):
        self.box, self.me = mailbox, me

    def send(self, peer, tag, src):
        self.box[(self.me, peer, tag)] = src

    def recv(self, peer, tag, dst):
        dst.copy_(self.box.pop((peer, self.me, tag)))

    def begin_frame(self):
        pass

    def end_frame(self):
        pass


class GlooTransport:
    """One process per band over torch.distributed point to point (gloo:
    sends are buffered, so posting sends before receives cannot deadlock)."""

    def __init__(self, dist):
        self.dist, self.pending = dist, []

    @staticmethod
    def _tag(tag):
        kind, l, side = tag  # the same integer in every process
        return (("img", "dem", "par").index(kind) * 16 + l) * 3 + ("top", "bottom", "-").index(side) + 1

    def send(self, peer, tag, src):
        self.pending.append(self.dist.isend(src.contiguous(), peer, tag=self._tag(tag)))

    def recv(self, peer, tag, dst):
        buf = torch.empty_like(dst, memory_format=torch.contiguous_format)
        self.dist.recv(buf, peer, tag=self._tag(tag))
        dst.copy_(buf)

    def begin_frame(self):
        pass

    def end_frame(self):
        for r in self.pending:
            r.wait()
        self.pending = []


class PeerTransport:
    """One process per GPU (torchrun).  setup() maps the neighbours' band
    buffers and flag words into this process through CUDA IPC (handles
    traded once through the process group: plumbing, not the data path) and
    enables peer access; send() is one ssb_halo_put (P2P stores into the
    neighbour's receive slot + a system-scope release of the frame's
    generation on the neighbour's flag for that tag), recv() an
    ssb_flag_wait on this band's own flag.  Flags count frames, so buffers
    are reused frame after frame without resets."""

    def __init__(self, dist, band: BandForward, device):
        from . import ops
        self.ops, self.dist, self.band, self.dev = ops, dist, band, torch.device(device)
        self.tags = []
        for l in range(band.L):
            for kd, _ in band._image_tags(l):
                self.tags += [(kd, l, "top"), (kd, l, "bottom")]
            if l >= 1:
                self.tags.append(("par", l, "-"))
        # one flag per incoming tag, plus "the neighbour above / below has
        # finished reading this band's frame" (back-pressure for the next frame)
        self.flags = torch.zeros(len(self.tags) + 2, dtype=torch.int32, device=self.dev)
        self.done_up, self.done_dn = len(self.tags), len(self.tags) + 1
        self.gen = 0
        self.peers = {}

    def setup(self):
        from torch.multiprocessing.reductions import reduce_tensor
        b = self.band
        mine = {"img": [reduce_tensor(t) for t in b.img], "dem": reduce_tensor(b.dem) if b.dem is not None else None,
                "par": [None] + [reduce_tensor(t) for t in b.par[1:]], "flags": reduce_tensor(self.flags),
                "device": self.dev.index}
        allh = [None] * self.dist.get_world_size()
        self.dist.all_gather_object(allh, mine)
        for peer in (b.up, b.dn):
            if peer is None:
                continue
            h = allh[peer]
            self.ops.enable_peer(self.dev.index, h["device"])
            rebuild = lambda r: r[0](*r[1]) if r is not None else None  # noqa: E731
            shadow = BandForward.__new__(BandForward)
            shadow.__dict__.update({k: v for k, v in b.__dict__.items()})
            pb = b.bands[peer]
            shadow.band, shadow.index = pb, peer
            shadow.rows = [level_rows(pb.own, l, b.H) for l in range(b.L)]
            shadow.hl = [e - a for a, e in shadow.rows]
            shadow.img = [rebuild(r) for r in h["img"]]
            shadow.dem = rebuild(h["dem"])
            shadow.par = [None] + [rebuild(r) for r in h["par"][1:]]
            self.peers[peer] = (shadow, rebuild(h["flags"]))

    def begin_frame(self):
        # the neighbours must have consumed the previous frame's halos before
        # this frame's land in their buffers
        self.gen += 1
        if self.band.up is not None:
            self.ops.flag_wait(self.flags[self.done_up], self.gen - 1, self.dev)
        if self.band.dn is not None:
            self.ops.flag_wait(self.flags[self.done_dn], self.gen - 1, self.dev)

    def send(self, peer, tag, src):
        shadow, pflags = self.peers[peer]
        self.ops.halo_put(shadow.recv_view(tag), src, pflags[self.tags.index(tag)], self.gen)

    def recv(self, peer, tag, dst):
        self.ops.flag_wait(self.flags[self.tags.index(tag)], self.gen, self.dev)

    def end_frame(self):
        # tell each neighbour its halos of this frame are consumed (an empty
        # put: just the release of the generation on the neighbour's flag)
        b = self.band
        for peer, slot in ((b.up, self.done_dn), (b.dn, self.done_up)):
            if peer is not None:
                self.ops.flag_release(self.peers[peer][1][slot], self.gen, self.dev)


# ---------------------------------------------------------------------------
# drivers


def forward_emulated(noisy, logits, demod=None, *, ksize, bands: int, blend="native", compute=None):
    """All bands of one frame on the tensors' device, in lockstep through
    LocalTransport (the correctness reference of the distributed path):
    returns the stitched (B, C, H, W) output."""
    B, Cc, H, W = noisy.shape
    L = len(logits)
    pl = plan(H, L, ksize, bands)
    compute = compute or CudaCompute(ksize, blend)
    engines = []
    for g in range(bands):
        e = BandForward(pl, g, H, W, L, ksize, compute, channels=Cc, batch=B, dtype=noisy.dtype,
                        logit_dtype=logits[0].dtype, device=noisy.device, demod=demod is not None, blend=blend)
        a, b = pl[g].own
        e.noisy_own.copy_(noisy[:, :, a:b])
        if demod is not None:
            e.demod_own.copy_(demod[:, :, a:b])
        for l, z in enumerate(logits):
            la, lb = level_rows(pl[g].own, l, H)
            e.logits_own[l].copy_(z[:, :, la:lb])
        engines.append(e)
    box = {}
    gens = [e.steps(LocalTransport(box, g)) for g, e in enumerate(engines)]
    live = list(range(bands))
    while live:
        nxt = []
        for g in live:
            if next(gens[g]) != "done":
                nxt.append(g)
        live = nxt
    out = torch.empty_like(noisy)
    for g, e in enumerate(engines):
        a, b = pl[g].own
        out[:, :, a:b] = e.out_own
    return out
