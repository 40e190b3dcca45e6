"""Torch-tensor API over the sm_100a kernels (device-resident, planar layout).

Layouts (all contiguous CUDA tensors):
  images  (B, C, H, W)   float32 or float64, any C
  logits  list over levels l of (B, C_l, H_l, W_l), H_l = ceil(H / 2^l),
          C_l = k*k (+4 upsample logits, or +1 tied blend logit, if l < L-1)
          (+k*k temporal logits at l = 0 when a history `prev` is given)
          float32 / bfloat16 (with float32 images) or float64 (with float64)

Every call goes through libssb200.so (include/ssb_api.h) on the current torch
stream.  There is no eager/PyTorch fallback for any op in this module.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check

_DT = {torch.float32: _lib.SSB_F32, torch.bfloat16: _lib.SSB_BF16, torch.float64: _lib.SSB_F64}


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _need(t, name, device=None, dtype=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} must live on {device}")
    return t


# ---------------------------------------------------------------------------
# geometry


def level_shapes(height: int, width: int, levels: int) -> list[tuple[int, int]]:
    shapes = [(height, width)]
    while len(shapes) < levels:
        h, w = shapes[-1]
        shapes.append(((h + 1) // 2, (w + 1) // 2))
    return shapes


def logit_channels(level: int, levels: int, ksize: int, has_prev: bool = False,
                   blend: str = "native") -> int:
    n = ksize * ksize
    if level < levels - 1:
        n += 4 if blend == "native" else 1
    if level == 0 and has_prev:
        n += ksize * ksize
    return n


def _desc(noisy, logits, demod, prev, ksize, blend) -> _lib.PyrDesc:
    B, Cc, H, W = noisy.shape
    L = len(logits)
    if L < 1 or L > _lib.SSB_MAX_LEVELS:
        raise ValueError(f"need 1..{_lib.SSB_MAX_LEVELS} levels of logits")
    if ksize is None:
        k2 = logits[-1].shape[1]
        ksize = int(round(k2 ** 0.5))
    if blend not in ("native", "tied"):
        raise ValueError("blend must be 'native' or 'tied'")
    for l, ((h, w), z) in enumerate(zip(level_shapes(H, W, L), logits)):
        expect = (B, logit_channels(l, L, ksize, prev is not None, blend), h, w)
        if tuple(z.shape) != expect:
            raise ValueError(f"level {l} logits must have shape {expect}, got {tuple(z.shape)}")
        if z.dtype != logits[0].dtype:
            raise ValueError("all logit levels must share one dtype")
    d = _lib.PyrDesc()
    d.batch, d.channels, d.height, d.width = B, Cc, H, W
    d.levels, d.ksize = L, ksize
    d.image_dtype = _DT[noisy.dtype]
    d.logit_dtype = _DT[logits[0].dtype]
    d.has_prev = int(prev is not None)
    d.has_demod = int(demod is not None)
    d.blend_mode = _lib.SSB_BLEND_TIED if blend == "tied" else _lib.SSB_BLEND_NATIVE
    return d


@dataclass
class PyramidTape:
    """Device tape of one forward call (opaque to callers, like the reference's
    ReconTape): pooled levels and partial reconstructions plus the inputs."""
    desc: _lib.PyrDesc
    buf: torch.Tensor | None
    noisy: torch.Tensor
    logits: list
    demod: torch.Tensor | None
    prev: torch.Tensor | None
    out: torch.Tensor
    demod_given: bool = True  # False: demod is the identity stand-in below

    @property
    def levels(self) -> int:
        return self.desc.levels


@dataclass
class PyramidGrads:
    logits: list | None
    demod: torch.Tensor | None
    input: torch.Tensor
    prev: torch.Tensor | None


_IDENTITY_DEMOD: dict = {}


def _identity_demod(noisy):
    """demod=None (reconstruct_core's default) on the float32 3-channel path
    runs the fused demodulating level kernels (TMA pipeline, level-0-last
    backward) with an all-ones demod: max(1, 1e-3) = 1 and rcp(1) = 1 exactly,
    so outputs and input gradients are those of the undemodulated filter; the
    ones are allocated once per shape and device (SSB_NO_IDENTITY_DEMOD=1 keeps
    the generic no-demod kernels)."""
    key = (noisy.device, tuple(noisy.shape))
    t = _IDENTITY_DEMOD.get(key)
    if t is None:
        t = torch.ones(noisy.shape, dtype=torch.float32, device=noisy.device)
        _IDENTITY_DEMOD[key] = t
    return t


def pyramid_forward(noisy, logits, demod=None, prev=None, *, ksize=None, blend="native",
                    out=None) -> tuple[torch.Tensor, PyramidTape]:
    """Coarse-to-fine reconstruction (ref pyramid.py `reconstruct_core`)."""
    lib = _lib.load()
    _need(noisy, "noisy")
    if noisy.dim() != 4 or noisy.dtype not in (torch.float32, torch.float64):
        raise ValueError("noisy must be (B, C, H, W) float32/float64")
    dev = noisy.device
    logits = [_need(z, f"logits[{l}]", dev) for l, z in enumerate(logits)]
    for name, t in (("demod", demod), ("prev", prev)):
        if t is not None:
            _need(t, name, dev, noisy.dtype)
            if t.shape != noisy.shape:
                raise ValueError(f"{name} must match noisy's shape")
    demod_given = demod is not None
    if (demod is None and prev is None and noisy.dtype == torch.float32 and noisy.shape[1] == 3
            and len(logits) >= 2 and os.environ.get("SSB_NO_IDENTITY_DEMOD") != "1"):
        demod = _identity_demod(noisy)
    d = _desc(noisy, logits, demod, prev, ksize, blend)
    tb = C.c_size_t()
    check(lib.ssb_pyr_tape_bytes(C.byref(d), C.byref(tb)), "ssb_pyr_tape_bytes")
    buf = torch.empty(max(tb.value, 1), dtype=torch.uint8, device=dev)
    if out is None:
        out = torch.empty_like(noisy)
    else:
        _need(out, "out", dev, noisy.dtype)
        if out.shape != noisy.shape:
            raise ValueError("out must match noisy's shape")
    io = _lib.PyrFwdIO()
    io.noisy, io.demod, io.prev, io.out = (_ptr(noisy), _ptr(demod), _ptr(prev), _ptr(out))
    for l, z in enumerate(logits):
        io.logits[l] = z.data_ptr()
    with torch.cuda.device(dev):
        check(lib.ssb_pyr_forward(C.byref(d), C.byref(io), _ptr(buf), _stream(dev)),
              "ssb_pyr_forward")
    return out, PyramidTape(d, buf, noisy, logits, demod, prev, out, demod_given)


def pyramid_backward(tape: PyramidTape, upstream, want_param_grads: bool = True,
                     accumulate_into: list | None = None) -> PyramidGrads:
    """Exact gradients of sum(upstream * out) (ref `reconstruct_backward`).

    accumulate_into: optional list of per-level logit-gradient tensors that
    receive ``+=`` instead of being overwritten (e.g. summing the two frames
    of an optimisation window without an extra pass); each must have exactly
    its level's logits shape (B, C_l, H_l, W_l) -- per-frame accumulators."""
    lib = _lib.load()
    dev = tape.noisy.device
    _need(upstream, "upstream", dev, tape.noisy.dtype)
    if upstream.shape != tape.noisy.shape:
        raise ValueError("upstream must match the filter output's shape")
    d = tape.desc
    wb = C.c_size_t()
    check(lib.ssb_pyr_workspace_bytes(C.byref(d), C.byref(wb)), "ssb_pyr_workspace_bytes")
    ws = torch.empty(max(wb.value, 1), dtype=torch.uint8, device=dev)
    g_noisy = torch.empty_like(tape.noisy)
    g_demod = (torch.empty_like(tape.noisy)
               if (want_param_grads and tape.demod is not None and tape.demod_given) else None)
    g_prev = torch.empty_like(tape.noisy) if tape.prev is not None else None
    io = _lib.PyrBwdIO()
    io.noisy, io.demod, io.prev = _ptr(tape.noisy), _ptr(tape.demod), _ptr(tape.prev)
    io.out, io.upstream = _ptr(tape.out), _ptr(upstream)
    io.g_noisy, io.g_demod, io.g_prev = _ptr(g_noisy), _ptr(g_demod), _ptr(g_prev)
    g_logits = None
    if want_param_grads:
        if accumulate_into is not None:
            # one (B, C_l, H_l, W_l) tensor per level, the logits' own shape:
            # the kernels index it per frame (no frame-summed accumulators)
            if len(accumulate_into) != len(tape.logits):
                raise ValueError(f"accumulate_into needs {len(tape.logits)} tensors, got {len(accumulate_into)}")
            g_logits = [_need(g, f"accumulate_into[{l}]", dev, z.dtype)
                        for l, (g, z) in enumerate(zip(accumulate_into, tape.logits))]
            for l, (g, z) in enumerate(zip(g_logits, tape.logits)):
                if g.shape != z.shape:
                    raise ValueError(f"accumulate_into[{l}] must have the logits' shape {tuple(z.shape)}, "
                                     f"got {tuple(g.shape)}")
            io.accumulate_logits = 1
        else:
            g_logits = [torch.empty_like(z) for z in tape.logits]
        for l, g in enumerate(g_logits):
            io.g_logits[l] = g.data_ptr()
    for l, z in enumerate(tape.logits):
        io.logits[l] = z.data_ptr()
    with torch.cuda.device(dev):
        check(lib.ssb_pyr_backward(C.byref(d), C.byref(io), _ptr(tape.buf), _ptr(ws), _stream(dev)),
              "ssb_pyr_backward")
    return PyramidGrads(g_logits, g_demod, g_noisy, g_prev)


class _PyramidFilterFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, noisy, demod, prev, ksize, blend, *logits):
        out, tape = pyramid_forward(noisy, list(logits), demod, prev, ksize=ksize, blend=blend)
        ctx.tape = tape
        ctx.has_demod = demod is not None
        ctx.has_prev = prev is not None
        return out

    @staticmethod
    def backward(ctx, gout):
        want = any(ctx.needs_input_grad[5:]) or (ctx.has_demod and ctx.needs_input_grad[1])
        g = pyramid_backward(ctx.tape, gout.contiguous(), want_param_grads=want)
        glog = g.logits if g.logits is not None else [None] * ctx.tape.levels
        return (g.input, g.demod, g.prev, None, None, *glog)


def pyramid_filter(noisy, logits, demod=None, prev=None, *, ksize=None, blend="native"):
    """Autograd-enabled filter: out = remod(pyramid(demod(noisy), softmax(logits)))."""
    return _PyramidFilterFn.apply(noisy, demod, prev, ksize, blend, *logits)


# ---------------------------------------------------------------------------
# primitives (ref pyramid.py surface helpers)


def softmax_channels(logits, active=None):
    lib = _lib.load()
    _need(logits, "logits")
    B, Cc, H, W = logits.shape
    out = torch.empty_like(logits)
    with torch.cuda.device(logits.device):
        check(lib.ssb_softmax_channels(_DT[logits.dtype], B, Cc, H, W, Cc if active is None else active,
                                       _ptr(logits), _ptr(out), _stream(logits.device)),
              "ssb_softmax_channels")
    return out


def gather(image, weights, ksize):
    lib = _lib.load()
    _need(image, "image")
    _need(weights, "weights", image.device, image.dtype)
    B, Cc, H, W = image.shape
    if tuple(weights.shape) != (B, ksize * ksize, H, W):
        raise ValueError("weights must be (B, k*k, H, W)")
    out = torch.empty_like(image)
    with torch.cuda.device(image.device):
        check(lib.ssb_gather(_DT[image.dtype], B, Cc, H, W, ksize, _ptr(image), _ptr(weights),
                             _ptr(out), _stream(image.device)), "ssb_gather")
    return out


def upsample2(coarse, weights):
    lib = _lib.load()
    _need(coarse, "coarse")
    _need(weights, "weights", coarse.device, coarse.dtype)
    B, Cc, Hc, Wc = coarse.shape
    Hf, Wf = weights.shape[2:]
    if weights.shape[:2] != (B, 4):
        raise ValueError("weights must be (B, 4, Hf, Wf)")
    out = torch.empty((B, Cc, Hf, Wf), dtype=coarse.dtype, device=coarse.device)
    with torch.cuda.device(coarse.device):
        check(lib.ssb_upsample2(_DT[coarse.dtype], B, Cc, Hc, Wc, Hf, Wf, _ptr(coarse),
                                _ptr(weights), _ptr(out), _stream(coarse.device)), "ssb_upsample2")
    return out


def avgpool2(img):
    lib = _lib.load()
    _need(img, "img")
    B, Cc, H, W = img.shape
    out = torch.empty((B, Cc, (H + 1) // 2, (W + 1) // 2), dtype=img.dtype, device=img.device)
    with torch.cuda.device(img.device):
        check(lib.ssb_avgpool2(_DT[img.dtype], B, Cc, H, W, _ptr(img), _ptr(out),
                               _stream(img.device)), "ssb_avgpool2")
    return out


def build_pyramid(img, levels):
    lv = [img]
    for _ in range(levels - 1):
        lv.append(avgpool2(lv[-1]))
    return lv


# ---------------------------------------------------------------------------
# row bands (bands.py): one level on caller-laid-out buffers,
# strided pooling, and the peer-memory halo transport


def pyramid_forward_level(img, logits, *, ksize, demod=None, coarse=None, out=None, blend="native"):
    """One level of the coarse-to-fine reconstruction (ref pyramid.py:321-338)
    on row-extended band buffers: img / demod / out (B, C, H, W), logits
    (B, C_l, H, W) with C_l = k*k (+4 or +1 with a coarse level), coarse
    (B, C, Hc, Wc) whose row min((y + i) / 2, Hc - 1) is fine row y's parent.
    Every output pixel equals the full-frame ssb_pyr_forward's bit for bit."""
    lib = _lib.load()
    _need(img, "img")
    dev = img.device
    B, Cc, H, W = img.shape
    _need(logits, "logits", dev)
    nl = ksize * ksize + ((4 if blend == "native" else 1) if coarse is not None else 0)
    if tuple(logits.shape) != (B, nl, H, W):
        raise ValueError(f"logits must be {(B, nl, H, W)}, got {tuple(logits.shape)}")
    if demod is not None:
        _need(demod, "demod", dev, img.dtype)
        if demod.shape != img.shape:
            raise ValueError("demod must match img")
    hc = wc = 0
    if coarse is not None:
        _need(coarse, "coarse", dev, img.dtype)
        if coarse.dim() != 4 or coarse.shape[:2] != img.shape[:2]:
            raise ValueError("coarse must be (B, C, Hc, Wc)")
        hc, wc = coarse.shape[2], coarse.shape[3]
    if out is None:
        out = torch.empty_like(img)
    else:
        _need(out, "out", dev, img.dtype)
        if out.shape != img.shape:
            raise ValueError("out must match img")
    d = _lib.PyrLevelDesc(B, Cc, H, W, ksize, _DT[img.dtype], _DT[logits.dtype],
                          _lib.SSB_BLEND_TIED if blend == "tied" else _lib.SSB_BLEND_NATIVE,
                          int(coarse is not None), hc, wc, 0)
    with torch.cuda.device(dev):
        check(lib.ssb_pyr_forward_level(C.byref(d), _ptr(img), _ptr(demod), _ptr(logits), _ptr(coarse), _ptr(out),
                                        _stream(dev)), "ssb_pyr_forward_level")
    return out


def pool2_into(src, out, demod=None):
    """Count-correct 2x2 pooling of the (possibly row-offset) view `src`
    (B, C, H, W) into the view `out` (B, C, ceil(H/2), ceil(W/2)),
    demodulating on load when `demod` (same strides as src) is given: the
    pyramid build's own kernel.  Views must keep unit column stride and row
    stride W (row slices of contiguous planar buffers)."""
    lib = _lib.load()
    for name, t in (("src", src), ("out", out)) + ((("demod", demod),) if demod is not None else ()):
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if t.stride(3) != 1 or t.stride(2) != t.shape[3]:
            raise ValueError(f"{name} must be a row slice of a contiguous planar buffer")
    B, Cc, H, W = src.shape
    if tuple(out.shape) != (B, Cc, (H + 1) // 2, (W + 1) // 2):
        raise ValueError("out must be (B, C, ceil(H/2), ceil(W/2))")
    if demod is not None and (demod.shape != src.shape or demod.stride() != src.stride()):
        raise ValueError("demod must match src (shape and strides)")
    with torch.cuda.device(src.device):
        check(lib.ssb_pool2_strided(_DT[src.dtype], B, Cc, H, W, _ptr(src), src.stride(1), src.stride(0),
                                    _ptr(demod), _ptr(out), out.stride(1), out.stride(0), _stream(src.device)),
              "ssb_pool2_strided")
    return out


def halo_put(dst, src, flag=None, value=0):
    """Copy the row block `src` (B, C, rows, W view) into `dst` (same shape;
    may live on a peer GPU mapped through CUDA IPC) with P2P stores, then
    publish `value` into `flag` (int32 element, possibly on the peer) with a
    system-scope release store; stream-ordered on src's device."""
    lib = _lib.load()
    if dst.shape != src.shape or dst.dtype != src.dtype:
        raise ValueError("halo_put: dst and src must match")
    B, Cc, rows, W = src.shape
    for name, t in (("src", src), ("dst", dst)):
        if t.stride(3) != 1 or t.stride(2) != W or t.stride(0) != Cc * t.stride(1):
            raise ValueError(f"halo_put: {name} must be a row slice of a contiguous planar buffer")
    with torch.cuda.device(src.device):
        check(lib.ssb_halo_put(_ptr(dst), dst.stride(1), _ptr(src), src.stride(1), B * Cc, rows, W,
                               src.element_size(), _ptr(flag), int(value), _stream(src.device)), "ssb_halo_put")


def flag_release(flag, value, device=None):
    """Stream-ordered (on `device`'s current stream) system-scope release
    store of `value` into `flag` (an int32 element, possibly a peer GPU's
    mapped through CUDA IPC)."""
    lib = _lib.load()
    p = _ptr(flag)
    dev = device if device is not None else torch.cuda.current_device()
    with torch.cuda.device(dev):
        check(lib.ssb_halo_put(p, 0, p, 0, 1, 0, 1, 4, p, int(value), _stream(dev)), "ssb_halo_put")


def flag_wait(flag, value, device=None):
    """Block the current stream of `device` until flag >= value."""
    lib = _lib.load()
    dev = device or flag.device
    with torch.cuda.device(dev):
        check(lib.ssb_flag_wait(_ptr(flag), int(value), _stream(dev)), "ssb_flag_wait")


def enable_peer(device: int, peer: int):
    check(_lib.load().ssb_enable_peer(int(device), int(peer)), "ssb_enable_peer")


# ---------------------------------------------------------------------------
# placement (ref rng.py, density.py, estimators.py)


def uniform_grid(seed: int, height: int, width: int, frame0: int = 0, batch: int = 1,
                 frames=None, stream_id: int = 0, device="cuda"):
    lib = _lib.load()
    dev = torch.device(device)
    fr = None
    if frames is not None:
        fr = torch.as_tensor(frames, dtype=torch.int64, device=dev).contiguous()
        batch = fr.numel()
    u = torch.empty((batch, height, width), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        check(lib.ssb_uniform_grid(seed & (2**64 - 1), frame0, _ptr(fr), batch, height, width,
                                   stream_id & (2**64 - 1), _ptr(u), _stream(dev)),
              "ssb_uniform_grid")
    return u


def uniform_at(seed: int, frame: int, x: int, y: int, stream_id: int = 0, device="cuda"):
    """One variate u(seed, frame, x, y, stream) (ref rng.pixel_uniform): a
    one-element float64 device tensor."""
    lib = _lib.load()
    dev = torch.device(device)
    u = torch.empty((1,), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        check(lib.ssb_uniform_at(seed & (2**64 - 1), int(frame), int(x), int(y), stream_id & (2**64 - 1), _ptr(u),
                                 _stream(dev)), "ssb_uniform_at")
    return u


def normalize_density(scores, budget: float):
    lib = _lib.load()
    _need(scores, "scores", dtype=torch.float64)
    if scores.dim() == 2:
        scores = scores[None]
    B, H, W = scores.shape
    wb = C.c_size_t()
    check(lib.ssb_density_workspace_bytes(B, H, W, C.byref(wb)), "ssb_density_workspace_bytes")
    ws = torch.empty(wb.value, dtype=torch.uint8, device=scores.device)
    spp = torch.empty_like(scores)
    with torch.cuda.device(scores.device):
        check(lib.ssb_normalize_density(B, H, W, _ptr(scores), float(budget), _ptr(spp), _ptr(ws),
                                        _stream(scores.device)), "ssb_normalize_density")
    return spp


def allocate(spp, mode="stochastic", rank=None, frame0=0, seed=0, rule="stochastic",
             gumbel_temp=1.0):
    lib = _lib.load()
    _need(spp, "spp", dtype=torch.float64)
    if spp.dim() == 2:
        spp = spp[None]
    B, H, W = spp.shape
    if rule not in _lib.RULES:
        raise ValueError(f"unknown take rule {rule!r}")
    if mode not in ("stochastic", "dithered"):
        raise ValueError(f"unknown allocation mode {mode!r}")
    d = _lib.AllocDesc(B, H, W, _lib.RULES[rule], int(mode == "dithered"), 0, seed & (2**64 - 1),
                       frame0, float(gumbel_temp))
    rk = None
    if mode == "dithered":
        if rank is None:
            raise ValueError("dithered allocation requires a mask")
        rk = torch.as_tensor(rank, dtype=torch.int64, device=spp.device).contiguous()
        d.mask_size = rk.shape[0]
    base = torch.empty(spp.shape, dtype=torch.int64, device=spp.device)
    frac = torch.empty_like(spp)
    u = torch.empty_like(spp)
    taken = torch.empty(spp.shape, dtype=torch.uint8, device=spp.device)
    with torch.cuda.device(spp.device):
        check(lib.ssb_allocate(C.byref(d), _ptr(spp), _ptr(rk), _ptr(base), _ptr(frac), _ptr(u),
                               _ptr(taken), _stream(spp.device)), "ssb_allocate")
    return base, frac, u, taken.bool()


def _est_desc(variant, B, H, W, capacity, lam, gumbel_temp, density_floor):
    if variant not in _lib.VARIANTS:
        raise ValueError(f"{variant!r} is not a stochastic variant")
    return _lib.EstimateDesc(B, H, W, _lib.VARIANTS[variant], capacity, 0, float(lam),
                             float(gumbel_temp), float(density_floor))


def stochastic_core(variant, spp, frac, u, base_sum, holdout, lam=10.0, gumbel_temp=1.0,
                    density_floor=1e-8):
    lib = _lib.load()
    for n, t in (("spp", spp), ("frac", frac), ("u", u), ("base_sum", base_sum),
                 ("holdout", holdout)):
        _need(t, n, dtype=torch.float64)
    shape = spp.shape
    n = spp.numel()
    d = _est_desc(variant, 1, 1, n, 1, lam, gumbel_temp, density_floor)
    noisy = torch.empty(shape + (3,), dtype=torch.float64, device=spp.device)
    grad, contrib = torch.empty_like(noisy), torch.empty_like(noisy)
    drawn = torch.empty(shape, dtype=torch.uint8, device=spp.device)
    with torch.cuda.device(spp.device):
        check(lib.ssb_stochastic_core(C.byref(d), _ptr(spp), _ptr(frac), _ptr(u), _ptr(base_sum),
                                      _ptr(holdout), _ptr(noisy), _ptr(grad), _ptr(contrib),
                                      _ptr(drawn), _stream(spp.device)), "ssb_stochastic_core")
    return noisy, grad, contrib, drawn.bool()


def estimate(variant, spp, base, frac, u, samples, lam=10.0, gumbel_temp=1.0,
             density_floor=1e-8, want_planar32=False):
    """Bank read + stochastic_core (ref `_stochastic_estimate`); samples are
    (B, H, W, S, 3) float64 like SampleBank.samples."""
    lib = _lib.load()
    if spp.dim() == 2:
        spp, base, frac, u, samples = spp[None], base[None], frac[None], u[None], samples[None]
    B, H, W = spp.shape
    S = samples.shape[3]
    _need(samples, "samples", dtype=torch.float64)
    d = _est_desc(variant, B, H, W, S, lam, gumbel_temp, density_floor)
    noisy = torch.empty((B, H, W, 3), dtype=torch.float64, device=spp.device)
    grad, contrib = torch.empty_like(noisy), torch.empty_like(noisy)
    used = torch.empty((B, H, W), dtype=torch.int64, device=spp.device)
    n32 = torch.empty((B, 3, H, W), dtype=torch.float32, device=spp.device) if want_planar32 else None
    with torch.cuda.device(spp.device):
        check(lib.ssb_estimate(C.byref(d), _ptr(spp), _ptr(base), _ptr(frac), _ptr(u),
                               _ptr(samples), _ptr(noisy), _ptr(grad), _ptr(contrib), _ptr(used),
                               _ptr(n32), _stream(spp.device)), "ssb_estimate")
    return noisy, grad, contrib, used, n32


def place(scores, bank, budget: float, variant: str = "stochastic", seed: int = 0, frame0: int = 0,
          lam: float = 10.0, gumbel_temp: float = 1.0, density_floor: float = 1e-8, noisy=None,
          want_grad=False, want_spp=False, want_taken=False, want_drawn=False, workspace=None):
    """Fused placement for any stochastic estimator variant (ref
    normalize_density -> allocate(rule=take_rule(variant)) -> estimate over a
    SampleBank; density.py:55-65,209-233, estimators.py:90-149):
    scores (B,H,W) f32, bank (B,S,3,H,W) f32 -> dict with noisy (B,3,H,W) f32
    (>= 0) and, on request, grad (d noisy / d density, (B,3,H,W) f32), spp
    (B,H,W) f32, taken / drawn (B,H,W) u8.  Counts and masks are exact (the
    uniforms are compared as integers against frac * 2^53)."""
    lib = _lib.load()
    _need(scores, "scores", dtype=torch.float32)
    _need(bank, "bank", scores.device, torch.float32)
    if variant not in _lib.VARIANTS:
        raise ValueError(f"{variant!r} is not a stochastic variant")
    if scores.dim() != 3:
        raise ValueError("scores must be (B, H, W)")
    B, H, W = scores.shape
    S = bank.shape[1]
    if bank.dim() != 5 or tuple(bank.shape) != (B, S, 3, H, W):
        raise ValueError("bank must be (B, S, 3, H, W)")
    dev = scores.device
    if noisy is None:
        noisy = torch.empty((B, 3, H, W), dtype=torch.float32, device=dev)
    else:
        _need(noisy, "noisy", dev, torch.float32)
        if tuple(noisy.shape) != (B, 3, H, W):
            raise ValueError("noisy must be (B, 3, H, W)")
    out = {"noisy": noisy}
    out["grad"] = torch.empty((B, 3, H, W), dtype=torch.float32, device=dev) if want_grad else None
    out["spp"] = torch.empty((B, H, W), dtype=torch.float32, device=dev) if want_spp else None
    out["taken"] = torch.empty((B, H, W), dtype=torch.uint8, device=dev) if want_taken else None
    out["drawn"] = torch.empty((B, H, W), dtype=torch.uint8, device=dev) if want_drawn else None
    if workspace is None:
        wb = C.c_size_t()
        check(lib.ssb_density_workspace_bytes(B, H, W, C.byref(wb)), "ssb_density_workspace_bytes")
        workspace = torch.empty(wb.value, dtype=torch.uint8, device=dev)
    d = _lib.PlaceDesc(B, H, W, S, _lib.VARIANTS[variant], 0, seed & (2**64 - 1), frame0, float(budget))
    cfg = _lib.PlaceCfg(float(lam), float(gumbel_temp), float(density_floor))
    io = _lib.PlaceIO(scores.data_ptr(), bank.data_ptr(), noisy.data_ptr(),
                      *[(out[k].data_ptr() if out[k] is not None else None)
                        for k in ("grad", "spp", "taken", "drawn")])
    with torch.cuda.device(dev):
        check(lib.ssb_place(C.byref(d), C.byref(cfg), C.byref(io), _ptr(workspace), _stream(dev)), "ssb_place")
    return out


def place_fused(scores, bank, budget: float, seed: int = 0, frame0: int = 0, noisy=None,
                want_spp=False, want_taken=False, workspace=None):
    """Inference placement (stochastic rule): scores (B,H,W) f32, bank
    (B,S,3,H,W) f32 -> (noisy (B,3,H,W) f32, spp or None, taken or None)."""
    r = place(scores, bank, budget, "stochastic", seed=seed, frame0=frame0, noisy=noisy, want_spp=want_spp,
              want_taken=want_taken, workspace=workspace)
    return r["noisy"], r["spp"], r["taken"]


def infer(scores, bank, demod, logits, budget: float, *, ksize, seed: int = 0, frame0: int = 0,
          noisy=None, out=None, workspace=None):
    """The inference path of one (batch of) frame(s): the stochastic fused
    placement, then reconstruct_core with demod (density.py:55-65,209-233;
    estimators.py:90-149; pyramid.py:292-345), float32, native blend.  Small
    frames (B*H*W <= 2^20, bank capacity 2, W % 4 == 0) run as ONE cooperative
    kernel (``ssb_infer_small``: noisy identical to ``place_fused``, the
    output within float32 rounding of ``pyramid_forward``); others as
    place_fused + pyramid_forward.  ``workspace``: the small-frame kernel's
    (``ssb_infer_small_workspace_bytes``; allocated when None, unused on the
    two-call path).  Returns (out, noisy)."""
    lib = _lib.load()
    _need(scores, "scores", dtype=torch.float32)
    B, H, W = scores.shape
    dev = scores.device
    if noisy is None:
        noisy = torch.empty((B, 3, H, W), dtype=torch.float32, device=dev)
    if out is None:
        out = torch.empty((B, 3, H, W), dtype=torch.float32, device=dev)
    small = (B * H * W <= (1 << 20) and bank.dim() == 5 and bank.shape[1] == 2 and W % 4 == 0 and B <= 8
             and all(z.dtype == torch.float32 for z in logits) and ksize in (3, 5, 7))
    if small:
        _need(bank, "bank", dev, torch.float32)
        _need(demod, "demod", dev, torch.float32)
        L = len(logits)
        shapes = level_shapes(H, W, L)
        for l, (z, (h, w)) in enumerate(zip(logits, shapes)):
            _need(z, f"logits[{l}]", dev, torch.float32)
            if tuple(z.shape) != (B, logit_channels(l, L, ksize), h, w):
                raise ValueError(f"logits[{l}] must be {(B, logit_channels(l, L, ksize), h, w)}")
        if tuple(bank.shape) != (B, 2, 3, H, W) or tuple(demod.shape) != (B, 3, H, W):
            raise ValueError("bank must be (B, 2, 3, H, W) and demod (B, 3, H, W)")
        if workspace is None:
            wb = C.c_size_t()
            check(lib.ssb_infer_small_workspace_bytes(B, H, W, L, C.byref(wb)), "ssb_infer_small_workspace_bytes")
            workspace = torch.empty(wb.value, dtype=torch.uint8, device=dev)
        d = _lib.PlaceDesc(B, H, W, 2, _lib.VARIANTS["stochastic"], 0, seed & (2**64 - 1), frame0, float(budget))
        lp = (C.c_void_p * L)(*[z.data_ptr() for z in logits])
        with torch.cuda.device(dev):
            rc = lib.ssb_infer_small(C.byref(d), _ptr(scores), _ptr(bank), _ptr(demod), L, ksize, lp, _ptr(noisy),
                                     _ptr(out), _ptr(workspace), _stream(dev))
        if rc == 0:
            return out, noisy
        if rc != _lib.SSB_EUNSUPPORTED:
            check(rc, "ssb_infer_small")
    place_fused(scores, bank, budget, seed=seed, frame0=frame0, noisy=noisy)
    pyramid_forward(noisy, logits, demod, ksize=ksize, out=out)
    return out, noisy


# ---------------------------------------------------------------------------
# temporal path: images.py warp_array / warp_backward


def _img_dtype(t, name):
    if t.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"{name} must be float32 or float64")
    return _DT[t.dtype]


def warp(prev, motion, want_validity=True):
    """Bilinear backward warp (ref `warp_array`, images.py:88-119).
    prev (B, C, H, W), motion (B, 2, H, W) = (mx, my), same dtype ->
    (out (B, C, H, W), validity (B, H, W) or None)."""
    lib = _lib.load()
    _need(prev, "prev")
    _need(motion, "motion", prev.device, prev.dtype)
    dt = _img_dtype(prev, "prev")
    if prev.dim() != 4 or motion.dim() != 4 or motion.shape[1] != 2 or \
            prev.shape[0] != motion.shape[0] or prev.shape[2:] != motion.shape[2:]:
        raise ValueError("warp: image and motion dimensions must match")
    B, Cc, H, W = prev.shape
    out = torch.empty_like(prev)
    val = torch.empty((B, H, W), dtype=prev.dtype, device=prev.device) if want_validity else None
    with torch.cuda.device(prev.device):
        check(lib.ssb_warp(dt, B, Cc, H, W, _ptr(prev), _ptr(motion), _ptr(out), _ptr(val),
                           _stream(prev.device)), "ssb_warp")
    return out, val


def warp_backward(grad_out, motion):
    """Transpose of `warp` w.r.t. prev (ref `warp_backward`, images.py:122-147):
    a deterministic gather in the reference's summation order."""
    lib = _lib.load()
    _need(grad_out, "grad_out")
    _need(motion, "motion", grad_out.device, grad_out.dtype)
    dt = _img_dtype(grad_out, "grad_out")
    if grad_out.dim() != 4 or motion.dim() != 4 or motion.shape[1] != 2 or \
            grad_out.shape[0] != motion.shape[0] or grad_out.shape[2:] != motion.shape[2:]:
        raise ValueError("warp: image and motion dimensions must match")
    B, Cc, H, W = grad_out.shape
    wb = C.c_size_t()
    check(lib.ssb_warp_backward_workspace_bytes(B, H, W, C.byref(wb)), "ssb_warp_backward_workspace_bytes")
    ws = torch.empty(wb.value, dtype=torch.uint8, device=grad_out.device)
    gp = torch.empty_like(grad_out)
    with torch.cuda.device(grad_out.device):
        check(lib.ssb_warp_backward(dt, B, Cc, H, W, _ptr(grad_out), _ptr(motion), _ptr(gp), _ptr(ws),
                                    _stream(grad_out.device)), "ssb_warp_backward")
    return gp


# ---------------------------------------------------------------------------
# estimator backward to the density scores


def score_grad(scores, g_input, grad_density, budget: float, sigma: float = 1.5):
    """Gradient of the loss w.r.t. the density scores (optimize.py:244-251):
    scores (B, H, W); g_input / grad_density (B, F, C, H, W) -- per frame the
    filter's input gradient and the estimator's d(noisy)/d(spp).  Returns
    g_scores (B, H, W), same dtype (float64 arithmetic inside)."""
    lib = _lib.load()
    _need(scores, "scores")
    dt = _img_dtype(scores, "scores")
    _need(g_input, "g_input", scores.device, scores.dtype)
    _need(grad_density, "grad_density", scores.device, scores.dtype)
    if scores.dim() == 2:
        scores = scores[None]
    if g_input.dim() == 4:
        g_input, grad_density = g_input[None], grad_density[None]
    B, H, W = scores.shape
    if g_input.dim() != 5 or g_input.shape != grad_density.shape or g_input.shape[0] != B or \
            tuple(g_input.shape[3:]) != (H, W):
        raise ValueError("score_grad: g_input / grad_density must be (B, F, C, H, W) matching scores")
    if not budget > 0:
        raise ValueError("budget must be positive")
    F, Cc = g_input.shape[1], g_input.shape[2]
    wb = C.c_size_t()
    check(lib.ssb_score_grad_workspace_bytes(B, H, W, C.byref(wb)), "ssb_score_grad_workspace_bytes")
    ws = torch.empty(wb.value, dtype=torch.uint8, device=scores.device)
    out = torch.empty_like(scores)
    with torch.cuda.device(scores.device):
        check(lib.ssb_score_grad(dt, B, F, Cc, H, W, _ptr(g_input), _ptr(grad_density), _ptr(scores),
                                 float(budget), float(sigma), _ptr(out), _ptr(ws),
                                 _stream(scores.device)), "ssb_score_grad")
    return out


# ---------------------------------------------------------------------------
# tonemap + loss epilogue


def _tmo(tmo):
    vals = [float(v) for v in tmo]
    if len(vals) != 5:
        raise ValueError("tmo must be (exposure, contrast, saturation, toe, shoulder)")
    return (C.c_double * 5)(*vals)  # passed by reference (ctypes array -> double*)


def tonemap(radiance, tmo):
    """Filmic tonemap (ref `tonemap_array`, tonemap.py:87-88): radiance
    (B, 3, H, W) -> LDR (B, 3, H, W); tmo = (exposure, contrast, saturation,
    toe, shoulder)."""
    lib = _lib.load()
    _need(radiance, "radiance")
    dt = _img_dtype(radiance, "radiance")
    if radiance.dim() != 4 or radiance.shape[1] != 3:
        raise ValueError("radiance must be (B, 3, H, W)")
    B, _, H, W = radiance.shape
    out = torch.empty_like(radiance)
    with torch.cuda.device(radiance.device):
        check(lib.ssb_tonemap(dt, B, H, W, _tmo(tmo), _ptr(radiance), _ptr(out), _stream(radiance.device)),
              "ssb_tonemap")
    return out


def tonemap_backward(radiance, tmo, upstream):
    """d(tonemap)/d(radiance) applied to `upstream` (ref `tonemap_backward`,
    tonemap.py:95-118)."""
    lib = _lib.load()
    _need(radiance, "radiance")
    dt = _img_dtype(radiance, "radiance")
    _need(upstream, "upstream", radiance.device, radiance.dtype)
    if radiance.dim() != 4 or radiance.shape[1] != 3 or upstream.shape != radiance.shape:
        raise ValueError("radiance / upstream must be (B, 3, H, W)")
    B, _, H, W = radiance.shape
    g = torch.empty_like(radiance)
    with torch.cuda.device(radiance.device):
        check(lib.ssb_tonemap_backward(dt, B, H, W, _tmo(tmo), _ptr(radiance), _ptr(upstream), _ptr(g),
                                       _stream(radiance.device)), "ssb_tonemap_backward")
    return g


def _loss_inputs(img, ref, ldr0_w, ref_w, validity, mask, name):
    """Shared checks of `losses` / `loss_epilogue` (the reference's
    ValueErrors, losses.py:58-91)."""
    _need(img, name)
    dt = _img_dtype(img, name)
    dev = img.device
    _need(ref, "ref", dev, img.dtype)
    if img.dim() != 4 or img.shape[1] != 3 or ref.shape != img.shape:
        raise ValueError("loss: image dimensions must match")
    if (ldr0_w is None) != (ref_w is None):
        raise ValueError("loss: the warped history needs both ldr0_w and ref_w")
    B, _, H, W = img.shape
    for t, nm in ((ldr0_w, "ldr0_w"), (ref_w, "ref_w")):
        if t is not None:
            _need(t, nm, dev, img.dtype)
            if t.shape != img.shape:
                raise ValueError("temporal loss: image dimensions must match")
    for t, nm in ((validity, "validity"), (mask, "mask")):
        if t is not None:
            _need(t, nm, dev, img.dtype)
            if tuple(t.shape) != (B, H, W):
                raise ValueError(f"{nm} must be (B, H, W)")
    if validity is not None and ldr0_w is None:
        raise ValueError("validity needs the warped history")
    return dt, dev, B, H, W


def loss_epilogue(radiance, ref, tmo, ldr0_w=None, ref_w=None, validity=None, mask=None, want_ldr=False,
                  want_losses=True):
    """The evaluate_step epilogue in one kernel (optimize.py:219-231 over
    tonemap.py / losses.py): tonemap(radiance), the spatial / temporal /
    combined losses against `ref` (and the warped history), and the gradient
    of the combined loss chained through the tonemap to the radiance.  Equals
    tonemap -> losses(want_grads=True) -> tonemap_backward (float64:
    bit-identical).  Returns a dict: 'grad_radiance', 'g_ldr0_w' (with a
    history), 'losses' (B, 3) float64, 'ldr' (want_ldr)."""
    lib = _lib.load()
    dt, dev, B, H, W = _loss_inputs(radiance, ref, ldr0_w, ref_w, validity, mask, "radiance")
    grad = torch.empty_like(radiance)
    g0 = torch.empty_like(radiance) if ldr0_w is not None else None
    ldr = torch.empty_like(radiance) if want_ldr else None
    vals = torch.empty((B, 3), dtype=torch.float64, device=dev) if want_losses else None
    wb = C.c_size_t()
    check(lib.ssb_losses_workspace_bytes(B, C.byref(wb)), "ssb_losses_workspace_bytes")
    ws = torch.empty(wb.value, dtype=torch.uint8, device=dev)
    t = _tmo(tmo)
    with torch.cuda.device(dev):
        check(lib.ssb_epilogue(dt, B, H, W, t, _ptr(radiance), _ptr(ref), _ptr(ldr0_w), _ptr(ref_w),
                               _ptr(validity), _ptr(mask), _ptr(ldr), _ptr(vals), _ptr(grad), _ptr(g0), _ptr(ws),
                               _stream(dev)), "ssb_epilogue")
    return {"grad_radiance": grad, "g_ldr0_w": g0, "losses": vals, "ldr": ldr}


def losses(ldr1, ref, ldr0_w=None, ref_w=None, validity=None, mask=None, want_maps=True,
           want_grads=False):
    """Masked spatial, temporal and max-combined losses (losses.py:58-91) and,
    with want_grads, their gradients w.r.t. ldr1 and the warped history as
    optimize.evaluate_step forms them (optimize.py:219-231).  Images
    (B, 3, H, W); validity / mask (B, H, W).  Returns a dict with 'losses'
    (B, 3) float64 = (spatial, temporal, combined), the maps, 'g_ldr1',
    'g_ldr0_w'."""
    lib = _lib.load()
    dt, dev, B, H, W = _loss_inputs(ldr1, ref, ldr0_w, ref_w, validity, mask, "ldr1")
    maps = [torch.empty((B, H, W), dtype=ldr1.dtype, device=dev) for _ in range(3)] if want_maps else [None] * 3
    vals = torch.empty((B, 3), dtype=torch.float64, device=dev)
    g1 = torch.empty_like(ldr1) if want_grads else None
    g0 = torch.empty_like(ldr1) if (want_grads and ldr0_w is not None) else None
    wb = C.c_size_t()
    check(lib.ssb_losses_workspace_bytes(B, C.byref(wb)), "ssb_losses_workspace_bytes")
    ws = torch.empty(wb.value, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        check(lib.ssb_losses(dt, B, H, W, _ptr(ldr1), _ptr(ref), _ptr(ldr0_w), _ptr(ref_w), _ptr(validity),
                             _ptr(mask), _ptr(maps[0]), _ptr(maps[1]), _ptr(maps[2]), _ptr(vals), _ptr(g1),
                             _ptr(g0), _ptr(ws), _stream(dev)), "ssb_losses")
    return {"losses": vals, "spatial_map": maps[0], "temporal_map": maps[1], "combined_map": maps[2],
            "g_ldr1": g1, "g_ldr0_w": g0}
