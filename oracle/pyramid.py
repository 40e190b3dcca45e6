"""Gather-pyramid filter, forward and exact backward -- CPU oracle (test-only).

Restates the reference's Appendix-A pyramid (`pkg/src/sparse_sampler/pyramid.py`)
with the kernel radius r and the level count L as parameters instead of the
reference's hard-coded 5x5 taps and LEVELS = 5.  Arithmetic order follows the
reference exactly so that k = 5 reproduces it bit-for-bit in float64:

* joint per-pixel softmax, max-subtracted (`pyramid.py:93-120`)
* iterated count-correct 2x2 box pooling (`pyramid.py:127-156`)
* k x k clamp-to-edge gather, taps accumulated dy-major from zeros
  (`pyramid.py:30,173-195`)
* learned 2x2 upsample with clamped parent indices (`pyramid.py:216-260`)
* coarse-to-fine reconstruction + demod/remod (`pyramid.py:292-345`)
* two-sweep exact backward with the clamp "fold" (`pyramid.py:362-455`)

Arrays are the reference's HWC float64 layout.  Level-l logits carry
``channel_count(l)`` channels: k*k denoise taps, then 4 upsample taps (levels
with a coarser neighbour), then k*k temporal taps (level 0 only).  With
``blend="tied"`` the 4 upsample logits are replaced by a single blend logit
that is broadcast to the 4 taps (its gradient is the sum of the four).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

UPSAMPLE_TAPS = 4
DEMOD_FLOOR = 1e-3


# ---------------------------------------------------------------------------
# geometry


def tap_offsets(k: int) -> list[tuple[int, int]]:
    """Tap order of a k x k footprint: dy-major, dx-minor (ref pyramid.py:30)."""
    r = k // 2
    return [(dy, dx) for dy in range(-r, r + 1) for dx in range(-r, r + 1)]


def level_shapes(height: int, width: int, levels: int) -> list[tuple[int, int]]:
    """(H_l, W_l) per level, halving with ceil (ref pyramid.py:33-38)."""
    shapes = [(height, width)]
    while len(shapes) < levels:
        h, w = shapes[-1]
        shapes.append(((h + 1) // 2, (w + 1) // 2))
    return shapes


def channel_count(level: int, levels: int, k: int, temporal: bool = True,
                  blend: str = "native") -> int:
    """Logit channels at `level` (ref pyramid.py:41-46 generalised)."""
    taps = k * k
    n = taps
    if level < levels - 1:
        n += UPSAMPLE_TAPS if blend == "native" else 1
    if level == 0 and temporal:
        n += taps
    return n


def infer_geometry(logits: list[np.ndarray]) -> tuple[int, int]:
    """(levels, k) from a reference-layout kernel field."""
    levels = len(logits)
    k = int(round(np.sqrt(logits[-1].shape[-1])))
    if k * k != logits[-1].shape[-1] or k % 2 == 0:
        raise ValueError("coarsest level must carry k*k logits with k odd")
    return levels, k


# ---------------------------------------------------------------------------
# per-pixel softmax


def softmax_channels(x: np.ndarray) -> np.ndarray:
    m = x.max(axis=-1, keepdims=True)
    e = np.exp(x - m)
    return e / e.sum(axis=-1, keepdims=True)


def softmax_channels_backward(w: np.ndarray, gw: np.ndarray) -> np.ndarray:
    dot = (w * gw).sum(axis=-1, keepdims=True)
    return w * (gw - dot)


def expand_blend(logits: list[np.ndarray], k: int) -> list[np.ndarray]:
    """Tied blend mode -> native layout: broadcast the blend logit to 4 taps."""
    taps = k * k
    out = []
    for l, arr in enumerate(logits):
        if l < len(logits) - 1:
            b = arr[:, :, taps:taps + 1]
            arr = np.concatenate([arr[:, :, :taps], np.repeat(b, 4, axis=2),
                                  arr[:, :, taps + 1:]], axis=2)
        out.append(arr)
    return out


def collapse_blend_grads(glogits: list[np.ndarray], k: int) -> list[np.ndarray]:
    taps = k * k
    out = []
    for l, g in enumerate(glogits):
        if l < len(glogits) - 1:
            up = g[:, :, taps:taps + 4]
            gb = ((up[:, :, 0] + up[:, :, 1]) + up[:, :, 2]) + up[:, :, 3]
            g = np.concatenate([g[:, :, :taps], gb[:, :, None], g[:, :, taps + 4:]], axis=2)
        out.append(g)
    return out


def kernel_weights(logits: list[np.ndarray], k: int, temporal: bool) -> list[np.ndarray]:
    """Joint softmax per level; without history the level-0 temporal group is
    excluded and its weights are exactly zero (ref pyramid.py:93-109)."""
    active0 = k * k + (UPSAMPLE_TAPS if len(logits) > 1 else 0)
    weights = []
    for l, z in enumerate(logits):
        if l == 0 and not temporal and z.shape[-1] > active0:
            w = np.zeros_like(z)
            w[:, :, :active0] = softmax_channels(z[:, :, :active0])
        else:
            w = softmax_channels(z)
        weights.append(w)
    return weights


# ---------------------------------------------------------------------------
# pooling


def pool2(img: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Count-correct 2x2 mean; returns (coarse, counts) (ref pyramid.py:140-149)."""
    h, w = img.shape[:2]
    hc, wc = (h + 1) // 2, (w + 1) // 2
    tail = img.shape[2:]
    padded = np.zeros((2 * hc, 2 * wc) + tail)
    padded[:h, :w] = img
    blocks = padded.reshape(hc, 2, wc, 2, -1).sum(axis=(1, 3)).reshape((hc, wc) + tail)
    occupied = np.zeros((2 * hc, 2 * wc, 1))
    occupied[:h, :w] = 1.0
    counts = occupied.reshape(hc, 2, wc, 2, 1).sum(axis=(1, 3)).reshape(hc, wc, 1)
    return blocks / counts, counts


def pool2_adjoint(g: np.ndarray, counts: np.ndarray, fine_hw) -> np.ndarray:
    h, w = fine_hw[:2]
    spread = g / counts
    return np.repeat(np.repeat(spread, 2, axis=0), 2, axis=1)[:h, :w]


def pyramid_levels(img: np.ndarray, levels: int):
    lv = [img]
    counts = []
    for _ in range(levels - 1):
        c, n = pool2(lv[-1])
        lv.append(c)
        counts.append(n)
    return lv, counts


# ---------------------------------------------------------------------------
# k x k gather and its transposes


def edge_pad(img: np.ndarray, r: int) -> np.ndarray:
    return np.pad(img, ((r, r), (r, r), (0, 0)), mode="edge")


def gather_padded(padded: np.ndarray, w: np.ndarray, k: int) -> np.ndarray:
    r = k // 2
    h, wd = padded.shape[0] - 2 * r, padded.shape[1] - 2 * r
    acc = np.zeros((h, wd, padded.shape[2]))
    for t, (dy, dx) in enumerate(tap_offsets(k)):
        acc += w[:, :, t, None] * padded[r + dy:r + dy + h, r + dx:r + dx + wd]
    return acc


def gather(img: np.ndarray, w: np.ndarray, k: int) -> np.ndarray:
    """Per-pixel k x k gather, clamp-to-edge (ref `gather5`, pyramid.py:184-187)."""
    return gather_padded(edge_pad(img, k // 2), w, k)


def gather_weight_grad(gout: np.ndarray, padded: np.ndarray, k: int) -> np.ndarray:
    r = k // 2
    h, wd = gout.shape[:2]
    gw = np.empty((h, wd, k * k))
    for t, (dy, dx) in enumerate(tap_offsets(k)):
        gw[:, :, t] = (gout * padded[r + dy:r + dy + h, r + dx:r + dx + wd]).sum(axis=-1)
    return gw


def scatter_into_padded(gpad: np.ndarray, gout: np.ndarray, w: np.ndarray, k: int) -> None:
    """gpad += transpose of the padded gather (ref pyramid.py:452-455)."""
    r = k // 2
    h, wd = gout.shape[:2]
    for t, (dy, dx) in enumerate(tap_offsets(k)):
        gpad[r + dy:r + dy + h, r + dx:r + dx + wd] += w[:, :, t, None] * gout


def fold_edges(gpad: np.ndarray, r: int) -> np.ndarray:
    """Transpose of edge padding: the r outer rows/cols fold onto the edge
    pixel, outermost first (ref `_fold_pad2`, pyramid.py:206-213)."""
    def outer_sum(take):
        s = take(0)
        for i in range(1, r):
            s = s + take(i)
        return s

    gpad[:, r] += outer_sum(lambda i: gpad[:, i])
    gpad[:, -1 - r] += outer_sum(lambda i: gpad[:, -1 - i])
    core = gpad[:, r:gpad.shape[1] - r]
    core[r] += outer_sum(lambda i: core[i])
    core[-1 - r] += outer_sum(lambda i: core[-1 - i])
    return core[r:core.shape[0] - r].copy()


def gather_input_grad(gout: np.ndarray, w: np.ndarray, k: int) -> np.ndarray:
    r = k // 2
    h, wd, c = gout.shape
    gpad = np.zeros((h + 2 * r, wd + 2 * r, c))
    scatter_into_padded(gpad, gout, w, k)
    return fold_edges(gpad, r)


# ---------------------------------------------------------------------------
# learned 2x2 upsample


def parent_index(hf: int, wf: int, hc: int, wc: int):
    """Clamped parent indices per upsample tap (i, j) in
    (0,0),(0,1),(1,0),(1,1) order, i the row offset (ref pyramid.py:219-231)."""
    ys = np.arange(hf)
    xs = np.arange(wf)
    out = []
    for i in (0, 1):
        for j in (0, 1):
            iy = np.minimum((ys + i) // 2, hc - 1)
            ix = np.minimum((xs + j) // 2, wc - 1)
            out.append((iy[:, None], ix[None, :]))
    return out


def upsample(coarse: np.ndarray, w: np.ndarray) -> np.ndarray:
    hf, wf = w.shape[:2]
    hc, wc = coarse.shape[:2]
    acc = np.zeros((hf, wf, coarse.shape[2]))
    for t, (iy, ix) in enumerate(parent_index(hf, wf, hc, wc)):
        acc += w[:, :, t, None] * coarse[iy, ix]
    return acc


def upsample_weight_grad(gout: np.ndarray, coarse: np.ndarray) -> np.ndarray:
    hf, wf = gout.shape[:2]
    hc, wc = coarse.shape[:2]
    gw = np.empty((hf, wf, UPSAMPLE_TAPS))
    for t, (iy, ix) in enumerate(parent_index(hf, wf, hc, wc)):
        gw[:, :, t] = (gout * coarse[iy, ix]).sum(axis=-1)
    return gw


def upsample_coarse_grad(gout: np.ndarray, w: np.ndarray, coarse_hw) -> np.ndarray:
    hf, wf, c = gout.shape
    hc, wc = coarse_hw[:2]
    flat = np.zeros((hc * wc, c))
    for t, (iy, ix) in enumerate(parent_index(hf, wf, hc, wc)):
        np.add.at(flat, (iy * wc + ix).ravel(), (w[:, :, t, None] * gout).reshape(hf * wf, c))
    return flat.reshape(hc, wc, c)


# ---------------------------------------------------------------------------
# reconstruction


@dataclass
class Tape:
    k: int
    levels: int
    weights: list
    pads: list
    counts: list
    shapes: list
    lhat: dict
    temporal: bool
    prev_pad: np.ndarray | None
    prev_in: np.ndarray | None
    x0: np.ndarray
    out_pre: np.ndarray
    demod: np.ndarray | None
    dclamp: np.ndarray | None
    extra: dict = field(default_factory=dict)


@dataclass
class Grads:
    logits: list | None
    demod: np.ndarray | None
    input: np.ndarray
    prev: np.ndarray | None
    # per level: max |w * gw| and |w * sum(w gw)| -- the magnitude of the two
    # softmax-backward operands whose difference the logit gradient is (test
    # comparators use it as the cancellation-aware atol scale)
    operand_scale: list | None = None


def forward(noisy, logits, prev=None, demod=None, k: int | None = None,
            blend: str = "native"):
    """Coarse-to-fine reconstruction (ref `reconstruct_core`, pyramid.py:292-345).

    noisy (H, W, C) any C; logits: per-level (H_l, W_l, C_l) in the reference
    layout; returns (out, tape)."""
    noisy = np.asarray(noisy, dtype=np.float64)
    logits = [np.asarray(z, dtype=np.float64) for z in logits]
    if k is None:
        levels, k = infer_geometry(logits)
    levels = len(logits)
    if blend == "tied":
        logits = expand_blend(logits, k)
    taps = k * k
    r = k // 2
    temporal = prev is not None
    if demod is not None:
        dclamp = np.maximum(demod, DEMOD_FLOOR)
        x0 = noisy / dclamp
        prev_in = prev / dclamp if temporal else None
    else:
        dclamp = None
        x0 = noisy
        prev_in = prev
    w = kernel_weights(logits, k, temporal)
    lv, counts = pyramid_levels(x0, levels)
    pads = [edge_pad(a, r) for a in lv]
    lhat = {}
    top = levels - 1
    if top == 0:
        out = gather_padded(pads[0], w[0][:, :, :taps], k)
    else:
        lhat[top] = gather_padded(pads[top], w[top][:, :, :taps], k)
        for l in range(top - 1, 0, -1):
            lhat[l] = (gather_padded(pads[l], w[l][:, :, :taps], k)
                       + upsample(lhat[l + 1], w[l][:, :, taps:taps + UPSAMPLE_TAPS]))
        out = (gather_padded(pads[0], w[0][:, :, :taps], k)
               + upsample(lhat[1], w[0][:, :, taps:taps + UPSAMPLE_TAPS]))
    prev_pad = None
    if temporal:
        t0 = taps + (UPSAMPLE_TAPS if levels > 1 else 0)
        prev_pad = edge_pad(prev_in, r)
        out = out + gather_padded(prev_pad, w[0][:, :, t0:], k)
    out_pre = out
    if demod is not None:
        out = out * dclamp
    tape = Tape(k=k, levels=levels, weights=w, pads=pads, counts=counts,
                shapes=[a.shape for a in lv], lhat=lhat, temporal=temporal,
                prev_pad=prev_pad, prev_in=prev_in, x0=x0, out_pre=out_pre,
                demod=demod, dclamp=dclamp, extra={"blend": blend})
    return out, tape


def backward(tape: Tape, upstream, want_param_grads: bool = True) -> Grads:
    """Exact gradients of sum(upstream * out) (ref `reconstruct_backward`,
    pyramid.py:362-449)."""
    k, levels, w = tape.k, tape.levels, tape.weights
    taps = k * k
    r = k // 2
    upstream = np.asarray(upstream, dtype=np.float64)
    if tape.demod is not None:
        gout = upstream * tape.dclamp
        gdc = (upstream * tape.out_pre).copy()
    else:
        gout = upstream
        gdc = None
    gw = [np.zeros_like(a) for a in w] if want_param_grads else None
    gpads = [np.zeros_like(p) for p in tape.pads]
    gprev = None
    top = levels - 1
    t0 = taps + (UPSAMPLE_TAPS if levels > 1 else 0)

    # sweep 1, fine -> coarse
    g = gout
    for l in range(levels):
        wl = w[l]
        if want_param_grads:
            gw[l][:, :, :taps] = gather_weight_grad(g, tape.pads[l], k)
            if l < top:
                gw[l][:, :, taps:taps + UPSAMPLE_TAPS] = upsample_weight_grad(g, tape.lhat[l + 1])
        scatter_into_padded(gpads[l], g, wl[:, :, :taps], k)
        if l == 0 and tape.temporal:
            if want_param_grads:
                gw[0][:, :, t0:] = gather_weight_grad(gout, tape.prev_pad, k)
            gprev_pad = np.zeros_like(tape.prev_pad)
            scatter_into_padded(gprev_pad, gout, wl[:, :, t0:], k)
            gprev = fold_edges(gprev_pad, r)
        if l < top:
            g = upsample_coarse_grad(g, wl[:, :, taps:taps + UPSAMPLE_TAPS],
                                     tape.lhat[l + 1].shape)

    # sweep 2, coarse -> fine
    glevel = fold_edges(gpads[top], r)
    for l in range(top - 1, -1, -1):
        gl = pool2_adjoint(glevel, tape.counts[l], tape.shapes[l])
        gl += fold_edges(gpads[l], r)
        glevel = gl
    gx0 = glevel

    glogits = None
    if want_param_grads:
        glogits = []
        scales = []
        for l in range(levels):
            n = t0 if (l == 0 and not tape.temporal and w[0].shape[-1] > t0) else w[l].shape[-1]
            if n < w[l].shape[-1]:
                gz = np.zeros_like(gw[0])
                gz[:, :, :t0] = softmax_channels_backward(w[0][:, :, :t0], gw[0][:, :, :t0])
            else:
                gz = softmax_channels_backward(w[l], gw[l])
            glogits.append(gz)
            wg = w[l][:, :, :n] * gw[l][:, :, :n]
            dot = np.abs(wg.sum(axis=-1, keepdims=True)) * w[l][:, :, :n]
            scales.append(max(float(np.abs(wg).max(initial=0.0)), float(dot.max(initial=0.0))))
        if tape.extra.get("blend") == "tied":
            glogits = collapse_blend_grads(glogits, k)
            scales = [4.0 * x for x in scales]  # the blend gradient sums 4 taps

    gdemod = None
    if tape.demod is not None:
        gnoisy = gx0 / tape.dclamp
        gdc -= gx0 * tape.x0 / tape.dclamp
        if tape.temporal:
            gprev_full = gprev / tape.dclamp
            gdc -= gprev * tape.prev_in / tape.dclamp
            gprev = gprev_full
        if want_param_grads:
            gdemod = np.where(tape.demod > DEMOD_FLOOR, gdc, 0.0)
    else:
        gnoisy = gx0
    return Grads(logits=glogits, demod=gdemod, input=gnoisy, prev=gprev,
                 operand_scale=scales if want_param_grads else None)


# ---------------------------------------------------------------------------
# helpers for the test-suite and the CPU baseline


def random_logits(height: int, width: int, levels: int, k: int, rng,
                  temporal: bool = True, blend: str = "native", scale: float = 1.0):
    return [rng.normal(0.0, scale, (h, w, channel_count(l, levels, k, temporal, blend)))
            for l, (h, w) in enumerate(level_shapes(height, width, levels))]
