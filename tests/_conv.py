"""Layout conversion between the reference's HWC float64 arrays and the device
planar (B, C, H, W) tensors used by the CUDA path (test helper)."""
import numpy as np
import torch


def hwc_to_planar(a, dtype=torch.float64, device="cuda"):
    a = np.asarray(a)
    return torch.from_numpy(np.ascontiguousarray(a.transpose(2, 0, 1))[None]).to(device=device, dtype=dtype)


def planar_to_hwc(t):
    return t[0].permute(1, 2, 0).double().cpu().numpy()


def ref_logits_to_device(logits, k, temporal, dtype=torch.float64, device="cuda"):
    """Reference level-0 logits carry the temporal group; drop it when unread."""
    out = []
    L = len(logits)
    for l, z in enumerate(logits):
        if l == 0 and not temporal:
            z = z[:, :, :k * k + (4 if L > 1 else 0)]
        out.append(hwc_to_planar(z, dtype, device))
    return out


def device_glogits_to_ref(glogits, ref_logits, k, temporal):
    out = []
    for l, (g, z) in enumerate(zip(glogits, ref_logits)):
        a = planar_to_hwc(g)
        if a.shape[2] != z.shape[2]:
            full = np.zeros(z.shape)
            full[:, :, :a.shape[2]] = a
            a = full
        out.append(a)
    return out


def assert_close(got, ref, rtol, name="", atol_frac=None):
    """Per-tensor comparator: elementwise rtol with an
    atol floor of atol_frac * max|ref| taken over THIS tensor only, plus a
    relative-L2 bound ||got - ref|| / ||ref|| <= rtol."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    atol = (rtol if atol_frac is None else atol_frac) * max(np.abs(ref).max(initial=0.0), 1e-300)
    np.testing.assert_allclose(got, ref, rtol=rtol, atol=atol, err_msg=name)
    nref = float(np.sqrt(np.sum(ref * ref)))
    if nref > 0.0:
        rel = float(np.sqrt(np.sum((got - ref) ** 2))) / nref
        assert rel <= rtol, f"{name}: relative L2 error {rel:.3e} > {rtol:g}"


def assert_levels_close(got_levels, ref_levels, rtol, name="g_logits", scales=None):
    """Per-level logit-gradient parity: every level is its own tensor, so the
    atol floor is rtol * max|ref_l| of that level (coarse-level gradients are
    orders of magnitude below level 0's and would be unchecked by a floor
    taken over all levels), plus the per-level relative-L2 bound.

    scales (oracle `Grads.operand_scale`): per level, the magnitude of the two
    softmax-backward operands w*gw and w*sum(w gw) whose DIFFERENCE the logit
    gradient is.  Any float implementation errs by ~eps times that, so the
    floor is rtol * max(max|ref_l|, scale_l).  On ordinary levels scale_l is
    1-3x max|ref_l| (the floor is unchanged to that factor); it only matters on
    levels whose gradient cancels analytically -- a 1x1 coarse level, where
    all k*k taps read the same clamped pixel and the reference's own values
    are rounding noise ~1e-16 x scale_l.  The relative-L2 bound uses the same
    floor as its absolute term."""
    assert len(got_levels) == len(ref_levels)
    for l, (g, r) in enumerate(zip(got_levels, ref_levels)):
        g = np.asarray(g, dtype=np.float64)
        r = np.asarray(r, dtype=np.float64)
        m = float(np.abs(r).max(initial=0.0))
        if scales is None or scales[l] <= m:
            assert_close(g, r, rtol, f"{name}{l}")
            continue
        atol = rtol * scales[l]
        np.testing.assert_allclose(g, r, rtol=rtol, atol=atol, err_msg=f"{name}{l}")
        err = float(np.sqrt(np.sum((g - r) ** 2)))
        assert err <= rtol * float(np.sqrt(np.sum(r * r))) + atol * np.sqrt(r.size), \
            f"{name}{l}: L2 error {err:.3e} (operand scale {scales[l]:.3e})"
