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
    """rtol with an atol floor of atol_frac * max|ref|."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    atol = (rtol if atol_frac is None else atol_frac) * max(np.abs(ref).max(initial=0.0), 1e-300)
    np.testing.assert_allclose(got, ref, rtol=rtol, atol=atol, err_msg=name)
