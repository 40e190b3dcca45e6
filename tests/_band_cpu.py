"""CPU compute back end of the row-band protocol (test-only): the oracle's
own per-level arithmetic (oracle/pyramid.py forward: pool2, joint softmax,
clamp-padded k x k gather, clamped upsample, demod/remod) on torch CPU
float64 tensors (B, C, H, W), so a banded CPU run can be compared bit for bit
with oracle.forward on the full frame."""
import numpy as np
import torch

from oracle import pyramid as op


def _hwc(t):
    return t.permute(1, 2, 0).numpy()


def _put(dst, a):
    dst.copy_(torch.from_numpy(np.ascontiguousarray(a.transpose(2, 0, 1))))


class OracleCompute:
    def __init__(self, ksize):
        self.k = ksize

    @staticmethod
    def pool2(x):
        """Count-correct 2x2 mean (oracle.pool2's math) with a fixed per-pixel
        summation order ((v00 + v01) + v10) + v11: numpy's multi-axis sum in
        oracle.pool2 may pick its order from the array's size, which a band
        crop changes."""
        h, w = x.shape[:2]
        hc, wc = (h + 1) // 2, (w + 1) // 2
        p = np.zeros((2 * hc, 2 * wc) + x.shape[2:])
        p[:h, :w] = x
        occ = np.zeros((2 * hc, 2 * wc, 1))
        occ[:h, :w] = 1.0
        s = ((p[0::2, 0::2] + p[0::2, 1::2]) + p[1::2, 0::2]) + p[1::2, 1::2]
        c = ((occ[0::2, 0::2] + occ[0::2, 1::2]) + occ[1::2, 0::2]) + occ[1::2, 1::2]
        return s / c

    def pool(self, src, dst, demod=None):
        for b in range(src.shape[0]):
            x = _hwc(src[b])
            if demod is not None:
                x = x / np.maximum(_hwc(demod[b]), op.DEMOD_FLOOR)
            _put(dst[b], self.pool2(x))

    def forward_level(self, img, logits, demod, parent, out):
        k, taps = self.k, self.k * self.k
        for b in range(img.shape[0]):
            x = _hwc(img[b])
            if demod is not None:
                dcl = np.maximum(_hwc(demod[b]), op.DEMOD_FLOOR)
                x = x / dcl
            w = op.softmax_channels(_hwc(logits[b]))
            o = op.gather(x, w[:, :, :taps], k)
            if parent is not None:
                o = o + op.upsample(_hwc(parent[b]), w[:, :, taps:taps + op.UPSAMPLE_TAPS])
            if demod is not None:
                o = o * dcl
            _put(out[b], o)
