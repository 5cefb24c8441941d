"""Host check of the pixel-pair tap decomposition conv_span_px2 runs on the tensor cores
(paper_2601_04250_b200/csrc/gg_conv_span.cu): a TMEM lane holds the pixel pair
(2(q+i), 2(q+i)+1) of window origins; kernel row r's operand j = e + s is the pair row
q + i + ((r*Wp + j) >> 1), K half (r*Wp + j) & 1, multiplied with rows [off_j, off_j + N_j)
of the stacked slab [W(r,2); W(r,1); W(r,0)] into columns [col_j, col_j + N_j).  Replaying
exactly those index computations in numpy must give the 3x3 convolution on the
shared-border layout (odd pixel counts included) — no GPU needed."""

from __future__ import annotations

import numpy as np
import pytest

# (stack row offset, N, accumulator column) per j, as issued by the kernel
J_OPS = {0: (128, 64, 0), 1: (64, 128, 0), 2: (0, 128, 0), 3: (0, 64, 64)}


def shared_layout(x):
    """[n, s, s, c] -> flat shared-border buffer: (s+2) zero margin + n x (s+1)^2."""
    n, s, _, c = x.shape
    img = np.zeros((n, s + 1, s + 1, c), x.dtype)
    img[:, :s, :s] = x
    return np.concatenate([np.zeros((s + 2, c), x.dtype), img.reshape(-1, c)])


def px2_conv(xbuf, w, n, s):
    """Emulate conv_span_px2 on the flat shared-border buffer (margin included)."""
    c = w.shape[1]
    Wp = s + 1
    img = Wp * Wp
    mtot = n * img
    prows = (mtot + 1) // 2
    xp = np.zeros((prows + Wp + 130, 2, c), np.float64)     # pair rows, K halves; OOB rows zero
    flat = xbuf[: 2 * prows] if xbuf.shape[0] >= 2 * prows else np.pad(xbuf, ((0, 2 * prows - xbuf.shape[0]), (0, 0)))
    xp[:prows] = flat.reshape(prows, 2, c)
    # stacked slabs per kernel row: [W(r,2); W(r,1); W(r,0)], rows = output channels
    stack = [np.concatenate([w[:, :, r, 2], w[:, :, r, 1], w[:, :, r, 0]]) for r in range(3)]
    out = np.zeros((2 * prows + Wp + 1, c), np.float64)
    for q in range(0, prows, 128):
        lanes = np.arange(128)
        acc = np.zeros((128, 128))
        for r in range(3):
            for j in (1, 0, 2, 3):
                v = r * Wp + j
                a = xp[q + lanes + (v >> 1), v & 1]              # [128, c]
                off, nn, col = J_OPS[j]
                b = stack[r][off: off + nn]                       # [nn, c]
                acc[:, col: col + nn] += a @ b.T
        for e in range(2):
            m = 2 * (q + lanes) + e
            keep = m < mtot
            h, wcol = (m % img) // Wp, (m % img) % Wp
            real = keep & (h < s) & (wcol < s)
            o = acc[:, e * 64: e * 64 + 64] * real[:, None]
            dst = m + Wp + 1
            out[dst[keep]] = o[keep]
    return out


@pytest.mark.parametrize("n,s", [(2, 7), (3, 5), (1, 9)])
def test_px2_decomposition_matches_conv(n, s):
    rng = np.random.default_rng(n * 10 + s)
    c = 64
    x = rng.standard_normal((n, s, s, c))
    w = rng.standard_normal((c, c, 3, 3)) / 24.0
    xbuf = shared_layout(x)
    got = px2_conv(xbuf, w, n, s)
    # reference: zero-padded direct 3x3 convolution, placed in the same layout
    xpad = np.zeros((n, s + 2, s + 2, c))
    xpad[:, 1:-1, 1:-1] = x
    ref = np.zeros((n, s, s, c))
    for r in range(3):
        for t in range(3):
            ref += np.einsum("nhwc,oc->nhwo", xpad[:, r:r + s, t:t + s], w[:, :, r, t])
    want = shared_layout(ref)
    assert np.allclose(got[: want.shape[0]], want, atol=1e-9)
    assert not got[want.shape[0]:].any()
