"""ResNet-18 (torchvision architecture, 224x224) forward on sm_100a, NHWC bf16.

Every convolution is one implicit-GEMM tcgen05 kernel (gg_conv2d) with the
eval-mode BatchNorm folded into its weights/bias and the residual add + ReLU
fused into the epilogue; the 1x1 stride-2 downsample is a conv of the same
kernel.  Stem/head: gg_nchw_to_nhwc (fp32 NCHW -> bf16 NHWC, channels padded
to 8), gg_maxpool3x3s2, gg_avgpool, and the fc layer on gg_gemm with fp32
logits for the K3 epilogue.
"""

from __future__ import annotations

import ctypes as C

from . import _native
from .distilbert import OUT_F32, gemm


def _fold(conv, bn, cpad: int):
    """BN(conv(x)) == conv'(x) + b' in eval mode; weights -> [Cout, Kpad] (r, s, c) order."""
    import torch

    w = conv.weight.detach().float()
    cout, cin, R, S = w.shape
    scale = bn.weight.detach().float() / torch.sqrt(bn.running_var.detach().float() + bn.eps)
    bias = bn.bias.detach().float() - bn.running_mean.detach().float() * scale
    w = w * scale[:, None, None, None]
    wp = torch.zeros((cout, R, S, cpad), dtype=torch.float32)
    wp[:, :, :, :cin] = w.permute(0, 2, 3, 1).cpu()
    k = R * S * cpad
    kpad = (k + 63) // 64 * 64
    out = torch.zeros((cout, kpad), dtype=torch.float32)
    out[:, :k] = wp.reshape(cout, k)
    return out, bias.cpu(), kpad


class _Conv:
    def __init__(self, conv, bn, cpad, device):
        import torch
        w, b, self.kpad = _fold(conv, bn, cpad)
        self.w = w.to(device=device, dtype=torch.bfloat16).contiguous()
        self.b = b.to(device=device).contiguous()
        self.cout = w.shape[0]
        self.cin = cpad
        self.r, self.s = conv.kernel_size
        self.stride = conv.stride[0]
        self.pad = self.pad_hi = conv.padding[0]
        self.algo_macs_per_pixel = self.r * self.s * conv.in_channels * self.cout

    def out_hw(self, h, w):
        return ((h + self.pad + self.pad_hi - self.r) // self.stride + 1,
                (w + self.pad + self.pad_hi - self.s) // self.stride + 1)

    def __call__(self, lib, x, n, h, w, y, st, residual=None, relu=True, count=None):
        _native.check("gg_conv2d", lib.gg_conv2d(
            C.c_void_p(x), n, h, w, self.cin, _native.ptr(self.w), self.cout, self.r, self.s,
            self.stride, self.pad, self.kpad, _native.ptr(self.b),
            None if residual is None else C.c_void_p(residual), int(relu), C.c_void_p(y),
            self.pad_hi, _native.ptr(count), st))
        return self.out_hw(h, w)

    def flops(self, n, h, w):
        """Algorithmic FLOPs of the original convolution (padding channels excluded)."""
        ho, wo = self.out_hw(h, w)
        return 2.0 * n * ho * wo * self.algo_macs_per_pixel


class _StemConv(_Conv):
    """conv1 (7x7 / 2, pad 3, 3 -> 64) + bn1 as a 4x4 / 1 conv over the
    space-to-depth(2) input (16 channels: (dy, dx, c) of each 2x2 cell, 12 real).

    Output (ho, wo) reads input rows 2ho - 3 + r, r = 0..6; with r = 2i + dy - 1
    that is s2d row ho - 2 + i (i = 0..3) and sub-row dy, so
    w'[co, i, j, (dy*2+dx)*3 + c] = w[co, c, 2i+dy-1, 2j+dx-1] (0 outside 0..6),
    padding 2 before and 1 after.  K = 4*4*16 = 256 instead of 7*7*8 = 392(448).
    """

    def __init__(self, conv, bn, device):
        import torch
        w = conv.weight.detach().float().cpu()
        scale = bn.weight.detach().float() / torch.sqrt(bn.running_var.detach().float() + bn.eps)
        bias = bn.bias.detach().float() - bn.running_mean.detach().float() * scale
        w = w * scale.cpu()[:, None, None, None]
        cout = w.shape[0]
        wp = torch.zeros((cout, 4, 4, 16), dtype=torch.float32)
        for i in range(4):
            for dy in range(2):
                r = 2 * i + dy - 1
                if not 0 <= r <= 6:
                    continue
                for j in range(4):
                    for dx in range(2):
                        s = 2 * j + dx - 1
                        if not 0 <= s <= 6:
                            continue
                        for c in range(3):
                            wp[:, i, j, (dy * 2 + dx) * 3 + c] = w[:, c, r, s]
        self.w = wp.reshape(cout, 256).to(device=device, dtype=torch.bfloat16).contiguous()
        self.b = bias.to(device=device).contiguous()
        self.kpad, self.cout, self.cin = 256, cout, 16
        self.r = self.s = 4
        self.stride, self.pad, self.pad_hi = 1, 2, 1
        self.algo_macs_per_pixel = 7 * 7 * 3 * cout


class ResNet18B200:
    """Packed (BN-folded) weights + NHWC activation buffers for up to max_batch images."""

    def __init__(self, tv_model, max_batch: int = 64, image: int = 224, device="cuda"):
        torch = _native.require_cuda()
        self.lib = _native.load()
        self.device = torch.device(device)
        self.max_batch, self.image = max_batch, image
        m = tv_model.eval()
        self.stem = _StemConv(m.conv1, m.bn1, self.device)
        self.blocks = []
        cin = 64
        for layer in (m.layer1, m.layer2, m.layer3, m.layer4):
            for blk in layer:
                cout = blk.conv1.out_channels
                ds = None
                if blk.downsample is not None:
                    ds = _Conv(blk.downsample[0], blk.downsample[1], cin, self.device)
                self.blocks.append((_Conv(blk.conv1, blk.bn1, cin, self.device),
                                    _Conv(blk.conv2, blk.bn2, cout, self.device), ds))
                cin = cout
        self.num_classes = m.fc.out_features
        npad = (self.num_classes + 31) // 32 * 32
        wfc = torch.zeros((npad, m.fc.in_features), dtype=torch.float32)
        wfc[: self.num_classes] = m.fc.weight.detach().float().cpu()
        bfc = torch.zeros(npad, dtype=torch.float32)
        bfc[: self.num_classes] = m.fc.bias.detach().float().cpu()
        self.w_fc = wfc.to(self.device, torch.bfloat16).contiguous()
        self.b_fc = bfc.to(self.device).contiguous()
        B, H = max_batch, image
        z = dict(dtype=torch.bfloat16, device=self.device)
        self.x16 = torch.empty(B * (H // 2) * (H // 2) * 16, **z)   # space-to-depth stem input
        big = B * (H // 2) * (H // 2) * 64
        self.buf = [torch.empty(big, **z) for _ in range(3)]
        self.pooled = torch.empty((B, 512), **z)
        self.logits = torch.empty((B, npad), dtype=torch.float32, device=self.device)

    def flops(self, batch: int) -> float:
        """Algorithmic FLOPs (3.628 GF/img at 224x224)."""
        n, h = batch, self.image
        f = self.stem.flops(n, h // 2, h // 2)   # the stem runs on the s2d(2) input
        h = h // 4
        for c1, c2, ds in self.blocks:
            f += c1.flops(n, h, h)
            h2, _ = c1.out_hw(h, h)
            f += c2.flops(n, h2, h2)
            if ds is not None:
                f += ds.flops(n, h, h)
            h = h2
        f += 2.0 * n * 512 * self.num_classes
        return f

    def forward(self, images, batch: int | None = None, stream=None):
        """images: CUDA fp32 NCHW [B, 3, 224, 224].  Returns fp32 logits [B, 1000] (view)."""
        B = int(images.shape[0]) if batch is None else int(batch)
        assert B <= self.max_batch
        H = self.image
        st = _native.stream_ptr(stream)
        _native.check("gg_nchw_to_s2d16", self.lib.gg_nchw_to_s2d16(
            _native.ptr(images), B, H, H, _native.ptr(self.x16), st))
        return self.forward_s2d(B, stream=stream)

    def forward_s2d(self, B: int, stream=None, count=None):
        """Forward from self.x16 (bf16 space-to-depth(2) NHWC, 16 channels).
        count: optional CUDA int32 [1] = valid images (dynamic batch read on the device)."""
        lib = self.lib
        H = self.image
        st = _native.stream_ptr(stream)
        cnt = _native.ptr(count)
        a, b, c = (t.data_ptr() for t in self.buf)
        h, w = self.stem(lib, self.x16.data_ptr(), B, H // 2, H // 2, a, st, count=count)  # 112x112x64
        _native.check("gg_maxpool3x3s2", lib.gg_maxpool3x3s2(C.c_void_p(a), B, h, w, 64,
                                                            C.c_void_p(b), cnt, st))
        h, w = (h + 1) // 2, (w + 1) // 2                                      # 56x56x64
        cur, free = b, [a, c]
        for conv1, conv2, ds in self.blocks:
            t1 = free[0]
            h2, w2 = conv1(lib, cur, B, h, w, t1, st, relu=True, count=count)
            if ds is not None:
                # identity branch = 1x1/2 conv + BN; the block input is dead afterwards
                t2 = free[1]
                ds(lib, cur, B, h, w, t2, st, relu=False, count=count)
                conv2(lib, t1, B, h2, w2, cur, st, residual=t2, relu=True, count=count)
                free = [t1, t2]
            else:
                out = free[1]
                conv2(lib, t1, B, h2, w2, out, st, residual=cur, relu=True, count=count)
                free = [cur, t1]
                cur = out
            h, w = h2, w2
        _native.check("gg_avgpool", lib.gg_avgpool(C.c_void_p(cur), B, h * w, 512,
                                                   _native.ptr(self.pooled), cnt, st))
        gemm(lib, self.pooled.data_ptr(), 512, self.w_fc, self.logits.data_ptr(),
             self.logits.stride(0), B, self.w_fc.shape[0], 512, st, bias=self.b_fc,
             out_mode=OUT_F32, tile_n=64, count=count, rows_per_item=1)
        return self.logits[:B, : self.num_classes]


def random_model(seed: int = 0):
    """Seeded random-init torchvision ResNet-18 (no pretrained weights offline)."""
    import torch
    import torchvision

    torch.manual_seed(seed)
    return torchvision.models.resnet18(weights=None).eval()
