"""ResNet-18 (torchvision architecture, 224x224) forward on sm_100a, NHWC fp16 (csrc/gg_act.cuh).

Layout: every stage's activations live in the shared-border layout ([s+2 zero
rows][N, s+1, s+1, C]: one zero row and column per image, which are also the next
row's / image's left / top border), 3-31 % fewer positions for the span convs
than [s+2, s+2] at 56² / 28² / 14² / 7².
Three buffers per stage, zeroed once.  Then:

  stem+pool  gg_stem_pool_span: conv1 7x7/2 + bn1 + ReLU as a 4x4/1 span conv
             over the space-to-depth(2) input, one stem row per tile, with the
             3x3/2 max pool in the epilogue (smem row + register partials),
             written into the interior of the layer-1 buffer; the stem output
             never reaches memory (GG_STEM_UNFUSED=1: gg_stem_s2d_span +
             gg_maxpool3x3s2)
  3x3 / 1    gg_conv3x3_shared: one
             TMA span load per 64-channel block feeds all nine taps (shifted UMMA
             descriptors); CTA pairs for Cout >= 128; border positions written as
             zeros
  3x3 / 2    gg_conv2d_ds: TMA im2col of the previous stage's buffer, fused with
  + 1x1 / 2  the block's downsample (the 1x1/2 reads the 3x3's centre-tap tiles;
             second TMEM accumulator), both outputs in the shared-border layout
  head       gg_avgpool_fc: fp32 average pool over the shared-border 8x8 map
             (divides by 49) + fp32 fc (fp32 weights) -> fp32 logits for K3

Eval-mode BatchNorm is folded into every conv's weights/bias; residual add and
ReLU are fused into the conv epilogues.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _native


def _fold(conv, bn):
    """BN(conv(x)) == conv'(x) + b' in eval mode.  Returns ([Cout, R, S, Cin] fp32, bias)."""
    import torch

    w = conv.weight.detach().float()
    scale = bn.weight.detach().float() / torch.sqrt(bn.running_var.detach().float() + bn.eps)
    bias = bn.bias.detach().float() - bn.running_mean.detach().float() * scale
    w = w * scale[:, None, None, None]
    return w.permute(0, 2, 3, 1).contiguous().cpu(), bias.cpu()


class _Conv:
    """Generic implicit-GEMM conv (gg_conv2d): weights [Cout, R*S*Cin] (r, s, c order)."""

    def __init__(self, conv, bn, device, pad=None, pad_hi=None, out_pad=0):
        import torch
        w, b = _fold(conv, bn)
        cout, R, S, cin = w.shape
        k = R * S * cin
        kpad = (k + 63) // 64 * 64
        wk = torch.zeros((cout, kpad), dtype=torch.float32)
        wk[:, :k] = w.reshape(cout, k)
        self.w = wk.to(device=device, dtype=torch.float16).contiguous()
        self.b = b.to(device=device).contiguous()
        self.kpad, self.cout, self.cin = kpad, cout, cin
        self.r, self.s = R, S
        self.stride = conv.stride[0]
        self.pad = conv.padding[0] if pad is None else pad
        self.pad_hi = self.pad if pad_hi is None else pad_hi
        self.out_pad = out_pad
        self.algo_macs_per_pixel = R * S * conv.in_channels * cout

    def out_hw(self, h, w):
        return ((h + self.pad + self.pad_hi - self.r) // self.stride + 1,
                (w + self.pad + self.pad_hi - self.s) // self.stride + 1)

    def __call__(self, lib, x, n, h, w, y, st, residual=None, relu=True, count=None):
        _native.check("gg_conv2d", lib.gg_conv2d(
            C.c_void_p(x), n, h, w, self.cin, _native.ptr(self.w), self.cout, self.r, self.s,
            self.stride, self.pad, self.kpad, _native.ptr(self.b),
            None if residual is None else C.c_void_p(residual), int(relu), C.c_void_p(y),
            self.pad_hi, self.out_pad, _native.ptr(count), st))
        return self.out_hw(h, w)

    def flops(self, n, ho, wo):
        """Algorithmic FLOPs of the original convolution (padding channels excluded)."""
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
        w, bias = _fold(conv, bn)            # [64, 7, 7, 3]
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
                            wp[:, i, j, (dy * 2 + dx) * 3 + c] = w[:, r, s, c]
        self.w = wp.reshape(cout, 256).to(device=device, dtype=torch.float16).contiguous()
        self.b = bias.to(device=device).contiguous()
        self.kpad, self.cout, self.cin = 256, cout, 16
        self.r = self.s = 4
        self.stride, self.pad, self.pad_hi, self.out_pad = 1, 2, 1, 0
        self.algo_macs_per_pixel = 7 * 7 * 3 * cout

    def __call__(self, lib, x, n, h, w, y, st, residual=None, relu=True, count=None):
        """x: zero-bordered space-to-depth input [n, h+3, w+3, 16] (gg_nchw_to_s2d16 /
        gg_stem_gather with padded=1); y: dense [n, h, w, 64]."""
        assert residual is None
        _native.check("gg_stem_s2d_span", lib.gg_stem_s2d_span(
            C.c_void_p(x), n, h, w, _native.ptr(self.w), self.cout, _native.ptr(self.b), int(relu),
            C.c_void_p(y), _native.ptr(count), st))
        return h, w

    def im2col(self, lib, x, n, h, w, y, st, relu=True, count=None):
        """Cross-check path: the same conv through gg_conv2d's 16-channel im2col
        mode on the dense [n, h, w, 16] space-to-depth input."""
        return _Conv.__call__(self, lib, x, n, h, w, y, st, relu=relu, count=count)


class _SpanConv:
    """3x3 / 1 conv on padded activations (gg_conv3x3_padded); weights in
    (channel block, tap, channel) K order."""

    def __init__(self, conv, bn, device, shared: bool = False):
        import torch
        self.shared = shared                 # shared-border layout (layers 2-4)
        w, b = _fold(conv, bn)               # [Cout, 3, 3, Cin]
        cout, _, _, cin = w.shape
        wk = w.reshape(cout, 9, cin // 64, 64).permute(0, 2, 1, 3).reshape(cout, 9 * cin)
        self.w = wk.to(device=device, dtype=torch.float16).contiguous()
        self.b = b.to(device=device).contiguous()
        self.cin, self.cout = cin, cout
        self.algo_macs_per_pixel = 9 * cin * cout

    def __call__(self, lib, x, n, h, w, y, st, residual=None, relu=True, count=None):
        fn = lib.gg_conv3x3_shared if self.shared else lib.gg_conv3x3_padded
        _native.check("gg_conv3x3", fn(
            C.c_void_p(x), n, h, w, self.cin, _native.ptr(self.w), self.cout, _native.ptr(self.b),
            None if residual is None else C.c_void_p(residual), int(relu), C.c_void_p(y),
            _native.ptr(count), st))
        return h, w

    def flops(self, n, ho, wo):
        return 2.0 * n * ho * wo * self.algo_macs_per_pixel


class ResNet18B200:
    """Packed (BN-folded) weights + padded NHWC activation buffers for up to max_batch images."""

    def __init__(self, tv_model, max_batch: int = 64, image: int = 224, device="cuda"):
        torch = _native.require_cuda()
        self.lib = _native.load()
        # stream-K workspace now, before any CUDA graph capture of the forward
        _native.check("gg_streamk_reserve", self.lib.gg_streamk_reserve())
        self.device = torch.device(device)
        self.max_batch, self.image = max_batch, image
        m = tv_model.eval()
        dev = self.device
        self.stem = _StemConv(m.conv1, m.bn1, dev)
        # stages: (blocks, geometry of the stage's padded buffers)
        self.blocks = []
        cin = 64
        for li, layer in enumerate((m.layer1, m.layer2, m.layer3, m.layer4)):
            for bi, blk in enumerate(layer):
                cout = blk.conv1.out_channels
                if blk.conv1.stride[0] == 2:
                    # 3x3/2 on the previous stage's padded buffer: pad 0 (physical padding)
                    c1 = _Conv(blk.conv1, blk.bn1, dev, pad=0, pad_hi=0, out_pad=1)
                else:
                    c1 = self._stride1(blk.conv1, blk.bn1, dev, li)
                ds = None
                if blk.downsample is not None:
                    # 1x1/2 reads interior pixel (2ho+1, 2wo+1) of the padded input: pad -1
                    ds = _Conv(blk.downsample[0], blk.downsample[1], dev, pad=-1, pad_hi=-1,
                               out_pad=1)
                self.blocks.append((li, c1, self._stride1(blk.conv2, blk.bn2, dev, li), ds))
                cin = cout
        self.num_classes = m.fc.out_features
        # fp32 head (avgpool + fc): no bf16 rounding after the last conv
        self.w_fc = m.fc.weight.detach().float().to(dev).contiguous()
        self.b_fc = m.fc.bias.detach().float().to(dev).contiguous()
        B, H = max_batch, image
        z = dict(dtype=torch.float16, device=dev)
        # zero-bordered space-to-depth stem input [B, H/2+3, H/2+3, 16] (interior rewritten)
        self.x16 = torch.zeros(B * (H // 2 + 3) * (H // 2 + 3) * 16, **z)
        # GG_STEM_UNFUSED=1: separate stem conv + max pool kernels (A/B and cross-check)
        self.fuse_stem_pool = os.environ.get("GG_STEM_UNFUSED", "0") != "1"
        self.stem_out = torch.empty(B * (H // 2) * (H // 2) * 64 if not self.fuse_stem_pool else 0, **z)
        self.sizes = [H // 4, H // 8, H // 16, H // 32]             # 56, 28, 14, 7
        chans = [64, 128, 256, 512]
        # three zero-bordered buffers per stage (zeroed once; interiors rewritten every forward)
        # layer 1: zero-bordered [B, 58, 58, 64]; layers 2-4: shared-border layout
        # ([s+2 zero rows][B, s+1, s+1, C]: one zero row / column per image, 7-31 %
        # fewer positions for the span convs than [s+2, s+2])
        self.stage_bufs = [[torch.zeros(self._stage_rows(i, s, B) * c, **z) for _ in range(3)]
                           for i, (s, c) in enumerate(zip(self.sizes, chans))]
        self.pooled = torch.empty((B, 512), dtype=torch.float32, device=dev)
        self.logits = torch.empty((B, self.num_classes), dtype=torch.float32, device=dev)

    @staticmethod
    def _stage_rows(stage: int, s: int, batch: int) -> int:
        """Rows (pixels) of a shared-border stage buffer: (s+2) margin + batch x (s+1)^2."""
        return (s + 2) + batch * (s + 1) * (s + 1)

    def _stride1(self, conv, bn, dev, stage):
        return _SpanConv(conv, bn, dev, shared=True)

    def flops(self, batch: int) -> float:
        """Algorithmic FLOPs (3.628 GF/img at 224x224)."""
        n = batch
        f = self.stem.flops(n, self.image // 2, self.image // 2)
        for li, c1, c2, ds in self.blocks:
            s = self.sizes[li]
            f += c1.flops(n, s, s) + c2.flops(n, s, s)
            if ds is not None:
                f += ds.flops(n, s, s)
        f += 2.0 * n * 512 * self.num_classes
        return f

    def forward(self, images, batch: int | None = None, stream=None):
        """images: CUDA fp32 NCHW [B, 3, 224, 224].  Returns fp32 logits [B, 1000] (view)."""
        B = int(images.shape[0]) if batch is None else int(batch)
        assert B <= self.max_batch
        H = self.image
        st = _native.stream_ptr(stream)
        _native.check("gg_nchw_to_s2d16", self.lib.gg_nchw_to_s2d16(
            _native.ptr(images), B, H, H, 1, _native.ptr(self.x16), st))
        return self.forward_s2d(B, stream=stream)

    def forward_s2d(self, B: int, stream=None, count=None, x16=None):
        """Forward from self.x16 (or `x16`: the same layout, e.g. a second input slot)
        (fp16 space-to-depth(2) NHWC, 16 channels).
        count: optional CUDA int32 [1] = valid images (dynamic batch read on the device)."""
        lib = self.lib
        H = self.image
        st = _native.stream_ptr(stream)
        cnt = _native.ptr(count)
        x16 = self.x16 if x16 is None else x16
        bufs = [[t.data_ptr() for t in stage] for stage in self.stage_bufs]
        if self.fuse_stem_pool:
            # stem conv + max pool in one kernel: the 112x112x64 stem output never leaves the SM
            _native.check("gg_stem_pool_span", lib.gg_stem_pool_span(
                C.c_void_p(x16.data_ptr()), B, H // 2, H // 2, _native.ptr(self.stem.w), 64,
                _native.ptr(self.stem.b), C.c_void_p(bufs[0][0]), 2, cnt, st))
        else:
            h, w = self.stem(lib, x16.data_ptr(), B, H // 2, H // 2, self.stem_out.data_ptr(),
                             st, count=count)                                     # 112x112x64 dense
            _native.check("gg_maxpool3x3s2", lib.gg_maxpool3x3s2(
                _native.ptr(self.stem_out), B, h, w, 64, C.c_void_p(bufs[0][0]), 2, cnt, st))
        cur, free = bufs[0][0], [bufs[0][1], bufs[0][2]]
        stage = 0
        for li, c1, c2, ds in self.blocks:
            s = self.sizes[li]
            if li != stage:   # first block of a new stage: strided conv + downsample
                # one kernel (gg_conv2d_ds): the 1x1/2 downsample rides on the 3x3/2's
                # centre-tap tiles; shared-border input and outputs
                sp = self.sizes[stage] + 1                       # previous per-image extent
                t1, t2, out = bufs[li]
                _native.check("gg_conv2d_ds", lib.gg_conv2d_ds(
                    C.c_void_p(cur), B, sp, sp, c1.cin, _native.ptr(c1.w), c1.cout,
                    _native.ptr(c1.b), C.c_void_p(t1), _native.ptr(ds.w), _native.ptr(ds.b),
                    C.c_void_p(t2), 1, 1, cnt, st))
                c2(lib, t1, B, s, s, out, st, residual=t2, relu=True, count=count)
                cur, free = out, [t1, t2]
                stage = li
            else:
                t1, out = free
                c1(lib, cur, B, s, s, t1, st, relu=True, count=count)
                c2(lib, t1, B, s, s, out, st, residual=cur, relu=True, count=count)
                free = [cur, t1]
                cur = out
        s = self.sizes[-1]
        # shared-border map: per image (s+1)^2 positions after an (s+2)-row margin, zeros
        # outside the s x s interior (divide by s^2)
        _native.check("gg_avgpool_fc", lib.gg_avgpool_fc(
            C.c_void_p(cur + (s + 2) * 512 * 2), B, (s + 1) * (s + 1), 512, s * s,
            _native.ptr(self.w_fc), _native.ptr(self.b_fc), self.num_classes,
            _native.ptr(self.pooled), _native.ptr(self.logits), self.logits.stride(0), cnt, st))
        return self.logits[:B]


def random_model(seed: int = 0):
    """Seeded random-init torchvision ResNet-18 (no pretrained weights offline)."""
    import torch
    import torchvision

    torch.manual_seed(seed)
    return torchvision.models.resnet18(weights=None).eval()
