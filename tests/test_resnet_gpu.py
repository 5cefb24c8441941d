"""ResNet-18 forward (implicit-GEMM tcgen05 convs, fp16 storage) vs torchvision eager fp32.

Oracle: torchvision eager in IEEE fp32 (cuDNN / cuBLAS TF32 disabled by
tests/conftest.py).  Logits: the north star's 2e-2 ABSOLUTE bound on every
logit (b = 2 and b = 64).  Single convolutions are checked against torch's
fp32 conv2d on the same 16-bit inputs, within 2e-2 relative to the output
scale (one rounding of the output).
"""

from __future__ import annotations

import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_2601_04250_b200 import _native
    return torch, _native, _native.load()


@pytest.mark.parametrize("n,h,cin,cout,r,stride,pad,res", [
    (2, 56, 64, 64, 3, 1, 1, True), (2, 56, 64, 128, 3, 2, 1, False), (2, 56, 64, 128, 1, 2, 0, False),
    (1, 14, 256, 512, 3, 2, 1, False), (1, 7, 512, 512, 3, 1, 1, True), (2, 30, 8, 64, 7, 2, 3, False),
    (3, 28, 128, 256, 3, 1, 1, True)])
def test_conv_vs_torch(env, n, h, cin, cout, r, stride, pad, res):
    torch, nat, lib = env
    g = torch.Generator(device="cuda").manual_seed(n * h + cin)
    x = torch.randn((n, cin, h, h), device="cuda", generator=g).to(torch.float16)
    w = (torch.randn((cout, cin, r, r), device="cuda", generator=g) / (cin * r * r) ** 0.5).to(torch.float16)
    b = torch.randn(cout, device="cuda", generator=g)
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=stride, padding=pad)
    ho = ref.shape[2]
    resid = torch.randn((n, ho, ho, cout), device="cuda", generator=g).to(torch.float16) if res else None
    if res:
        ref = ref + resid.float().permute(0, 3, 1, 2)
    ref = torch.relu(ref)
    k = r * r * cin
    kpad = (k + 63) // 64 * 64
    wk = torch.zeros((cout, kpad), dtype=torch.float16, device="cuda")
    wk[:, :k] = w.permute(0, 2, 3, 1).reshape(cout, k)
    xn = x.permute(0, 2, 3, 1).contiguous()
    y = torch.empty((n, ho, ho, cout), dtype=torch.float16, device="cuda")
    nat.check("gg_conv2d", lib.gg_conv2d(nat.ptr(xn), n, h, h, cin, nat.ptr(wk), cout, r, r, stride,
                                         pad, kpad, nat.ptr(b), nat.ptr(resid), 1, nat.ptr(y),
                                         -1, 0, None, nat.stream_ptr()))
    got = y.float().permute(0, 3, 1, 2)
    err = (got - ref).abs().max().item()
    assert err <= 2e-2 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("n,h,cin,cout,r,stride,pad,res", [
    (64, 7, 512, 512, 3, 1, 1, True), (64, 14, 256, 512, 3, 2, 1, False), (8, 14, 256, 256, 3, 1, 1, True),
    (64, 14, 256, 512, 1, 2, 0, False)])
def test_conv_stream_k(env, n, h, cin, cout, r, stride, pad, res):
    """Stream-K im2col conv (layer-3/4 shapes) == data-parallel within bf16 rounding,
    bit-identical across runs."""
    torch, nat, lib = env
    g = torch.Generator(device="cuda").manual_seed(n * h + cin + cout)
    x = torch.randn((n, h, h, cin), device="cuda", generator=g).to(torch.float16)
    w = (torch.randn((cout, r * r * cin), device="cuda", generator=g) / (cin * r * r) ** 0.5).to(torch.float16)
    b = torch.randn(cout, device="cuda", generator=g)
    ho = (h + 2 * pad - r) // stride + 1
    resid = torch.randn((n, ho, ho, cout), device="cuda", generator=g).to(torch.float16) if res else None
    outs = []
    assert lib.gg_streamk_reserve() == 0
    prev = lib.gg_streamk_mode(0)
    try:
        for mode in (0, 1, 1):
            lib.gg_streamk_mode(mode)
            y = torch.empty((n, ho, ho, cout), dtype=torch.float16, device="cuda")
            nat.check("gg_conv2d", lib.gg_conv2d(nat.ptr(x), n, h, h, cin, nat.ptr(w), cout, r, r,
                                                 stride, pad, r * r * cin, nat.ptr(b), nat.ptr(resid),
                                                 1, nat.ptr(y), -1, 0, None, nat.stream_ptr()))
            outs.append(y)
    finally:
        lib.gg_streamk_mode(prev)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2),
                                     w.float().reshape(cout, r, r, cin).permute(0, 3, 1, 2), b,
                                     stride=stride, padding=pad)
    if res:
        ref = ref + resid.float().permute(0, 3, 1, 2)
    ref = torch.relu(ref).permute(0, 2, 3, 1)
    scale = max(1.0, ref.abs().max().item())
    assert torch.equal(outs[1], outs[2])
    assert (outs[1].float() - ref).abs().max().item() <= 2e-2 * scale
    assert (outs[1].float() - outs[0].float()).abs().max().item() <= 1e-2 * scale


def test_space_to_depth_stem_vs_torch(env):
    """7x7/2 pad 3 conv (conv1+bn1) == 4x4/1 pad (2,1) conv over the s2d(2) input."""
    torch, nat, lib = env
    from paper_2601_04250_b200.resnet18 import _StemConv
    g = torch.Generator().manual_seed(3)
    conv = torch.nn.Conv2d(3, 64, 7, 2, 3, bias=False)
    bn = torch.nn.BatchNorm2d(64).eval()
    with torch.no_grad():
        conv.weight.copy_(torch.randn(conv.weight.shape, generator=g) * 0.1)
        bn.running_mean.copy_(torch.randn(64, generator=g) * 0.1)
        bn.running_var.copy_(torch.rand(64, generator=g) + 0.5)
        bn.weight.copy_(torch.rand(64, generator=g) + 0.5)
        bn.bias.copy_(torch.randn(64, generator=g) * 0.1)
    stem = _StemConv(conv, bn, "cuda")
    x = torch.randn((3, 3, 224, 224), generator=g).cuda()
    with torch.no_grad():
        ref = torch.relu(bn.cuda()(conv.cuda()(x.to(torch.float16).float())))
    # span path: zero-bordered s2d input
    x16p = torch.zeros((3, 115, 115, 16), dtype=torch.float16, device="cuda")
    nat.check("gg_nchw_to_s2d16", lib.gg_nchw_to_s2d16(nat.ptr(x), 3, 224, 224, 1, nat.ptr(x16p),
                                                       nat.stream_ptr()))
    y = torch.empty((3, 112, 112, 64), dtype=torch.float16, device="cuda")
    stem(lib, x16p.data_ptr(), 3, 112, 112, y.data_ptr(), nat.stream_ptr(), relu=True)
    got = y.float().permute(0, 3, 1, 2)
    err = (got - ref).abs().max().item()
    assert err <= 2e-2 * max(1.0, ref.abs().max().item()), err
    # im2col cross-check path: dense s2d input
    x16 = torch.empty((3, 112, 112, 16), dtype=torch.float16, device="cuda")
    nat.check("gg_nchw_to_s2d16", lib.gg_nchw_to_s2d16(nat.ptr(x), 3, 224, 224, 0, nat.ptr(x16),
                                                       nat.stream_ptr()))
    y2 = torch.empty_like(y)
    stem.im2col(lib, x16.data_ptr(), 3, 112, 112, y2.data_ptr(), nat.stream_ptr(), relu=True)
    err2 = (y2.float().permute(0, 3, 1, 2) - ref).abs().max().item()
    assert err2 <= 2e-2 * max(1.0, ref.abs().max().item()), err2


@pytest.mark.parametrize("n,hs,count,out_pad", [(3, 112, None, 0), (64, 112, None, 2), (64, 112, 37, 2),
                                                 (5, 32, None, 0), (7, 20, 6, 2), (1, 128, None, 0)])
def test_stem_pool_fused(env, n, hs, count, out_pad):
    """gg_stem_pool_span == gg_stem_s2d_span -> gg_maxpool3x3s2, bit for bit (max is
    order-free and bf16 rounding monotonic); pool-row bands that cross images, a
    device count below the batch, and the shared-border output's zero border."""
    torch, nat, lib = env
    from paper_2601_04250_b200.resnet18 import _StemConv
    g = torch.Generator().manual_seed(hs + n)
    conv = torch.nn.Conv2d(3, 64, 7, 2, 3, bias=False)
    bn = torch.nn.BatchNorm2d(64).eval()
    with torch.no_grad():
        conv.weight.copy_(torch.randn(conv.weight.shape, generator=g) * 0.1)
        bn.running_mean.copy_(torch.randn(64, generator=g) * 0.1)
        bn.running_var.copy_(torch.rand(64, generator=g) + 0.5)
        bn.weight.copy_(torch.rand(64, generator=g) + 0.5)
        bn.bias.copy_(torch.randn(64, generator=g) * 0.1)
    stem = _StemConv(conv, bn, "cuda")
    x = torch.randn((n, 3, 2 * hs, 2 * hs), generator=g).cuda()
    x16p = torch.zeros((n, hs + 3, hs + 3, 16), dtype=torch.float16, device="cuda")
    nat.check("gg_nchw_to_s2d16", lib.gg_nchw_to_s2d16(nat.ptr(x), n, 2 * hs, 2 * hs, 1, nat.ptr(x16p),
                                                       nat.stream_ptr()))
    cnt = torch.tensor([count], dtype=torch.int32, device="cuda") if count is not None else None
    y = torch.empty((n, hs, hs, 64), dtype=torch.float16, device="cuda")
    stem(lib, x16p.data_ptr(), n, hs, hs, y.data_ptr(), nat.stream_ptr(), relu=True)
    ho = hs // 2
    ref = torch.empty((n, ho, ho, 64), dtype=torch.float16, device="cuda")
    nat.check("gg_maxpool3x3s2", lib.gg_maxpool3x3s2(nat.ptr(y), n, hs, hs, 64, nat.ptr(ref), 0, None,
                                                     nat.stream_ptr()))
    if out_pad == 2:
        out = torch.zeros(((ho + 2) + n * (ho + 1) * (ho + 1), 64), dtype=torch.float16, device="cuda")
    else:
        out = torch.full((n, ho, ho, 64), -7.0, dtype=torch.float16, device="cuda")
    nat.check("gg_stem_pool_span", lib.gg_stem_pool_span(
        nat.ptr(x16p), n, hs, hs, nat.ptr(stem.w), 64, nat.ptr(stem.b), nat.ptr(out), out_pad,
        nat.ptr(cnt), nat.stream_ptr()))
    torch.cuda.synchronize()
    got = _from_shared(out, n, ho, 64) if out_pad == 2 else out
    k = n if count is None else count
    assert torch.equal(got[:k, :ho, :ho], ref[:k])
    if out_pad == 2:
        assert (got[:, ho] == 0).all() and (got[:, :, ho] == 0).all() and (out[: ho + 2] == 0).all()
        assert (got[k:] == 0).all()
    else:
        assert (got[k:] == -7.0).all()


def test_pools(env):
    torch, nat, lib = env
    x = torch.randn((2, 64, 112, 112), device="cuda").to(torch.float16)
    xn = x.permute(0, 2, 3, 1).contiguous()
    y = torch.empty((2, 56, 56, 64), dtype=torch.float16, device="cuda")
    nat.check("gg_maxpool3x3s2", lib.gg_maxpool3x3s2(nat.ptr(xn), 2, 112, 112, 64, nat.ptr(y),
                                                     0, None, nat.stream_ptr()))
    ref = torch.nn.functional.max_pool2d(x.float(), 3, 2, 1)
    assert torch.equal(y.float().permute(0, 3, 1, 2), ref)
    z = torch.empty((2, 64), dtype=torch.float16, device="cuda")
    nat.check("gg_avgpool", lib.gg_avgpool(nat.ptr(y), 2, 56 * 56, 64, nat.ptr(z), 0, None,
                                           nat.stream_ptr()))
    assert (z.float() - ref.mean(dim=(2, 3))).abs().max().item() < 1e-2
    # padded variants: maxpool into a zero-bordered buffer, avgpool over it with the interior count
    yp = torch.zeros((2, 58, 58, 64), dtype=torch.float16, device="cuda")
    nat.check("gg_maxpool3x3s2", lib.gg_maxpool3x3s2(nat.ptr(xn), 2, 112, 112, 64, nat.ptr(yp),
                                                     1, None, nat.stream_ptr()))
    assert torch.equal(yp[:, 1:-1, 1:-1], y) and (yp[:, 0] == 0).all() and (yp[:, :, -1] == 0).all()
    zp = torch.empty((2, 64), dtype=torch.float16, device="cuda")
    nat.check("gg_avgpool", lib.gg_avgpool(nat.ptr(yp), 2, 58 * 58, 64, nat.ptr(zp), 56 * 56, None,
                                           nat.stream_ptr()))
    assert (zp.float() - ref.mean(dim=(2, 3))).abs().max().item() < 1e-2


@pytest.mark.parametrize("n,h,cin,cout", [(64, 58, 64, 128), (64, 30, 128, 256), (64, 16, 256, 512),
                                         (3, 16, 256, 512)])
def test_conv2d_ds_fused(env, n, h, cin, cout):
    """3x3/2 conv + 1x1/2 downsample in one kernel (gg_conv2d_ds) == the two
    separate gg_conv2d launches, bit for bit (same K order per accumulator), on a
    zero-bordered input of padded extent h; both outputs zero-bordered."""
    torch, nat, lib = env
    g = torch.Generator(device="cuda").manual_seed(h + cin)
    x = torch.zeros((n, h, h, cin), dtype=torch.float16, device="cuda")
    x[:, 1:-1, 1:-1] = torch.randn((n, h - 2, h - 2, cin), device="cuda", generator=g).to(torch.float16)
    w = (torch.randn((cout, 9 * cin), device="cuda", generator=g) / (9 * cin) ** 0.5).to(torch.float16)
    wd = (torch.randn((cout, cin), device="cuda", generator=g) / cin ** 0.5).to(torch.float16)
    b = torch.randn(cout, device="cuda", generator=g)
    bd = torch.randn(cout, device="cuda", generator=g)
    ho = (h - 3) // 2 + 1
    shape = (n, ho + 2, ho + 2, cout)
    y1, yd1, y2, yd2 = (torch.zeros(shape, dtype=torch.float16, device="cuda") for _ in range(4))
    nat.check("gg_conv2d", lib.gg_conv2d(nat.ptr(x), n, h, h, cin, nat.ptr(w), cout, 3, 3, 2, 0, 9 * cin,
                                         nat.ptr(b), None, 1, nat.ptr(y1), 0, 1, None, nat.stream_ptr()))
    nat.check("gg_conv2d", lib.gg_conv2d(nat.ptr(x), n, h, h, cin, nat.ptr(wd), cout, 1, 1, 2, -1, cin,
                                         nat.ptr(bd), None, 0, nat.ptr(yd1), -1, 1, None, nat.stream_ptr()))
    nat.check("gg_conv2d_ds", lib.gg_conv2d_ds(nat.ptr(x), n, h, h, cin, nat.ptr(w), cout, nat.ptr(b),
                                               nat.ptr(y2), nat.ptr(wd), nat.ptr(bd), nat.ptr(yd2), 0, 0,
                                               None, nat.stream_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert torch.equal(yd1, yd2)
    # and against torch on the interior
    xi = x.float().permute(0, 3, 1, 2)
    ref = torch.relu(torch.nn.functional.conv2d(xi, w.float().reshape(cout, 3, 3, cin).permute(0, 3, 1, 2),
                                                b, stride=2))
    got = y2[:, 1:-1, 1:-1].float().permute(0, 3, 1, 2)
    assert (got - ref).abs().max().item() <= 2e-2 * max(1.0, ref.abs().max().item())


def _to_shared(t, s):
    """[n, s, s, c] interior -> shared-border buffer [(s+2) margin][n, s+1, s+1, c] (flat rows)."""
    import torch
    n, _, _, c = t.shape
    img = torch.zeros((n, s + 1, s + 1, c), dtype=t.dtype, device=t.device)
    img[:, :s, :s] = t
    return torch.cat([torch.zeros((s + 2, c), dtype=t.dtype, device=t.device), img.reshape(-1, c)])


def _from_shared(buf, n, s, c):
    return buf[s + 2:].reshape(n, s + 1, s + 1, c)


@pytest.mark.parametrize("n,s,c,cout", [(64, 56, 64, 64), (3, 56, 64, 64), (1, 7, 64, 64), (5, 9, 64, 64),
                                        (64, 28, 128, 128), (64, 14, 256, 256), (64, 7, 512, 512),
                                        (3, 7, 512, 512)])
def test_conv3x3_shared_border(env, n, s, c, cout):
    """Span conv on the shared-border layout (layers 1-4; C = Cout = 64 runs the
    pixel-pair kernel conv_span_px2, odd pixel counts included) vs torch's padded
    conv, with residual; the zero row / column of every image stays zero."""
    torch, nat, lib = env
    from tests.test_conv_span_gpu import pack_span_weights
    g = torch.Generator(device="cuda").manual_seed(s + c)
    x = torch.randn((n, s, s, c), device="cuda", generator=g).to(torch.float16)
    r = torch.randn((n, s, s, cout), device="cuda", generator=g).to(torch.float16)
    w = (torch.randn((cout, c, 3, 3), device="cuda", generator=g) / (9 * c) ** 0.5).to(torch.float16)
    b = torch.randn(cout, device="cuda", generator=g)
    xs, rs = _to_shared(x, s), _to_shared(r, s)
    ys = torch.full_like(_to_shared(torch.zeros((n, s, s, cout), dtype=torch.float16, device="cuda"), s), 0)
    # a canary region right after the output buffer must stay untouched
    rows = ys.shape[0]
    yc = torch.cat([ys, torch.full((64, cout), 7.0, dtype=torch.float16, device="cuda")])
    nat.check("gg_conv3x3_shared", lib.gg_conv3x3_shared(
        nat.ptr(xs), n, s, s, c, nat.ptr(pack_span_weights(w)), cout, nat.ptr(b), nat.ptr(rs), 1,
        nat.ptr(yc), None, nat.stream_ptr()))
    torch.cuda.synchronize()
    assert (yc[rows:] == 7.0).all()
    ys = yc[:rows]
    ref = torch.relu(torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2), w.float(), b, padding=1) +
                     r.float().permute(0, 3, 1, 2))
    got = _from_shared(ys, n, s, cout)
    err = (got[:, :s, :s].float().permute(0, 3, 1, 2) - ref).abs().max().item()
    assert err <= 2e-2 * max(1.0, ref.abs().max().item()), err
    assert (got[:, s] == 0).all() and (got[:, :, s] == 0).all() and (ys[: s + 2] == 0).all()


@pytest.mark.parametrize("n,s,cin,cout,in_shared", [(64, 56, 64, 128, 0), (64, 28, 128, 256, 1),
                                                    (64, 14, 256, 512, 1), (2, 14, 256, 512, 1)])
def test_conv2d_ds_shared_border(env, n, s, cin, cout, in_shared):
    """Fused stride-2 conv + downsample reading a bordered (layer 1) or shared-border
    input and writing shared-border outputs, vs torch."""
    torch, nat, lib = env
    g = torch.Generator(device="cuda").manual_seed(s + cin)
    x = torch.randn((n, s, s, cin), device="cuda", generator=g).to(torch.float16)
    if in_shared:
        xb, ext = _to_shared(x, s), s + 1
    else:
        xb = torch.zeros((n, s + 2, s + 2, cin), dtype=torch.float16, device="cuda")
        xb[:, 1:-1, 1:-1] = x
        ext = s + 2
    w = (torch.randn((cout, 9 * cin), device="cuda", generator=g) / (9 * cin) ** 0.5).to(torch.float16)
    wd = (torch.randn((cout, cin), device="cuda", generator=g) / cin ** 0.5).to(torch.float16)
    b = torch.randn(cout, device="cuda", generator=g)
    bd = torch.randn(cout, device="cuda", generator=g)
    so = s // 2
    y = _to_shared(torch.zeros((n, so, so, cout), dtype=torch.float16, device="cuda"), so)
    yd = y.clone()
    nat.check("gg_conv2d_ds", lib.gg_conv2d_ds(nat.ptr(xb), n, ext, ext, cin, nat.ptr(w), cout, nat.ptr(b),
                                               nat.ptr(y), nat.ptr(wd), nat.ptr(bd), nat.ptr(yd), in_shared, 1,
                                               None, nat.stream_ptr()))
    torch.cuda.synchronize()
    xi = x.float().permute(0, 3, 1, 2)
    ref = torch.relu(torch.nn.functional.conv2d(xi, w.float().reshape(cout, 3, 3, cin).permute(0, 3, 1, 2),
                                                b, stride=2, padding=1))
    refd = torch.nn.functional.conv2d(xi, wd.float().reshape(cout, cin, 1, 1), bd, stride=2)
    got = _from_shared(y, n, so, cout)[:, :so, :so].float().permute(0, 3, 1, 2)
    gotd = _from_shared(yd, n, so, cout)[:, :so, :so].float().permute(0, 3, 1, 2)
    for a, rr in ((got, ref), (gotd, refd)):
        assert (a - rr).abs().max().item() <= 2e-2 * max(1.0, rr.abs().max().item())
    assert (_from_shared(y, n, so, cout)[:, so] == 0).all()


@pytest.mark.parametrize("n,c,h,w", [(3, 64, 29, 31), (1, 128, 9, 10), (2, 8, 7, 5)])
def test_maxpool_ragged_shapes(env, n, c, h, w):
    """Blocked max pool (4 x 2 outputs per thread) at sizes that leave partial blocks: exact."""
    torch, nat, lib = env
    x = torch.randn((n, c, h, w), device="cuda").to(torch.float16)
    xn = x.permute(0, 2, 3, 1).contiguous()
    ref = torch.nn.functional.max_pool2d(x.float(), 3, 2, 1)
    ho, wo = ref.shape[2], ref.shape[3]
    y = torch.full((n, ho, wo, c), 7.0, dtype=torch.float16, device="cuda")
    nat.check("gg_maxpool3x3s2", lib.gg_maxpool3x3s2(nat.ptr(xn), n, h, w, c, nat.ptr(y), 0, None,
                                                     nat.stream_ptr()))
    assert torch.equal(y.float().permute(0, 3, 1, 2), ref)


@pytest.mark.parametrize("batch", [2, 64])
def test_resnet18_logits_vs_eager(env, batch):
    torch = env[0]
    from paper_2601_04250_b200.resnet18 import ResNet18B200, random_model
    model = random_model(0)
    x = torch.randn((batch, 3, 224, 224), generator=torch.Generator().manual_seed(1))
    assert not torch.backends.cudnn.allow_tf32       # IEEE fp32 oracle (conftest.py)
    with torch.no_grad():
        ref = model.cuda()(x.cuda()).float()
    net = ResNet18B200(model, max_batch=batch)
    out = net.forward(x.cuda())
    torch.cuda.synchronize()
    scale = ref.abs().max().item()
    err = (out - ref).abs().max().item()
    print(f"resnet18 b={batch}: max |logit err| = {err:.3e}, logit scale {scale:.3f}, "
          f"argmax agree {(out.argmax(1) == ref.argmax(1)).float().mean().item():.3f}")
    assert err <= 2e-2, err                           # absolute (north star)


@pytest.mark.parametrize("padded", [0, 1])
def test_stem_gather(env, padded):
    """uint8 HWC pool -> normalized space-to-depth(2) 16-channel input, through
    batch ids (modulo the pool) and a device count (rows past it untouched)."""
    torch, nat, lib = env
    g = torch.Generator().manual_seed(5)
    pool = torch.randint(0, 256, (5, 224, 224, 3), dtype=torch.uint8, generator=g).cuda()
    ids = torch.tensor([3, 7, 0, 12], dtype=torch.int32, device="cuda")
    count = torch.tensor([3], dtype=torch.int32, device="cuda")
    mean = torch.tensor([0.485, 0.456, 0.406], dtype=torch.float32)
    std = torch.tensor([0.229, 0.224, 0.225], dtype=torch.float32)
    shape = (4, 115, 115, 16) if padded else (4, 112, 112, 16)
    y = torch.full(shape, 9.0, dtype=torch.float16, device="cuda")
    nat.check("gg_stem_gather", lib.gg_stem_gather(
        nat.ptr(pool), 5, nat.ptr(ids), nat.ptr(count), 4, 224, 224,
        mean.numpy().ctypes.data_as(C.c_void_p), std.numpy().ctypes.data_as(C.c_void_p), padded,
        nat.ptr(y), nat.stream_ptr()))
    torch.cuda.synchronize()
    # same fp32 arithmetic as the kernel: x * fl32(1/255), then (. - mean) / std
    imgs = pool[(ids[:3] % 5).long()].float() * torch.tensor(1.0 / 255.0, dtype=torch.float32).cuda()
    norm = (imgs - mean.cuda()) / std.cuda()
    s2d = norm.reshape(3, 112, 2, 112, 2, 3).permute(0, 1, 3, 2, 4, 5).reshape(3, 112, 112, 12)
    if padded:   # undo the SW32 pre-swizzle: cells with bit 2 of the linear index set are swapped
        q = torch.arange(115 * 115 * 4, device="cuda").reshape(4, 115, 115)
        sw = ((q >> 2) & 1).bool()
        y = torch.where(sw[..., None], torch.cat([y[..., 8:], y[..., :8]], dim=-1), y)
    got = y[:3, 2:-1, 2:-1] if padded else y[:3]
    assert torch.equal(got[..., :12].float(), s2d.to(torch.float16).float())
    assert (got[..., 12:].float() == 0).all()
    assert (y[3].float() == 9.0).all()                            # beyond the count
    if padded:
        assert (y[:3, :2].float() == 9.0).all()                   # borders not written


def test_conv3x3_shared_border_px2_count(env):
    """Pixel-pair layer-1 conv with a device image count below the batch (the serving
    loop's dynamic batch): the counted images match torch."""
    torch, nat, lib = env
    from tests.test_conv_span_gpu import pack_span_weights
    n, s, c, k = 6, 56, 64, 3
    g = torch.Generator(device="cuda").manual_seed(77)
    x = torch.randn((n, s, s, c), device="cuda", generator=g).to(torch.float16)
    r = torch.randn((n, s, s, c), device="cuda", generator=g).to(torch.float16)
    w = (torch.randn((c, c, 3, 3), device="cuda", generator=g) / (9 * c) ** 0.5).to(torch.float16)
    b = torch.randn(c, device="cuda", generator=g)
    xs, rs = _to_shared(x, s), _to_shared(r, s)
    ys = torch.zeros_like(xs)
    cnt = torch.tensor([k], dtype=torch.int32, device="cuda")
    nat.check("gg_conv3x3_shared", lib.gg_conv3x3_shared(
        nat.ptr(xs), n, s, s, c, nat.ptr(pack_span_weights(w)), c, nat.ptr(b), nat.ptr(rs), 1,
        nat.ptr(ys), nat.ptr(cnt), nat.stream_ptr()))
    torch.cuda.synchronize()
    ref = torch.relu(torch.nn.functional.conv2d(x[:k].float().permute(0, 3, 1, 2), w.float(), b, padding=1) +
                     r[:k].float().permute(0, 3, 1, 2))
    got = _from_shared(ys, n, s, c)[:k, :s, :s].float().permute(0, 3, 1, 2)
    assert (got - ref).abs().max().item() <= 2e-2 * max(1.0, ref.abs().max().item())
