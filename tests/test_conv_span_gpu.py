"""3x3/1 span convolution on padded activations (gg_conv3x3_padded) vs torch fp32."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu


def pack_span_weights(w):
    """[Cout, C, 3, 3] -> [Cout, C/64, 3, 3, 64] flattened (K order: block, tap, channel)."""
    cout, c = w.shape[:2]
    return (w.permute(0, 2, 3, 1).reshape(cout, 9, c // 64, 64).permute(0, 2, 1, 3)
            .reshape(cout, 9 * c).contiguous())


@pytest.mark.parametrize("n,h,c,cout,res", [(2, 56, 64, 64, True), (2, 28, 128, 128, False),
                                            (3, 14, 256, 256, True), (2, 7, 512, 512, True),
                                            (1, 7, 64, 128, False), (64, 56, 64, 64, True),
                                            (64, 28, 128, 128, True), (64, 7, 512, 512, True)])
def test_span_conv_vs_torch(n, h, c, cout, res):
    import torch
    from paper_2601_04250_b200 import _native as nat
    lib = nat.load()
    g = torch.Generator(device="cuda").manual_seed(n * h + c)
    x = torch.randn((n, c, h, h), device="cuda", generator=g).to(torch.float16)
    w = (torch.randn((cout, c, 3, 3), device="cuda", generator=g) / (9 * c) ** 0.5).to(torch.float16)
    b = torch.randn(cout, device="cuda", generator=g)
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, padding=1)
    xp = torch.zeros((n, h + 2, h + 2, c), dtype=torch.float16, device="cuda")
    xp[:, 1:-1, 1:-1] = x.permute(0, 2, 3, 1)
    rp = None
    if res:
        rp = torch.zeros((n, h + 2, h + 2, cout), dtype=torch.float16, device="cuda")
        rp[:, 1:-1, 1:-1] = torch.randn((n, h, h, cout), device="cuda", generator=g).to(torch.float16)
        ref = ref + rp[:, 1:-1, 1:-1].float().permute(0, 3, 1, 2)
    ref = torch.relu(ref)
    y = torch.full((n, h + 2, h + 2, cout), 7.0, dtype=torch.float16, device="cuda")
    y[0, 0] = 0  # the first (W+3) positions are never written: zero them like a fresh buffer
    y[0, 1, 0] = 0
    wk = pack_span_weights(w)
    nat.check("gg_conv3x3_padded", lib.gg_conv3x3_padded(
        nat.ptr(xp), n, h, h, c, nat.ptr(wk), cout, nat.ptr(b), nat.ptr(rp), 1, nat.ptr(y), None,
        nat.stream_ptr()))
    torch.cuda.synchronize()
    got = y[:, 1:-1, 1:-1].float().permute(0, 3, 1, 2)
    err = (got - ref).abs().max().item()
    assert err <= 2e-2 * max(1.0, ref.abs().max().item()), err
    # borders (except the never-written first W+3 positions) are zeros
    border = torch.ones((n, h + 2, h + 2), dtype=torch.bool, device="cuda")
    border[:, 1:-1, 1:-1] = False
    assert (y[border].float() == 0).all()


@pytest.mark.parametrize("n,h,c,cout", [(64, 7, 512, 512), (64, 14, 256, 256), (64, 28, 128, 128)])
def test_span_pair_stream_k(n, h, c, cout, monkeypatch):
    """CTA-pair span conv with stream-K over (pair tile, channel block) forced on and
    off: both match torch within the bf16 tolerance, and the stream-K result is
    bit-identical across runs (segments summed in k order, any arrival order)."""
    import torch
    from paper_2601_04250_b200 import _native as nat
    lib = nat.load()
    g = torch.Generator(device="cuda").manual_seed(n + h + c)
    x = torch.randn((n, c, h, h), device="cuda", generator=g).to(torch.float16)
    w = (torch.randn((cout, c, 3, 3), device="cuda", generator=g) / (9 * c) ** 0.5).to(torch.float16)
    b = torch.randn(cout, device="cuda", generator=g)
    xp = torch.zeros((n, h + 2, h + 2, c), dtype=torch.float16, device="cuda")
    xp[:, 1:-1, 1:-1] = x.permute(0, 2, 3, 1)
    rp = torch.zeros((n, h + 2, h + 2, cout), dtype=torch.float16, device="cuda")
    rp[:, 1:-1, 1:-1] = torch.randn((n, h, h, cout), device="cuda", generator=g).to(torch.float16)
    ref = torch.relu(torch.nn.functional.conv2d(x.float(), w.float(), b, padding=1) +
                     rp[:, 1:-1, 1:-1].float().permute(0, 3, 1, 2))
    wk = pack_span_weights(w)
    outs = []
    for mode in ("0", "1", "1"):
        monkeypatch.setenv("GG_SPAN_SK", mode)
        y = torch.zeros((n, h + 2, h + 2, cout), dtype=torch.float16, device="cuda")
        nat.check("gg_conv3x3_padded", lib.gg_conv3x3_padded(
            nat.ptr(xp), n, h, h, c, nat.ptr(wk), cout, nat.ptr(b), nat.ptr(rp), 1, nat.ptr(y), None,
            nat.stream_ptr()))
        outs.append(y)
    torch.cuda.synchronize()
    scale = max(1.0, ref.abs().max().item())
    for y in outs:
        got = y[:, 1:-1, 1:-1].float().permute(0, 3, 1, 2)
        assert (got - ref).abs().max().item() <= 2e-2 * scale
    assert torch.equal(outs[1], outs[2])
