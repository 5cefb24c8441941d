"""DistilBERT forward (tcgen05 GEMMs + attention + LN) vs transformers eager fp32.

Tolerance: the north star's 2e-2 for the bf16 path, on the logits; the
attention and LayerNorm kernels are also checked alone against fp32 torch.
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


def test_attention_kernel(env):
    torch, nat, lib = env
    B, H, S, D = 3, 12, 128, 64
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((B, H, S, D), device="cuda", generator=g)
    k = torch.randn((B, H, S, D), device="cuda", generator=g)
    v = torch.randn((B, H, S, D), device="cuda", generator=g)
    mask = torch.ones((B, S), dtype=torch.int32, device="cuda")
    mask[1, 100:] = 0
    qkv = torch.empty(3 * B * H * S * D, dtype=torch.bfloat16, device="cuda")
    plane = B * H * S * D
    qb, kb, vb = q.to(torch.bfloat16), k.to(torch.bfloat16), v.to(torch.bfloat16)
    qkv[:plane] = qb.flatten()
    qkv[plane:2 * plane] = kb.flatten()
    qkv[2 * plane:] = vb.transpose(2, 3).contiguous().flatten()
    ctx = torch.empty((B * S, H * D), dtype=torch.bfloat16, device="cuda")
    nat.check("gg_attention", lib.gg_attention(nat.ptr(qkv), nat.ptr(mask), nat.ptr(ctx), H * D,
                                               B, H, S, None, nat.stream_ptr()))
    s = qb.float() @ kb.float().transpose(2, 3)
    s = s.masked_fill(mask[:, None, None, :] == 0, float("-inf"))
    ref = torch.softmax(s, dim=-1) @ vb.float()
    ref = ref.transpose(1, 2).reshape(B * S, H * D)
    err = (ctx.float() - ref).abs().max().item()
    assert err < 2e-2, err


def test_layernorm_kernel(env):
    torch, nat, lib = env
    x = torch.randn((1000, 768), device="cuda").to(torch.bfloat16)
    gmm = torch.randn(768, device="cuda")
    bta = torch.randn(768, device="cuda")
    y = torch.empty_like(x)
    nat.check("gg_layernorm", lib.gg_layernorm(nat.ptr(x), 768, nat.ptr(y), 768, nat.ptr(gmm),
                                               nat.ptr(bta), 1000, 768, C.c_float(1e-12),
                                               None, 1, nat.stream_ptr()))
    ref = torch.nn.functional.layer_norm(x.float(), (768,), gmm, bta, 1e-12)
    # bf16 output: one rounding of |y| (half an ulp = 2^-9 relative) plus fp32 statistics
    assert ((y.float() - ref).abs() <= 4e-3 * ref.abs() + 1e-2).all()


@pytest.mark.parametrize("batch", [4, 128])
def test_distilbert_logits_vs_eager(env, batch):
    torch = env[0]
    from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
    model = random_model(0)
    ids = torch.randint(0, model.config.vocab_size, (batch, 128), generator=torch.Generator().manual_seed(1))
    mask = torch.ones((batch, 128), dtype=torch.int64)
    if batch > 2:
        mask[2, 64:] = 0
    with torch.no_grad():
        ref = model.cuda()(input_ids=ids.cuda(), attention_mask=mask.cuda()).logits.float()
    net = DistilBertB200(model, max_batch=batch)
    out = net.forward(ids.to(torch.int32).cuda(), mask.to(torch.int32).cuda())
    torch.cuda.synchronize()
    err = (out - ref).abs().max().item()
    print(f"distilbert b={batch}: max |logit err| = {err:.3e}, |ref| max {ref.abs().max().item():.3f}")
    assert err <= 2e-2, err


@pytest.mark.parametrize("fold", [True, False])
def test_distilbert_layernorm_folding(env, fold, monkeypatch):
    """b = 32 (M = 4096, the CTA-pair path): the LayerNorm-folded encoder
    (gg_gemm_ln: row statistics partials, W diag(gamma) + column-sum correction,
    LayerNorm'd residual on the fly) and the LayerNorm-kernel encoder both match
    transformers eager fp32 within the bf16 bound; with a key mask."""
    torch = env[0]
    from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
    monkeypatch.setenv("GG_LN_UNFUSED", "0" if fold else "1")
    model = random_model(0)
    ids = torch.randint(0, model.config.vocab_size, (32, 128), generator=torch.Generator().manual_seed(3))
    mask = torch.ones((32, 128), dtype=torch.int64)
    mask[5, 100:] = 0
    with torch.no_grad():
        ref = model.cuda()(input_ids=ids.cuda(), attention_mask=mask.cuda()).logits.float()
    net = DistilBertB200(model, max_batch=32)
    assert net.fused_ln == fold
    out = net.forward(ids.to(torch.int32).cuda(), mask.to(torch.int32).cuda())
    torch.cuda.synchronize()
    err = (out - ref).abs().max().item()
    print(f"distilbert b=32 fold={fold}: max |logit err| = {err:.3e}")
    assert err <= 2e-2, err


def test_distilbert_dependency_chain(env):
    """Tile-level dependencies (gg_dep) between the encoder's kernels produce the
    same logits bit for bit as grid-wide waits, at the full batch and at a
    dynamic count (the counters of units beyond the count are never awaited),
    over repeated forwards (counters re-zeroed per forward), inside a CUDA graph."""
    torch = env[0]
    from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
    model = random_model(0)
    ids = torch.randint(0, model.config.vocab_size, (128, 128),
                        generator=torch.Generator().manual_seed(5)).to(torch.int32).cuda()
    mask = torch.ones((128, 128), dtype=torch.int32, device="cuda")
    mask[7, 90:] = 0
    net = DistilBertB200(model, max_batch=128)
    assert net.fused_ln
    outs = {}
    for use in (False, True):
        net.use_deps = use
        for cnt in (128, 45):
            count = torch.tensor([cnt], dtype=torch.int32, device="cuda")
            for _ in range(3):
                out = net.forward(ids, mask, count=count).clone()
            outs[(use, cnt)] = out
    torch.cuda.synchronize()
    for cnt in (128, 45):
        assert torch.equal(outs[(True, cnt)][:cnt], outs[(False, cnt)][:cnt])
    # the captured graph replays the chain (memset node + kernels) identically
    net.use_deps = True
    count = torch.tensor([128], dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        net.forward(ids, mask, count=count, stream=s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            gout = net.forward(ids, mask, count=count, stream=s)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(gout, outs[(True, 128)])


def test_distilbert_fused_ffn(env):
    """gg_ffn_pair (lin1 + GELU and lin2 + residual in one persistent kernel, one
    tile queue, per-unit readiness) gives the same logits bit for bit as the two
    GEMM launches, at the full batch and at a dynamic count, and inside a graph."""
    torch = env[0]
    from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
    model = random_model(0)
    ids = torch.randint(0, model.config.vocab_size, (128, 128),
                        generator=torch.Generator().manual_seed(8)).to(torch.int32).cuda()
    mask = torch.ones((128, 128), dtype=torch.int32, device="cuda")
    mask[3, 70:] = 0
    net = DistilBertB200(model, max_batch=128)
    outs = {}
    for fused in (False, True):
        net.use_ffn_fused = fused
        for cnt in (128, 37):
            count = torch.tensor([cnt], dtype=torch.int32, device="cuda")
            for _ in range(2):
                out = net.forward(ids, mask, count=count).clone()
            outs[(fused, cnt)] = out
    torch.cuda.synchronize()
    for cnt in (128, 37):
        assert torch.equal(outs[(True, cnt)][:cnt], outs[(False, cnt)][:cnt])
    net.use_ffn_fused = True
    count = torch.tensor([128], dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        net.forward(ids, mask, count=count, stream=s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            gout = net.forward(ids, mask, count=count, stream=s)
    for _ in range(4):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(gout, outs[(True, 128)])


@pytest.mark.parametrize("batch", [4, 128])
def test_distilbert_fused_head(env, batch):
    """gg_cls_head (CLS LayerNorm + pre_classifier + ReLU + classifier in one launch)
    agrees with the three-launch head (LayerNorm kernel + two tcgen05 GEMMs) within
    the bf16 rounding of the pooled activation, is deterministic (fixed-order
    column-block reduction), honours a dynamic count that ends inside a 16-row
    block, and replays inside a CUDA graph (arrival counters re-zeroed)."""
    torch = env[0]
    from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
    model = random_model(0)
    ids = torch.randint(0, model.config.vocab_size, (batch, 128),
                        generator=torch.Generator().manual_seed(9)).to(torch.int32).cuda()
    mask = torch.ones((batch, 128), dtype=torch.int32, device="cuda")
    mask[1, 50:] = 0
    net = DistilBertB200(model, max_batch=batch)
    cnts = (batch, 37) if batch > 37 else (batch, 3)
    outs = {}
    for fused in (False, True):
        net.fused_head = fused
        for cnt in cnts:
            count = torch.tensor([cnt], dtype=torch.int32, device="cuda")
            outs[(fused, cnt)] = [net.forward(ids, mask, count=count).clone() for _ in range(2)]
    torch.cuda.synchronize()
    for cnt in cnts:
        a, b = outs[(True, cnt)], outs[(False, cnt)]
        assert torch.equal(a[0][:cnt], a[1][:cnt])
        err = (a[0][:cnt] - b[0][:cnt]).abs().max().item()
        print(f"fused head b={batch} count={cnt}: max |logit diff| vs 3-launch head = {err:.3e}")
        assert err <= 1e-2, err
    net.fused_head = True
    count = torch.tensor([batch], dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        net.forward(ids, mask, count=count, stream=s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            gout = net.forward(ids, mask, count=count, stream=s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(gout, outs[(True, batch)][0])
