"""tcgen05 GEMM (gg_gemm_bf16) vs a plain PyTorch fp32 reference of the same op."""

from __future__ import annotations

import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_2601_04250_b200 import _native
    return torch, _native, _native.load()


def run_gemm(env, A, B, bias=None, residual=None, act=0, tile_n=0):
    torch, nat, lib = env
    M, K = A.shape
    N = B.shape[0]
    D = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    rc = lib.gg_gemm_bf16(nat.ptr(A), A.stride(0), nat.ptr(B), B.stride(0), nat.ptr(D), D.stride(0),
                          M, N, K, nat.ptr(bias), nat.ptr(residual),
                          residual.stride(0) if residual is not None else 0, act, tile_n,
                          nat.stream_ptr())
    nat.check("gg_gemm_bf16", rc)
    return D


def reference(A, B, bias, residual, act):
    import torch
    y = A.float() @ B.float().t()
    if bias is not None:
        y = y + bias.float()
    if residual is not None:
        y = y + residual.float()
    if act == 1:
        y = torch.relu(y)
    elif act == 2:
        y = torch.nn.functional.gelu(y)
    return y


@pytest.mark.parametrize("M,N,K,tile_n", [
    (128, 256, 64, 256), (256, 256, 128, 256), (300, 512, 768, 0), (1000, 768, 768, 0),
    (16384, 2304, 768, 0), (16384, 768, 3072, 0), (4096, 3072, 768, 128), (513, 64, 1024, 64),
    (128, 32, 768, 64), (5000, 768, 768, 0), (4096, 512, 1536, 0)])
def test_gemm_shapes(env, M, N, K, tile_n):
    torch = env[0]
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn((M, K), device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn((N, K), device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    D = run_gemm(env, A, B, tile_n=tile_n)
    ref = reference(A, B, None, None, 0)
    torch.cuda.synchronize()
    err = (D.float() - ref).abs().max().item()
    # bf16 output rounding of O(1) values plus fp32 accumulation order: 2e-2 (north-star bf16 tolerance)
    assert err <= 2e-2 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("act", [0, 1, 2])
@pytest.mark.parametrize("M", [777, 4500])   # single-CTA tiles / CTA-pair tiles
def test_gemm_fused_epilogue(env, act, M):
    torch = env[0]
    g = torch.Generator(device="cuda").manual_seed(act)
    N, K = 768, 768
    A = torch.randn((M, K), device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn((N, K), device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda", generator=g)
    res = torch.randn((M, N), device="cuda", generator=g).to(torch.bfloat16)
    D = run_gemm(env, A, B, bias=bias, residual=res, act=act)
    ref = reference(A, B, bias, res, act)
    err = (D.float() - ref).abs().max().item()
    assert err <= 2e-2 * max(1.0, ref.abs().max().item()), err


def test_gemm_rejects_bad_shapes(env):
    torch, nat, lib = env
    A = torch.zeros((128, 100), dtype=torch.bfloat16, device="cuda")
    B = torch.zeros((64, 100), dtype=torch.bfloat16, device="cuda")
    D = torch.zeros((128, 64), dtype=torch.bfloat16, device="cuda")
    rc = lib.gg_gemm_bf16(nat.ptr(A), 100, nat.ptr(B), 100, nat.ptr(D), 64, 128, 64, 100,
                          None, None, 0, 0, 0, nat.stream_ptr())
    assert rc != 0


@pytest.mark.parametrize("M,N,K,act,res", [
    (16384, 768, 3072, 0, True), (16384, 768, 768, 0, True), (1000, 768, 768, 2, False),
    (300, 2304, 768, 1, True), (128, 256, 4096, 0, False), (16384, 3072, 768, 2, False)])
def test_gemm_stream_k(env, M, N, K, act, res):
    """Stream-K split of the (tile, k-block) space: same result as data-parallel
    tiles within bf16 rounding of a different fp32 summation order, vs the fp32
    reference at the bf16 tolerance, and bit-identical across runs (segments are
    summed in k order whatever order they arrive in)."""
    torch, nat, lib = env
    g = torch.Generator(device="cuda").manual_seed(M + N + K + act)
    A = torch.randn((M, K), device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn((N, K), device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda", generator=g)
    resid = torch.randn((M, N), device="cuda", generator=g).to(torch.bfloat16) if res else None
    assert lib.gg_streamk_reserve() == 0
    prev = lib.gg_streamk_mode(0)
    try:
        d_dp = run_gemm(env, A, B, bias=bias, residual=resid, act=act)
        lib.gg_streamk_mode(1)
        d_sk = run_gemm(env, A, B, bias=bias, residual=resid, act=act)
        d_sk2 = run_gemm(env, A, B, bias=bias, residual=resid, act=act)
    finally:
        lib.gg_streamk_mode(prev)
    torch.cuda.synchronize()
    ref = reference(A, B, bias, resid, act)
    scale = max(1.0, ref.abs().max().item())
    assert torch.equal(d_sk, d_sk2)
    assert (d_sk.float() - ref).abs().max().item() <= 2e-2 * scale
    assert (d_sk.float() - d_dp.float()).abs().max().item() <= 1e-2 * scale


def test_sm_reserve_grids_same_results(env):
    """gg_set_sm_reserve: validation (even, >= 0, below the SM count; returns the
    previous value) and persistent grids sized to the remaining SMs compute the same
    bits: a DistilBERT forward captured with 2 SMs reserved (the pipelined serving
    loop's setting) equals the full-grid forward exactly."""
    torch, nat, lib = env
    from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
    assert lib.gg_set_sm_reserve(3) == -1 and lib.gg_set_sm_reserve(-2) == -1
    assert lib.gg_set_sm_reserve(100000) == -1
    net = DistilBertB200(random_model(0), max_batch=64)
    ids = torch.randint(0, 30522, (64, 128), generator=torch.Generator().manual_seed(4)).to(torch.int32).cuda()
    full = net.forward(ids).clone()
    outs = []
    for reserve in (2, 4):
        prev = lib.gg_set_sm_reserve(reserve)
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    out = net.forward(ids, stream=s)
        finally:
            assert lib.gg_set_sm_reserve(prev) == reserve
        g.replay()
        torch.cuda.synchronize()
        outs.append(out.clone())
    for o in outs:
        assert torch.equal(o, full)
