"""Quick device-time probe of the hot kernels (CUDA events; not a bench number)."""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def timeit(fn, iters=20, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def graph_time(fn, iters=20):
    """Device time per call of fn replayed from a CUDA graph (no host overhead)."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s), torch.no_grad():
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    return timeit(lambda: g.replay(), iters=iters)


def main():
    from paper_2601_04250_b200 import _native
    from paper_2601_04250_b200.distilbert import DistilBertB200, random_model as dmodel
    from paper_2601_04250_b200.resnet18 import ResNet18B200, random_model as rmodel

    out = {}
    lib = _native.load()
    # GEMM at DistilBERT shapes
    for (M, N, K) in [(16384, 2304, 768), (16384, 768, 768), (16384, 3072, 768), (16384, 768, 3072),
                      (8192, 8192, 8192)]:
        A = torch.randn((M, K), device="cuda").to(torch.bfloat16)
        B = torch.randn((N, K), device="cuda").to(torch.bfloat16)
        D = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)

        def run():
            lib.gg_gemm_bf16(_native.ptr(A), K, _native.ptr(B), K, _native.ptr(D), N, M, N, K, None,
                             None, 0, 0, 0, _native.stream_ptr())
        ms = timeit(run)
        out[f"gemm_{M}x{N}x{K}"] = {"ms": ms, "tflops": 2 * M * N * K / ms / 1e9}
        ms_t = timeit(lambda: torch.matmul(A, B.t()))
        out[f"gemm_{M}x{N}x{K}"]["torch_tflops"] = 2 * M * N * K / ms_t / 1e9
    # full forwards
    dm = dmodel(0)
    net = DistilBertB200(dm, max_batch=128)
    ids = torch.randint(0, 30522, (128, 128), device="cuda", dtype=torch.int32)
    ms = graph_time(lambda: net.forward(ids, stream=torch.cuda.current_stream()))
    out["distilbert_b128_graph"] = {"ms": ms, "tflops": net.flops(128) / ms / 1e9}
    # the same model in PyTorch (transformers eager, bf16, SDPA attention: cuBLAS + fused
    # attention kernels), graph-captured so host overhead is excluded
    hf = dm.cuda().to(torch.bfloat16).eval()
    ids64 = ids.long()
    with torch.no_grad():
        for _ in range(3):
            hf(input_ids=ids64)
    ms_hf = graph_time(lambda: hf(input_ids=ids64))
    out["torch_distilbert_b128_bf16_graph"] = {"ms": ms_hf, "tflops": net.flops(128) / ms_hf / 1e9,
                                               "attn_impl": getattr(hf.config, "_attn_implementation", None)}
    del hf
    rm = rmodel(0)
    rnet = ResNet18B200(rm, max_batch=64)
    x = torch.randn((64, 3, 224, 224), device="cuda")
    ms = graph_time(lambda: rnet.forward(x, stream=torch.cuda.current_stream()))
    out["resnet18_b64_graph"] = {"ms": ms, "tflops": rnet.flops(64) / ms / 1e9}
    torch.backends.cudnn.benchmark = True   # cuDNN autotuned algorithms
    rm = rm.cuda().to(memory_format=torch.channels_last).half()
    with torch.no_grad():
        xh = x.half().to(memory_format=torch.channels_last)
        ms = graph_time(lambda: rm(xh))
    out["torch_resnet18_b64_fp16_graph"] = {"ms": ms, "tflops": rnet.flops(64) / ms / 1e9}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
