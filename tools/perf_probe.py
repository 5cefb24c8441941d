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
    ms = timeit(lambda: net.forward(ids))
    out["distilbert_b128"] = {"ms": ms, "tflops": net.flops(128) / ms / 1e9}
    rm = rmodel(0)
    rnet = ResNet18B200(rm, max_batch=64)
    x = torch.randn((64, 3, 224, 224), device="cuda")
    ms = timeit(lambda: rnet.forward(x))
    out["resnet18_b64"] = {"ms": ms, "tflops": rnet.flops(64) / ms / 1e9}
    rm = rm.cuda().to(memory_format=torch.channels_last).half()
    with torch.no_grad():
        xh = x.half().to(memory_format=torch.channels_last)
        ms = timeit(lambda: rm(xh))
    out["torch_resnet18_b64_fp16"] = {"ms": ms}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
