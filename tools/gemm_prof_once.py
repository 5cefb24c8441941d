"""One plain pair-GEMM launch per shape with GG_GEMM_PROF timelines (probe; not a bench).

    GG_GEMM_PROF=1 python tools/gemm_prof_once.py M N K [M N K ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402


def main():
    from paper_2601_04250_b200 import _native
    lib = _native.load()
    a = [int(x) for x in sys.argv[1:]]
    for i in range(0, len(a), 3):
        M, N, K = a[i:i + 3]
        A = torch.randn((M, K), device="cuda").to(torch.bfloat16)
        B = torch.randn((N, K), device="cuda").to(torch.bfloat16)
        D = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
        for _ in range(2):
            lib.gg_gemm_bf16(_native.ptr(A), K, _native.ptr(B), K, _native.ptr(D), N, M, N, K, None, None,
                             0, 0, 0, _native.stream_ptr())
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
