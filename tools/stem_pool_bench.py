"""Device time of gg_stem_pool_span alone (batch 64, 224^2) under GG_STEMPOOL_DBG experiment bits.

    python tools/stem_pool_bench.py [dbg ...]
Not a bench number."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402


def main():
    from paper_2601_04250_b200 import _native as nat
    lib = nat.load()
    n, hs = int(os.environ.get("N", "64")), 112
    x16 = torch.randn(((n * (hs + 3) * (hs + 3)), 16), device="cuda").to(torch.bfloat16)
    w = (torch.randn((64, 256), device="cuda") * 0.05).to(torch.bfloat16)
    b = torch.randn(64, device="cuda")
    ho = hs // 2
    out = torch.zeros(((ho + 2) + n * (ho + 1) * (ho + 1), 64), dtype=torch.bfloat16, device="cuda")
    for dbg in (sys.argv[1:] or ["0"]):
        os.environ["GG_STEMPOOL_DBG"] = dbg
        def run():
            nat.check("gg_stem_pool_span", lib.gg_stem_pool_span(
                nat.ptr(x16), n, hs, hs, nat.ptr(w), 64, nat.ptr(b), nat.ptr(out), 2, None, None))
        for _ in range(5):
            run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(50):
            run()
        e1.record()
        torch.cuda.synchronize()
        print(f"dbg {dbg}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")


if __name__ == "__main__":
    main()
