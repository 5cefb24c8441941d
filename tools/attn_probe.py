"""Attention kernel alone at the DistilBERT b128 shape (probe, not a bench value).

    python tools/attn_probe.py [reps]        (GG_ATTN_SIMPLE=1: the per-item kernel)

Times gg_attention over a resident qkv buffer with CUDA events (graph of reps
launches), prints us/launch and the achieved DRAM-equivalent bandwidth of its
algorithmic traffic (qkv read 75.5 MB + ctx write 25.2 MB), next to a plain
device copy of the same byte count.
"""

import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2601_04250_b200 import _native  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    lib = _native.load()
    B, H, S, D = 128, 12, 128, 64
    qkv = (torch.randn(3 * B * H * S * D, device="cuda") * 0.5).to(torch.bfloat16)
    ctx = torch.empty((B * S, H * D), device="cuda", dtype=torch.bfloat16)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def attn():
        _native.check("gg_attention", lib.gg_attention(_native.ptr(qkv), None, _native.ptr(ctx), H * D, B,
                                                       H, S, None, _native.stream_ptr()))

    def attn_cold():
        flush.zero_()
        attn()
    nbytes = qkv.numel() * 2 + ctx.numel() * 2
    us = timed(attn, reps)
    us_flush = timed(flush.zero_, reps)
    us_cold = timed(attn_cold, reps) - us_flush
    src = torch.empty(nbytes // 2, dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    us_copy = timed(lambda: dst.copy_(src), reps)
    print(f"attention ({'simple' if os.environ.get('GG_ATTN_SIMPLE') else 'persistent'}): "
          f"{us:.2f} us warm-L2, {us_cold:.2f} us after a 256 MB L2 flush; "
          f"{nbytes / us / 1e3:.0f} / {nbytes / us_cold / 1e3:.0f} GB/s algorithmic; "
          f"copy of the same bytes {us_copy:.2f} us ({nbytes / us_copy / 1e3:.0f} GB/s)")


if __name__ == "__main__":
    main()
