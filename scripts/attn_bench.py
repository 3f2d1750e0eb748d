#!/usr/bin/env python
"""MLA prefill block at DeepSeek-V3 shapes: the sm_100a path (dwdp_mla_forward)
vs the library arm (cuBLAS + FlashAttention-2), CUDA-event timed, same weights.
Prints one JSON line per (tokens, sequence length)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_01621_b200.attention import MlaAttention  # noqa: E402


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dev = torch.device("cuda:0")
    m = MlaAttention(dev, seed=7)
    for T, L in ((8192, 8192), (32768, 8192), (32768, 2048)):
        seqs = [L] * (T // L)
        x = (torch.randn(T, 7168, device=dev) * 0.5).to(torch.bfloat16)
        m.backend = "native"
        tn = timed(lambda: m.forward(x, seqs))
        m.backend = "library"
        tl = timed(lambda: m.forward(x, seqs))
        fl = m.flops(seqs)
        att = sum(2.0 * m.H * (l * (l + 1) / 2) * (m.nope + m.rope + m.v) for l in seqs)
        print(json.dumps({"tokens": T, "seq_len": L, "native_ms": tn, "library_ms": tl,
                          "native_tflops": fl / tn / 1e9, "library_tflops": fl / tl / 1e9,
                          "attention_core_share_of_flops": att / fl}), flush=True)
    m.close()


if __name__ == "__main__":
    main()
