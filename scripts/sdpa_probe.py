"""Which fused attention path runs the MLA prefill shapes on this GPU, and how fast."""
import time

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

dev = torch.device("cuda:0")
H, L, D = 128, 8192, 192
q = torch.randn(1, H, L, D, device=dev, dtype=torch.bfloat16)
k = torch.randn_like(q)
v = torch.randn_like(q)
flops = 2 * H * L * L / 2 * (D + 128)


def bench(fn, name):
    try:
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 3
        print(f"{name}: {dt * 1e3:.2f} ms, {flops / dt / 1e12:.0f} TFLOP/s", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{name}: unavailable ({str(e)[:120]})", flush=True)


for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
    def f(be=be):
        with sdpa_kernel(be):
            return F.scaled_dot_product_attention(q, k, v, is_causal=True)
    bench(f, str(be))
try:
    from flash_attn import flash_attn_func
    qt, kt, vt = (t.transpose(1, 2).contiguous() for t in (q, k, v))
    bench(lambda: flash_attn_func(qt, kt, vt, causal=True), "flash_attn 2")
except Exception as e:  # noqa: BLE001
    print("flash_attn import failed", str(e)[:120])
