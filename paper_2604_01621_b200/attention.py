"""DeepSeek-V3/R1 MLA prefill block as the attention step of the DWDP prefetch
window.

The paper hides the pull of layer l+1's experts behind MoE(l) + Attention(l+1)
(PAPER.md:168-171); the reference models attention only as cost entries
(`attention_entries`, src/modelspec.cpp:38-55). It runs on the compute stream
between the MoE layers, so the one-sided prefetch the runtime issued at
MoE(l)'s gate overlaps it exactly as in the paper's schedule.

backend="native" (default): the block through libdwdp.so's C-ABI
(dwdp_mla_forward) on sm_100a kernels only -- the five projections on the
tcgen05 grouped-GEMM kernel, RMSNorm / RoPE / K-V assembly kernels and the
tcgen05 causal flash-attention core (csrc/attn_sm100.cu); qk 128 + 64, v 128.
backend="library": the same block from library ops (cuBLAS through
torch.matmul, FlashAttention-2), kept as the comparison arm.

Shapes (DeepSeek-V3 config): hidden 7168, 128 heads, q_lora_rank 1536,
kv_lora_rank 512, qk_nope 128, qk_rope 64, v_head 128. Weights are random
(seeded) bf16. Per token it costs 2 * (h*1536 + 1536*128*192 + h*576 +
512*128*256 + 128*128*h) FLOP of projections (~0.37 GFLOP) plus causal
attention 2 * 128 * L/2 * (192 + 128) per token of an L-token sequence.
"""
from __future__ import annotations

import math

try:  # library attention kernel (FlashAttention-2 wheel in this image)
    from flash_attn import flash_attn_func as _flash
except Exception:  # noqa: BLE001
    _flash = None


class MlaAttention:
    def __init__(self, device, seed: int = 0, hidden: int = 7168, heads: int = 128,
                 q_lora: int = 1536, kv_lora: int = 512, nope: int = 128, rope: int = 64,
                 v_dim: int = 128, theta: float = 10000.0, backend: str = "native"):
        import torch

        assert backend in ("native", "library"), backend
        self.backend, self.device, self.theta = backend, device, theta
        self._handle, self._cap = None, 0
        self.h, self.H, self.nope, self.rope, self.v = hidden, heads, nope, rope, v_dim
        self.kv_lora = kv_lora
        g = torch.Generator(device=device).manual_seed(seed)

        def w(o, i):
            return (torch.randn(o, i, generator=g, device=device) / math.sqrt(i)).to(torch.bfloat16)

        self.wq_a = w(q_lora, hidden)
        self.wq_b = w(heads * (nope + rope), q_lora)
        self.wkv_a = w(kv_lora + rope, hidden)
        self.wkv_b = w(heads * (nope + v_dim), kv_lora)
        self.wo = w(hidden, heads * v_dim)
        self.inv_freq = 1.0 / (theta ** (torch.arange(0, rope, 2, device=device, dtype=torch.float32) / rope))
        # native backend: kv_a rows zero-padded to a multiple of 256 (GEMM n-blocks)
        rows = (kv_lora + rope + 255) // 256 * 256
        self.wkv_a_pad = torch.zeros((rows, hidden), dtype=torch.bfloat16, device=device)
        self.wkv_a_pad[:kv_lora + rope] = self.wkv_a

    def close(self) -> None:
        if self._handle is not None:
            from ._lib import check, lib
            check(lib().dwdp_mla_destroy(self._handle))
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def _native(self, x, seqs):
        import ctypes as C

        import numpy as np
        import torch

        from ._lib import MlaConfigC, MlaWeightsC, check, lib
        T = x.shape[0]
        if self._handle is None or T > self._cap:
            self.close()
            cap = max(T, 128)
            cfg = MlaConfigC(self.h, self.H, self.wq_a.shape[0], self.kv_lora, self.nope, self.rope, self.v,
                             x.device.index or 0, cap, self.theta,
                             1.0 / math.sqrt(self.nope + self.rope))
            h = C.c_void_p()
            check(lib().dwdp_mla_create(C.byref(cfg), C.byref(h)))
            self._handle, self._cap = h, cap
        w = MlaWeightsC(self.wq_a.data_ptr(), self.wq_b.data_ptr(), self.wkv_a_pad.data_ptr(),
                        self.wkv_b.data_ptr(), self.wo.data_ptr())
        y = torch.empty((T, self.h), dtype=torch.bfloat16, device=x.device)
        sl = np.ascontiguousarray(seqs, dtype=np.int64)
        x = x.contiguous()
        check(lib().dwdp_mla_forward(self._handle, C.byref(w), x.data_ptr(), T, sl.ctypes.data, len(sl),
                                     y.data_ptr(), torch.cuda.current_stream().cuda_stream))
        return y

    def flops(self, seqs: list[int]) -> float:
        """Algorithmic FLOP of forward() over sequences of these lengths."""
        T = sum(seqs)
        proj = 2.0 * T * (self.h * self.wq_a.shape[0] + self.wq_a.shape[0] * self.wq_b.shape[0]
                          + self.h * self.wkv_a.shape[0] + self.kv_lora * self.wkv_b.shape[0]
                          + self.H * self.v * self.h)
        att = sum(2.0 * self.H * (L * (L + 1) / 2) * (self.nope + self.rope + self.v) for L in seqs)
        return proj + att

    @staticmethod
    def _rms(x, eps: float = 1e-6):
        import torch
        xf = x.float()
        return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).to(x.dtype)

    def _rope(self, x, pos):
        import torch
        ang = pos[:, None].float() * self.inv_freq[None, :]  # [T, rope/2]
        c, s = torch.cos(ang), torch.sin(ang)
        if x.dim() == 3:
            c, s = c[:, None, :], s[:, None, :]
        x1, x2 = x[..., 0::2].float(), x[..., 1::2].float()
        return torch.stack((x1 * c - x2 * s, x1 * s + x2 * c), dim=-1).flatten(-2).to(x.dtype)

    def forward(self, x, seqs: list[int]):
        """x [T, hidden] bf16 of sum(seqs) tokens (sequences back to back) ->
        attention output [T, hidden] bf16 (no residual)."""
        import torch
        import torch.nn.functional as F

        if self.backend == "native":
            return self._native(x, seqs)
        T, H = x.shape[0], self.H
        q = (self._rms(x @ self.wq_a.T) @ self.wq_b.T).view(T, H, self.nope + self.rope)
        kva = x @ self.wkv_a.T
        ckv, kr = kva[:, :self.kv_lora], kva[:, self.kv_lora:]
        kv = (self._rms(ckv) @ self.wkv_b.T).view(T, H, self.nope + self.v)
        pos = torch.cat([torch.arange(L, device=x.device) for L in seqs])
        q = torch.cat((q[..., :self.nope], self._rope(q[..., self.nope:], pos)), dim=-1)
        kr = self._rope(kr, pos)
        k = torch.cat((kv[..., :self.nope], kr[:, None, :].expand(T, H, self.rope)), dim=-1)
        # one head dim for q, k and v (v zero-padded to 192) keeps attention on
        # the fused flash kernels
        v = F.pad(kv[..., self.nope:], (0, self.nope + self.rope - self.v))
        out = torch.empty((T, H, self.v), dtype=x.dtype, device=x.device)
        s = 0
        for L in seqs:
            if _flash is not None:  # FlashAttention-2 (~296 TFLOP/s at head dim 192 on B200)
                o = _flash(q[s:s + L].unsqueeze(0), k[s:s + L].unsqueeze(0), v[s:s + L].unsqueeze(0),
                           causal=True)[0]
            else:
                from torch.nn.attention import SDPBackend, sdpa_kernel
                with sdpa_kernel(SDPBackend.FLASH_ATTENTION):
                    o = F.scaled_dot_product_attention(
                        q[s:s + L].transpose(0, 1).unsqueeze(0), k[s:s + L].transpose(0, 1).unsqueeze(0),
                        v[s:s + L].transpose(0, 1).unsqueeze(0), is_causal=True)[0].transpose(0, 1)
            out[s:s + L] = o[..., :self.v]
            s += L
        return out.view(T, H * self.v) @ self.wo.T


def split_sequences(tokens: int, requests: int) -> list[int]:
    """The rank's tokens as `requests` back-to-back sequences of near-equal
    length (RankBatch::mean_seq_len, workload.hpp:45-55)."""
    n = max(1, min(requests, tokens)) if tokens > 0 else 0
    if n == 0:
        return []
    base, rem = divmod(tokens, n)
    return [base + (1 if i < rem else 0) for i in range(n)]
