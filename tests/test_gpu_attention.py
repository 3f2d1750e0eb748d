"""The MLA attention block of the prefetch window (attention.py): causal
attention within each back-to-back sequence, RoPE positions restarting per
sequence, against an fp32 restatement with an explicit block-causal mask.

backend="native" is the sm_100a path (dwdp_mla_forward: tcgen05 projections,
tcgen05 flash-attention core, glue kernels); backend="library" the
cuBLAS + FlashAttention-2 comparison arm. Tolerance: normwise relative error
2e-2 against fp32 (bf16 activations, bf16 P in the PV product)."""
import math

import pytest
import torch

from paper_2604_01621_b200.attention import MlaAttention

pytestmark = pytest.mark.gpu

TOL = 2e-2


def _reference(m, x, seqs, kv_lora):
    """fp32 MLA prefill with a block-causal mask (einsum, one head group at a time)."""
    dev = x.device
    T = x.shape[0]
    H, nope, rope, vd = m.H, m.nope, m.rope, m.v
    f = lambda w: w.float()  # noqa: E731
    xf = x.float()

    def rms(v):
        return v * torch.rsqrt(v.pow(2).mean(-1, keepdim=True) + 1e-6)

    # bf16 round trips where the device stores bf16 intermediates
    bf = lambda v: v.to(torch.bfloat16).float()  # noqa: E731
    qa = bf(xf @ f(m.wq_a).T)
    q = bf(bf(rms(qa)) @ f(m.wq_b).T).view(T, H, nope + rope)
    kva = bf(xf @ f(m.wkv_a).T)
    kv = bf(bf(rms(kva[:, :kv_lora])) @ f(m.wkv_b).T).view(T, H, nope + vd)
    pos = torch.cat([torch.arange(L, device=dev) for L in seqs]).float()
    ang = pos[:, None] * m.inv_freq[None, :]
    c, s = torch.cos(ang), torch.sin(ang)

    def rot(v, c, s):
        a, b = v[..., 0::2], v[..., 1::2]
        return torch.stack((a * c - b * s, a * s + b * c), -1).flatten(-2)

    qr = rot(q[..., nope:], c[:, None], s[:, None])
    kr = rot(kva[:, kv_lora:kv_lora + rope], c, s)
    qq = torch.cat((q[..., :nope], qr), -1)
    kk = torch.cat((kv[..., :nope], kr[:, None].expand(T, H, rope)), -1)
    vv = kv[..., nope:]
    seg = torch.cat([torch.full((L,), i, device=dev) for i, L in enumerate(seqs)])
    idx = torch.arange(T, device=dev)
    mask = (seg[:, None] == seg[None, :]) & (idx[None, :] <= idx[:, None])
    o = torch.empty((T, H, vd), device=dev)
    for h0 in range(0, H, 8):
        hs = slice(h0, min(H, h0 + 8))
        att = torch.einsum("thd,shd->hts", qq[:, hs], kk[:, hs]) / math.sqrt(nope + rope)
        att = att.masked_fill(~mask, float("-inf")).softmax(-1)
        o[:, hs] = torch.einsum("hts,shd->thd", att, vv[:, hs])
    return bf(o.reshape(T, H * vd)) @ f(m.wo).T


def _rel(a, b):
    return float((a - b).norm() / b.norm())


def test_library_arm_matches_fp32_block_causal():
    dev = torch.device("cuda:0")
    m = MlaAttention(dev, seed=3, hidden=512, heads=4, q_lora=256, kv_lora=128, nope=32, rope=16, v_dim=32,
                     backend="library")
    seqs = [100, 57, 143]
    x = (torch.randn(sum(seqs), 512, device=dev) * 0.5).to(torch.bfloat16)
    assert _rel(m.forward(x, seqs).float(), _reference(m, x, seqs, 128)) < TOL


@pytest.mark.parametrize("seqs", [[100, 57, 143, 300, 1, 129], [128], [1], [513, 64, 255]])
def test_native_mla_matches_fp32(seqs):
    """Ragged sequences: partial query tiles, keys past a sequence's end (the
    next sequence's rows) masked, single-token sequences."""
    dev = torch.device("cuda:0")
    m = MlaAttention(dev, seed=11, hidden=512, heads=4, q_lora=256, kv_lora=128)
    x = (torch.randn(sum(seqs), 512, device=dev) * 0.5).to(torch.bfloat16)
    y = m.forward(x, seqs)
    torch.cuda.synchronize()
    err = _rel(y.float(), _reference(m, x, seqs, 128))
    m.close()
    assert err < TOL, err


def test_native_mla_long_sequence_many_heads():
    """One 4096-token sequence (64 KV tiles for the last query tile, the
    3-stage K/V ring wraps many times) over 16 heads."""
    dev = torch.device("cuda:0")
    m = MlaAttention(dev, seed=5, hidden=1024, heads=16, q_lora=512, kv_lora=256)
    seqs = [4096]
    x = (torch.randn(4096, 1024, device=dev) * 0.5).to(torch.bfloat16)
    y = m.forward(x, seqs)
    torch.cuda.synchronize()
    err = _rel(y.float(), _reference(m, x, seqs, 256))
    m.close()
    assert err < TOL, err


def test_native_matches_library_at_r1_shapes():
    """DeepSeek-V3 shapes (hidden 7168, 128 heads, q_lora 1536, kv_lora 512):
    the sm_100a block and the library arm agree (same weights)."""
    dev = torch.device("cuda:0")
    m = MlaAttention(dev, seed=7)
    seqs = [1024, 700, 324]
    x = (torch.randn(sum(seqs), 7168, device=dev) * 0.5).to(torch.bfloat16)
    yn = m.forward(x, seqs).float()
    m.backend = "library"
    yl = m.forward(x, seqs).float()
    torch.cuda.synchronize()
    m.close()
    assert _rel(yn, yl) < TOL
