"""The MLA attention stand-in of the prefetch window (attention.py): causal
attention within each back-to-back sequence, RoPE positions restarting per
sequence, against an fp32 restatement with an explicit block-causal mask."""
import math

import pytest
import torch

from paper_2604_01621_b200.attention import MlaAttention

pytestmark = pytest.mark.gpu


def test_mla_matches_fp32_block_causal():
    dev = torch.device("cuda:0")
    m = MlaAttention(dev, seed=3, hidden=512, heads=4, q_lora=256, kv_lora=128, nope=32, rope=16, v_dim=32)
    seqs = [100, 57, 143]
    T = sum(seqs)
    x = (torch.randn(T, 512, device=dev) * 0.5).to(torch.bfloat16)
    y = m.forward(x, seqs).float()
    # fp32 reference
    f = lambda w: w.float()  # noqa: E731
    xf = x.float()

    def rms(v):
        return v * torch.rsqrt(v.pow(2).mean(-1, keepdim=True) + 1e-6)

    H, nope, rope, vd = 4, 32, 16, 32
    q = (rms(xf @ f(m.wq_a).T) @ f(m.wq_b).T).view(T, H, nope + rope)
    kva = xf @ f(m.wkv_a).T
    kv = (rms(kva[:, :128]) @ f(m.wkv_b).T).view(T, H, nope + vd)
    pos = torch.cat([torch.arange(L, device=dev) for L in seqs]).float()
    ang = pos[:, None] * m.inv_freq[None, :]
    c, s = torch.cos(ang), torch.sin(ang)

    def rot(v, c, s):
        a, b = v[..., 0::2], v[..., 1::2]
        return torch.stack((a * c - b * s, a * s + b * c), -1).flatten(-2)

    qr = rot(q[..., nope:], c[:, None], s[:, None])
    kr = rot(kva[:, 128:], c, s)
    qq = torch.cat((q[..., :nope], qr), -1)
    kk = torch.cat((kv[..., :nope], kr[:, None].expand(T, H, rope)), -1)
    vv = kv[..., nope:]
    seg = torch.cat([torch.full((L,), i, device=dev) for i, L in enumerate(seqs)])
    idx = torch.arange(T, device=dev)
    mask = (seg[:, None] == seg[None, :]) & (idx[None, :] <= idx[:, None])
    att = torch.einsum("thd,shd->hts", qq, kk) / math.sqrt(nope + rope)
    att = att.masked_fill(~mask, float("-inf")).softmax(-1)
    o = torch.einsum("hts,shd->thd", att, vv).reshape(T, H * vd)
    ref = o @ f(m.wo).T
    err = float((y - ref).norm() / ref.norm())
    assert err < 2e-2, err
