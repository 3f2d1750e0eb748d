"""Host-side pieces of the attention window (no GPU): request splitting and
the FLOP count the bench reports."""
import torch

from paper_2604_01621_b200.attention import MlaAttention, split_sequences


def test_split_sequences():
    assert split_sequences(10, 3) == [4, 3, 3]
    assert split_sequences(5, 0) == [5]
    assert split_sequences(0, 4) == []
    assert sum(split_sequences(32768, 4)) == 32768


def test_mla_flops_formula():
    m = MlaAttention(torch.device("cpu"), hidden=512, heads=4, q_lora=256, kv_lora=128, nope=32, rope=16,
                     v_dim=32)
    L = 100
    proj = 2 * L * (512 * 256 + 256 * 4 * 48 + 512 * 144 + 128 * 4 * 64 + 4 * 32 * 512)
    att = 2 * 4 * (L * (L + 1) / 2) * (32 + 16 + 32)
    assert m.flops([L]) == proj + att
