"""The exact router (22-bit fixed point per row, exact integer dot products,
one fp32 rounding: DESIGN.md §4) against DeepSeek-V3 routing on float64
logits, on R1 shapes and the bench's own activations (counter hash 0xC0FFEE,
the R1 router weights of layer 0): the top-8 selections agree token for token
(with and without a noaux_tc selection bias)."""
import numpy as np
import pytest

import paper_2604_01621_b200 as D
from oracle import check as CK


@pytest.mark.parametrize("bias", [None, "zipf"])
def test_exact_router_agrees_with_fp64_routing(orc, bias):
    cfg = D.DwdpConfig(num_layers=1)
    oc = CK.moe_config(cfg)
    T = 2048
    x = orc.fill_bf16(0xC0FFEE, T * cfg.hidden, 1.0)
    sc = float(np.float32(1) / np.sqrt(np.float32(cfg.hidden)))
    wr = orc.fill_bf16(orc.tensor_seed(cfg.weight_seed, 0, cfg.num_experts + 1, 0), cfg.num_experts * cfg.hidden, sc)
    b = None if bias is None else (-0.04 * np.log(np.arange(cfg.num_experts) + 1.0)).astype(np.float32)
    _, idx, _ = orc.route(oc, x, T, wr, b)
    r = CK.fp64_agreement(oc, x, T, wr, idx, b)
    assert r["topk_set_mismatch_tokens"] == 0, r
    assert r["topk_order_mismatch_tokens"] == 0, r
