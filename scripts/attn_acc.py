#!/usr/bin/env python
"""Accuracy of the native MLA block against the fp32 restatement of
tests/test_gpu_attention.py (normwise relative error), for the attention
variant the environment selects (DWDP_ATTN_PAIR, DWDP_ATTN_SF16)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2604_01621_b200.attention import MlaAttention  # noqa: E402
from test_gpu_attention import _reference, _rel  # noqa: E402

dev = torch.device("cuda:0")
out = {"env": {k: os.environ.get(k) for k in ("DWDP_ATTN_PAIR", "DWDP_ATTN_SF16")}}
for name, kw, seqs, kvl in (("ragged", dict(hidden=512, heads=4, q_lora=256, kv_lora=128), [100, 57, 143, 300, 1, 129], 128),
                            ("long", dict(hidden=1024, heads=16, q_lora=512, kv_lora=256), [4096], 256)):
    m = MlaAttention(dev, seed=11, **kw)
    x = (torch.randn(sum(seqs), kw["hidden"], device=dev) * 0.5).to(torch.bfloat16)
    y = m.forward(x, seqs)
    torch.cuda.synchronize()
    out[name] = _rel(y.float(), _reference(m, x, seqs, kvl))
    m.close()
print(json.dumps(out))
