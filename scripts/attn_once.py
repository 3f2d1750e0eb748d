#!/usr/bin/env python
"""One MLA block forward at DeepSeek-V3 shapes (4 x 8192-token sequences) for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_01621_b200.attention import MlaAttention  # noqa: E402

dev = torch.device("cuda:0")
m = MlaAttention(dev, seed=7)
seqs = [8192] * 4
x = (torch.randn(sum(seqs), 7168, device=dev) * 0.5).to(torch.bfloat16)
for _ in range(2):
    m.forward(x, seqs)
torch.cuda.synchronize()
m.close()
print("ok")
