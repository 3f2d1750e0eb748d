#!/usr/bin/env python
"""Small-shape driver for compute-sanitizer runs (memcheck / racecheck /
synccheck / initcheck) of every kernel family the MoE path launches:

  bf16   router int8 GEMM + top-k, permute (count/scan/scatter + bulk copy),
         1-SM tcgen05 GEMM1+SwiGLU / GEMM2, combine
  pair   the same with the CTA-pair GEMMs (DWDP_GEMM_PAIR=1, cta_group::2)
  fp8    W8A8 e4m3 path (1-SM kind::f8f6f4 GEMMs, fp8 permute, row quantiser)
  nvfp4  W4A4 path (CTA-pair GEMM1 + 1-SM GEMM2, kind::mxf4nvf4, quantisers)
  dwdp   two DWDP ranks on one GPU: TMA pull kernel, copy-engine and hybrid
         plans, 4 layers across the double buffer, bitwise vs all-local

usage: compute-sanitizer --tool memcheck python scripts/sanitize_driver.py <case>
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2604_01621_b200 as D  # noqa: E402

MID = dict(num_layers=2, num_experts=64, hidden=1024, ffn=256, shared_ffn=256, top_k=6,
           n_group=8, topk_group=4, max_tokens=2048, weight_layers=2)


def x_of(T, h, seed):
    x = torch.empty((T, h), dtype=torch.bfloat16, device="cuda:0")
    D.fill_bf16(x, seed, 1.0)
    return x


def layer(cfg, Ts):
    c = D.DwdpContext(cfg)
    c.init_weights()
    for T in Ts:
        y = c.moe_forward(0, x_of(T, cfg.hidden, T))
        torch.cuda.synchronize()
        assert torch.isfinite(y.float()).all()
    c.close()


def main(case):
    if case == "bf16":
        layer(D.DwdpConfig.tiny(max_tokens=512), [1, 77, 300])
        layer(D.DwdpConfig(**MID), [5, 2000])
        a = torch.randn((300, 512), device="cuda:0").to(torch.bfloat16)
        b = torch.randn((256, 512), device="cuda:0").to(torch.bfloat16)
        D.gemm_bf16(a, b)
    elif case == "pair":
        os.environ["DWDP_GEMM_PAIR"] = "1"
        layer(D.DwdpConfig(**MID), [2000])
    elif case == "fp8":
        layer(D.DwdpConfig(**MID, weight_dtype=D.WEIGHT_FP8), [7, 2000])
    elif case == "nvfp4":
        layer(D.DwdpConfig(**MID, weight_dtype=D.WEIGHT_NVFP4), [7, 2000])
    elif case == "dwdp":
        full = D.DwdpContext(D.DwdpConfig(**MID))
        full.init_weights()
        for eng in (D.ENGINE_PULL, D.ENGINE_COPY, D.ENGINE_HYBRID):
            ranks = [D.DwdpContext(D.DwdpConfig(**MID, rank=r, group_size=2, engine=eng,
                                                slice_size=1 << 18)) for r in range(2)]
            for c in ranks:
                c.init_weights()
            D.DwdpContext.link_local(ranks)
            xs = [x_of(150 + 50 * r, MID["hidden"], r) for r in range(2)]
            for g in range(4):
                for r in range(2):
                    y = ranks[r].layer_forward(g, xs[r], residual=False)
                    torch.cuda.synchronize()
                    assert torch.equal(y, full.moe_forward(g % 2, xs[r])), (eng, g, r)
            for c in ranks:
                c.close()
        full.close()
    else:
        raise SystemExit(f"unknown case {case}")
    torch.cuda.synchronize()
    print(f"case {case} ok")


if __name__ == "__main__":
    main(sys.argv[1])
