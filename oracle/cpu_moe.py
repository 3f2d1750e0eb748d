"""ORACLE / TEST INFRASTRUCTURE ONLY — the CPU restatement of the MoE layer,
run with resident bf16 weights on all host cores. bench.py times it as the
reported CPU baseline (cpu_baseline / --impl reference); it is never the
measured product path.

The reference repository has no numerical MoE; its only CPU
code on this path is the discrete-event simulator, whose wall time bench.py
reports alongside (oracle/_ref, ref_simulate)."""
from __future__ import annotations

import os
import time

import numpy as np

from . import oracle as O


class CpuMoeLayer:
    """One synthetic R1-shaped layer (same counter-hash weights as the GPU)."""

    def __init__(self, cfg: O.MoeConfig, seed: int, layer: int = 0, bias=None):
        self.o = O.oracle()
        self.cfg, self.seed, self.layer = cfg, seed, layer
        h, f, E = cfg.hidden, cfg.ffn, cfg.num_experts
        sc = float(np.float32(1) / np.sqrt(np.float32(h)))
        self.sf = float(np.float32(1) / np.sqrt(np.float32(f)))
        self.sh = sc
        self.w_router = self.o.fill_bf16(self.o.tensor_seed(seed, layer, E + 1, 0), E * h, sc)
        self.bias = bias
        self.gate = [None] * (E + 1)
        self.up = [None] * (E + 1)
        self.down = [None] * (E + 1)

    def _materialise(self, experts):
        h, f = self.cfg.hidden, self.cfg.ffn
        for e in experts:
            if self.gate[e] is not None:
                continue
            ts = lambda t: self.o.tensor_seed(self.seed, self.layer, int(e), t)  # noqa: E731
            self.gate[e] = self.o.fill_bf16(ts(0), f * h, self.sh)
            self.up[e] = self.o.fill_bf16(ts(1), f * h, self.sh)
            self.down[e] = self.o.fill_bf16(ts(2), h * f, self.sf)

    def prepare(self, x_bf16: np.ndarray, T: int):
        """Materialise the weights the sample touches (outside any timed region)."""
        _, idx, _ = self.o.route(self.cfg, x_bf16, T, self.w_router, self.bias)
        need = set(np.unique(idx).tolist())
        if self.cfg.shared_ffn:
            need.add(self.cfg.num_experts)
        self._materialise(sorted(need))

    def forward(self, x_bf16: np.ndarray, T: int, nthreads: int = 0):
        _, idx, _ = self.o.route(self.cfg, x_bf16, T, self.w_router, self.bias)
        missing = [e for e in np.unique(idx).tolist() if self.gate[e] is None]
        if missing:
            raise RuntimeError(f"experts {missing[:4]}... not materialised; call prepare()")
        return self.o.moe_forward_bf16w(self.cfg, x_bf16, T, self.w_router, self.bias, self.gate,
                                        self.up, self.down, nthreads)


def r1_config() -> O.MoeConfig:
    return O.MoeConfig(7168, 256, 8, 2048, 2048, 1, 8, 4, 1, 2.5)


def time_layer(tokens: int, layers: int, steps: int, warmup: int, seed: int = 2604_01621):
    """Tokens/s of the CPU MoE stack (L layers aliasing one weight set, as the
    GPU N=1 arm) over a bounded token sample; returns (tokens_per_s, cores, secs/step)."""
    cfg = r1_config()
    layer = CpuMoeLayer(cfg, seed)
    o = layer.o
    x = o.fill_bf16(0xC0FFEE, tokens * cfg.hidden, 1.0)
    layer.prepare(x, tokens)
    cores = os.cpu_count() or 1
    for _ in range(max(warmup, 1)):  # materialises every expert the stack touches
        h = x
        for _ in range(layers):
            layer.prepare(h, tokens)
            y, _, _ = layer.forward(h, tokens)
            h = O.bf16_round(O.bf16_to_f32(h).reshape(tokens, -1) + y).reshape(-1)
    t0 = time.perf_counter()
    for _ in range(steps):
        h = x
        for _ in range(layers):
            y, _, _ = layer.forward(h, tokens)
            h = O.bf16_round(O.bf16_to_f32(h).reshape(tokens, -1) + y).reshape(-1)
    dt = (time.perf_counter() - t0) / steps
    return tokens / dt, cores, dt
