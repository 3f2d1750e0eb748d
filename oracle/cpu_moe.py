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


def tiny_config() -> O.MoeConfig:
    """BASELINE config 1: h 512, E 16 top-2 softmax, f 1024."""
    return O.MoeConfig(512, 16, 2, 1024, 0, 0, 1, 1, 1, 1.0)


class CpuStack:
    """L layers aliasing one weight set (as the GPU N=1 arm), every expert
    materialised up front (outside timed regions)."""

    def __init__(self, cfg: O.MoeConfig, layers: int, seed: int = 2604_01621):
        self.layer = CpuMoeLayer(cfg, seed)
        self.layer._materialise(range(cfg.num_experts + (1 if cfg.shared_ffn else 0)))
        self.cfg, self.layers, self.o = cfg, layers, self.layer.o

    def input(self, T: int) -> np.ndarray:
        return self.o.fill_bf16(0xC0FFEE, T * self.cfg.hidden, 1.0)

    def forward(self, x: np.ndarray, T: int, layers: int | None = None) -> np.ndarray:
        h = x
        for _ in range(self.layers if layers is None else layers):
            y, _, _ = self.layer.forward(h, T)
            h = O.bf16_round(O.bf16_to_f32(h).reshape(T, -1) + y).reshape(-1)
        return h

    def tokens_per_s(self, T: int, layers: int | None = None, min_s: float = 0.5) -> float:
        """Stack tokens/s over repeated steps of T tokens (at least min_s of work)."""
        x = self.input(T)
        n, t0 = 0, time.perf_counter()
        while True:
            self.forward(x, T, layers)
            n += 1
            dt = time.perf_counter() - t0
            if dt >= min_s:
                return T * n / dt


def sweep(c1_tokens=(1, 7, 64, 1000), c2_tokens=(64, 256, 1024)) -> dict:
    """SURVEY.md §8(d) CPU timing: the oracle port on C1 (one layer) and on one
    C2 (R1-shaped) layer, tokens/s, all host cores."""
    out = {"cores": os.cpu_count() or 1, "c1_layer_tokens_per_s": {}, "c2_layer_tokens_per_s": {}}
    t0 = time.perf_counter()
    c1 = CpuStack(tiny_config(), 1)
    for T in c1_tokens:
        out["c1_layer_tokens_per_s"][str(T)] = c1.tokens_per_s(T, min_s=0.3)
    c2 = CpuStack(r1_config(), 1)
    for T in c2_tokens:
        out["c2_layer_tokens_per_s"][str(T)] = c2.tokens_per_s(T, min_s=0.0)
    out["wall_s"] = time.perf_counter() - t0
    return out
