"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes front-end over the two checkers built by oracle/Makefile:

* ``C`` — liboracle.so, the plain-C restatement (oracle/dwdp_oracle.c);
* ``REF`` — _ref/libdwdpref.so, the reference library compiled from
  /root/reference (None when it was never built).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference leg
may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(HERE, "liboracle.so")
_REF = os.path.join(HERE, "_ref", "libdwdpref.so")

i32, i64, u64, f32, f64 = C.c_int, C.c_int64, C.c_uint64, C.c_float, C.c_double
P = C.c_void_p


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(P)


class MoeConfig(C.Structure):
    _fields_ = [("hidden", i64), ("num_experts", C.c_int32), ("top_k", C.c_int32),
                ("ffn", i64), ("shared_ffn", i64), ("scoring", C.c_int32),
                ("n_group", C.c_int32), ("topk_group", C.c_int32),
                ("norm_topk", C.c_int32), ("routed_scale", f32),
                ("w8a8", C.c_int32)]


class _Api:
    """Same Python surface over either library (prefix 'oracle_' or 'ref_')."""

    def __init__(self, path: str, prefix: str):
        self.lib = C.CDLL(path)
        self.prefix = prefix
        L = self.lib
        g = lambda n: getattr(L, prefix + n)  # noqa: E731
        g("mix").restype = u64
        g("mix").argtypes = [u64, u64]
        g("rng_u64").argtypes = [u64, i32, P]
        g("rng_normal").argtypes = [u64, i32, f64, f64, P]
        g("build_placement").argtypes = [i32, i32, i32, P, P, P, P, P, i32]
        g("build_copy_plan").argtypes = [P, i32, u64, i32, P, P]
        g("route_tokens").argtypes = [i64, i32, i32, f64, u64, P]
        g("sample_batches").argtypes = [i32, f64, f64, f64, i64, i32, f64, u64,
                                        i32, i32, i32, i32, P, P, P]
        g("expert_shard_bytes").restype = f64
        g("expert_shard_bytes").argtypes = [i64, i64, f64]

    def _f(self, n):
        return getattr(self.lib, self.prefix + n)

    def mix(self, a: int, b: int) -> int:
        return int(self._f("mix")(a, b))

    def rng_u64(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        self._f("rng_u64")(seed, n, _ptr(out))
        return out

    def rng_normal(self, seed: int, n: int, mean: float, sd: float) -> np.ndarray:
        out = np.zeros(n, np.float64)
        self._f("rng_normal")(seed, n, mean, sd, _ptr(out))
        return out

    def build_placement(self, E: int, N: int, extra: int = 0):
        """-> (status, local_count, redundancy, local_sets[N][c], fetch[N][(e,src)])"""
        c = np.zeros(1, np.int32)
        red = np.zeros(1, np.int32)
        ls = np.zeros(N * E, np.int32)
        fe = np.zeros(N * E, np.int32)
        fs = np.zeros(N * E, np.int32)
        st = self._f("build_placement")(E, N, extra, _ptr(c), _ptr(red), _ptr(ls),
                                        _ptr(fe), _ptr(fs), N * E)
        if st:
            return st, None, None, None, None
        cc = int(c[0])
        local = [ls[r * cc:(r + 1) * cc].tolist() for r in range(N)]
        m = E - cc
        fetch = [list(zip(fe[r * m:(r + 1) * m].tolist(), fs[r * m:(r + 1) * m].tolist()))
                 for r in range(N)]
        return 0, cc, int(red[0]), local, fetch

    def build_copy_plan(self, shards, slice_size: int, dst: int = 0):
        """shards: [(peer, param, size, src_offset)] -> (status, [(param, src, src_off, dst_off, len)])"""
        sh = np.array(shards, np.int64).reshape(-1, 4) if shards else np.zeros((0, 4), np.int64)
        sh = np.ascontiguousarray(sh)
        n = np.zeros(1, np.int64)
        st = self._f("build_copy_plan")(_ptr(sh), len(sh), slice_size, dst, None, _ptr(n))
        if st:
            return st, None
        out = np.zeros((max(int(n[0]), 1), 5), np.int64)
        st = self._f("build_copy_plan")(_ptr(sh), len(sh), slice_size, dst, _ptr(out), _ptr(n))
        return st, [tuple(r) for r in out[: int(n[0])].tolist()]

    def route_tokens(self, tokens: int, E: int, k: int, skew: float, seed: int):
        out = np.zeros(E, np.int64)
        st = self._f("route_tokens")(tokens, E, k, skew, seed, _ptr(out))
        return st, out

    def sample_batches(self, kind: int, length: float, ratio: float, sd: float, mnt: int,
                       bpr: int, skew: float, seed: int, E: int, k: int, N: int, iters: int,
                       routed: bool = True):
        t = np.zeros(iters * N, np.int64)
        q = np.zeros(iters * N, np.int64)
        r = np.zeros(iters * N * E, np.int64) if routed else None
        st = self._f("sample_batches")(kind, length, ratio, sd, mnt, bpr, skew, seed, E, k, N,
                                       iters, _ptr(t), _ptr(q), _ptr(r))
        return st, t.reshape(iters, N), q.reshape(iters, N), (
            r.reshape(iters, N, E) if routed else None)

    def expert_shard_bytes(self, h: int, f: int, wb: float) -> float:
        return float(self._f("expert_shard_bytes")(h, f, wb))


class _Oracle(_Api):
    def __init__(self):
        super().__init__(_LIB, "oracle_")
        L = self.lib
        L.oracle_moe_entries.argtypes = [i64, i64, i64, f64, f64, f64, f64, i32, P]
        L.oracle_expf.restype = f32
        L.oracle_expf.argtypes = [f32]
        L.oracle_sigmoidf.restype = f32
        L.oracle_sigmoidf.argtypes = [f32]
        L.oracle_fill_bf16.argtypes = [u64, i64, f32, P]
        L.oracle_tensor_seed.restype = u64
        L.oracle_tensor_seed.argtypes = [u64, i32, i32, i32]
        L.oracle_route.argtypes = [P, P, i64, P, P, P, P, P]
        L.oracle_permute.restype = i64
        L.oracle_permute.argtypes = [P, i64, i32, i32, i32, P, P]
        L.oracle_moe_forward_seeded.argtypes = [P, u64, i32, P, i64, P, P, P, P, i32]
        L.oracle_e4m3_encode.argtypes = [P, i64, P]
        L.oracle_quant_row_e4m3.argtypes = [P, i64, P, P]
        L.oracle_nvfp4_quant_row.argtypes = [P, i64, P, P, P]
        L.oracle_nvfp4_sf_offset.argtypes = [i64, i64, i64]
        L.oracle_nvfp4_sf_offset.restype = i64
        L.oracle_e2m1_to_f32.argtypes = [C.c_uint8]
        L.oracle_e2m1_to_f32.restype = f32
        L.oracle_moe_forward_explicit.argtypes = [P, P, i64, P, P, P, P, P, P, P, P, P, P, P]
        L.oracle_moe_forward_bf16w.argtypes = [P, P, i64, P, P, P, P, P, P, P, P, i32]

    def moe_forward_bf16w(self, cfg: MoeConfig, x_bf16: np.ndarray, T: int,
                          w_router_bf16: np.ndarray, bias, gate: list, up: list, down: list,
                          nthreads: int = 0):
        """gate/up/down: per expert (E+1 entries, shared last) uint16 arrays or None."""
        n = cfg.num_experts + 1
        arr = lambda L: (C.c_void_p * n)(*[None if a is None else a.ctypes.data for a in L])  # noqa: E731
        y = np.zeros(T * cfg.hidden, np.float32)
        idx = np.zeros(T * cfg.top_k, np.int32)
        wts = np.zeros(T * cfg.top_k, np.float32)
        self.lib.oracle_moe_forward_bf16w(C.byref(cfg), _ptr(x_bf16), T, _ptr(w_router_bf16),
                                          _ptr(bias), arr(gate), arr(up), arr(down), _ptr(y),
                                          _ptr(idx), _ptr(wts), nthreads)
        return (y.reshape(T, cfg.hidden), idx.reshape(T, cfg.top_k),
                wts.reshape(T, cfg.top_k))

    def moe_entries(self, h, f, fs, wb, ab, tokens, pairs, touched):
        out = np.zeros(4, np.float64)
        self.lib.oracle_moe_entries(h, f, fs, wb, ab, tokens, pairs, touched, _ptr(out))
        return out

    def expf(self, x: float) -> float:
        return float(self.lib.oracle_expf(x))

    def sigmoidf(self, x: float) -> float:
        return float(self.lib.oracle_sigmoidf(x))

    def tensor_seed(self, base: int, layer: int, expert: int, t: int) -> int:
        return int(self.lib.oracle_tensor_seed(base, layer, expert, t))

    def fill_bf16(self, seed: int, n: int, scale: float) -> np.ndarray:
        out = np.zeros(n, np.uint16)
        self.lib.oracle_fill_bf16(seed, n, scale, _ptr(out))
        return out

    def route(self, cfg: MoeConfig, x_bf16: np.ndarray, T: int, w_router_bf16: np.ndarray,
              bias: np.ndarray | None):
        E, k = cfg.num_experts, cfg.top_k
        logits = np.zeros(T * E, np.float32)
        idx = np.zeros(T * k, np.int32)
        wts = np.zeros(T * k, np.float32)
        self.lib.oracle_route(C.byref(cfg), _ptr(x_bf16), T, _ptr(w_router_bf16), _ptr(bias),
                              _ptr(logits), _ptr(idx), _ptr(wts))
        return logits.reshape(T, E), idx.reshape(T, k), wts.reshape(T, k)

    def permute(self, idx: np.ndarray, E: int, align: int):
        T, k = idx.shape
        idx = np.ascontiguousarray(idx, np.int32)
        counts = np.zeros(E, np.int32)
        row_of = np.zeros(T * k, np.int64)
        total = self.lib.oracle_permute(_ptr(idx), T, E, k, align, _ptr(counts), _ptr(row_of))
        return int(total), counts, row_of.reshape(T, k)

    def e4m3_encode(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32).reshape(-1)
        out = np.zeros(x.size, np.uint8)
        self.lib.oracle_e4m3_encode(_ptr(x), x.size, _ptr(out))
        return out

    def quant_row_e4m3(self, v):
        v = np.ascontiguousarray(v, np.float32).reshape(-1)
        q = np.zeros(v.size, np.uint8)
        s = C.c_float()
        self.lib.oracle_quant_row_e4m3(_ptr(v), v.size, _ptr(q), C.byref(s))
        return q, s.value

    def nvfp4_quant_rows(self, v):
        """NVFP4 rows: codes [R][K/2], linear block scales [R][K/16] (e4m3 codes),
        row scales [R] -- the device recipe (kernels.cu nvfp4_block)."""
        v = np.ascontiguousarray(v, np.float32)
        R, K = v.shape
        codes = np.zeros((R, K // 2), np.uint8)
        sf = np.zeros((R, K // 16), np.uint8)
        s = np.zeros(R, np.float32)
        for r in range(R):
            self.lib.oracle_nvfp4_quant_row(_ptr(v[r]), K, _ptr(codes[r]), _ptr(sf[r]),
                                            s[r:].ctypes.data)
        return codes, sf, s

    @staticmethod
    def nvfp4_sf_atoms(sf: np.ndarray) -> np.ndarray:
        """Linear block scales [R][K/16] -> the device's 512-byte atom layout
        (ceil(R/128)*128*K/16 bytes; kernels.hpp nvfp4_sf_offset)."""
        R, nb = sf.shape
        K = nb * 16
        rows = np.arange(R, dtype=np.int64)[:, None]
        b = np.arange(nb, dtype=np.int64)[None, :]
        off = ((rows >> 7) * (K >> 6) + (b >> 2)) * 512 + (rows & 31) * 16 + ((rows >> 5) & 3) * 4 + (b & 3)
        out = np.zeros(((R + 127) // 128) * 128 * nb, np.uint8)
        out[off.reshape(-1)] = sf.reshape(-1)
        return out

    @staticmethod
    def nvfp4_dequant(codes: np.ndarray, sf: np.ndarray, s: np.ndarray | None = None) -> np.ndarray:
        """codes [R][K/2] + linear block scales [R][K/16] (+ row scales) -> fp32."""
        mag = np.array([0, .5, 1, 1.5, 2, 3, 4, 6], np.float32)
        lut = np.concatenate([mag, -mag])
        q = np.stack([codes & 15, codes >> 4], axis=-1).reshape(codes.shape[0], -1)
        v = lut[q]
        e = (sf >> 3) & 15
        m = (sf & 7).astype(np.float32)
        d = np.where(e > 0, (1 + m / 8) * np.exp2(e.astype(np.float32) - 7), m * 2.0 ** -9).astype(np.float32)
        v = v * np.repeat(d, 16, axis=1)
        return v if s is None else v * s[:, None]

    def moe_forward_seeded(self, cfg: MoeConfig, base: int, layer: int, x_bf16: np.ndarray,
                           T: int, bias: np.ndarray | None, nthreads: int = 0):
        y = np.zeros(T * cfg.hidden, np.float32)
        idx = np.zeros(T * cfg.top_k, np.int32)
        wts = np.zeros(T * cfg.top_k, np.float32)
        self.lib.oracle_moe_forward_seeded(C.byref(cfg), base, layer, _ptr(x_bf16), T,
                                           _ptr(bias), _ptr(y), _ptr(idx), _ptr(wts), nthreads)
        return (y.reshape(T, cfg.hidden), idx.reshape(T, cfg.top_k),
                wts.reshape(T, cfg.top_k))

    def moe_forward_explicit(self, cfg: MoeConfig, x, w_router, bias, w_gate, w_up, w_down,
                             s_gate=None, s_up=None, s_down=None):
        f32a = lambda a: None if a is None else np.ascontiguousarray(a, np.float32)  # noqa: E731
        x, w_router, bias = f32a(x), f32a(w_router), f32a(bias)
        w_gate, w_up, w_down = f32a(w_gate), f32a(w_up), f32a(w_down)
        s_gate, s_up, s_down = f32a(s_gate), f32a(s_up), f32a(s_down)
        T = x.shape[0]
        y = np.zeros((T, cfg.hidden), np.float32)
        idx = np.zeros((T, cfg.top_k), np.int32)
        wts = np.zeros((T, cfg.top_k), np.float32)
        self.lib.oracle_moe_forward_explicit(
            C.byref(cfg), _ptr(x), T, _ptr(w_router), _ptr(bias), _ptr(w_gate), _ptr(w_up),
            _ptr(w_down), _ptr(s_gate), _ptr(s_up), _ptr(s_down), _ptr(y), _ptr(idx), _ptr(wts))
        return y, idx, wts


class _Ref(_Api):
    def __init__(self):
        super().__init__(_REF, "ref_")
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_moe_entries.argtypes = [i64, i32, i32, i64, i64, f64, f64, f64, f64, i32, P]
        L.ref_simulate.argtypes = [i32, i32, i64, i32, i32, i64, i64, f64, f64, f64, f64, i32,
                                   i32, i32, i32, f64, f64, f64, i64, i32, u64, i32, u64, i32, P]
        L.ref_analytic.argtypes = [i64, i32, i32, i64, i64, f64, f64, f64, f64, i32, i64, P]
        L.ref_simulate_store.argtypes = [i32, i32, i32, i64, i32, i32, i64, i64, f64, f64, f64, f64,
                                         i32, i32, i32, i32, f64, f64, f64, i64, i32, u64, i32, u64,
                                         i32, P]
        L.ref_simulate_store_cal.argtypes = [i32, i32, i32, i64, i32, i32, i64, i64, f64, P, i32, i32,
                                             i32, i32, f64, f64, f64, i64, i32, u64, i32, u64, i32, P]
        L.ref_report_events.argtypes = [i32, P, P, P, P, P, P, P]
        L.ref_report_breakdown.argtypes = [i32, P, C.c_char_p, i32]
        L.ref_compare.argtypes = [P, P, P, C.c_char_p, i32]

    def moe_entries(self, h, f, fs, wb, ab, tokens, pairs, touched, E=256, k=8):
        out = np.zeros(4, np.float64)
        st = self.lib.ref_moe_entries(h, E, k, f, fs, wb, ab, tokens, pairs, touched, _ptr(out))
        assert st == 0, self.lib.ref_last_error()
        return out

    def simulate(self, dwdp: bool, layers, h, E, k, f, fs, wb, peak, mem_bw, link_bw, N, iters,
                 warmup, kind, length, ratio, sd, mnt, bpr, seed, tdm=True, slice_size=1 << 20,
                 merge_elim=True):
        out = np.zeros(3, np.float64)
        st = self.lib.ref_simulate(int(dwdp), layers, h, E, k, f, fs, wb, peak, mem_bw, link_bw,
                                   N, iters, warmup, kind, length, ratio, sd, mnt, bpr, seed,
                                   int(tdm), slice_size, int(merge_elim), _ptr(out))
        assert st == 0, self.lib.ref_last_error()
        return {"tokens_per_s": out[0], "latency_us": out[1], "exposed_us_per_layer": out[2]}

    def simulate_report(self, slot: int, dwdp: bool, layers, h, E, k, f, fs, wb, peak, mem_bw,
                        link_bw, N, iters, warmup, kind, length, ratio, sd, mnt, bpr, seed,
                        tdm=True, slice_size=1 << 20, merge_elim=True):
        """Run the reference simulator into report slot `slot`; return its
        events, iteration spans, breakdown (35 packed doubles) and CSV."""
        n = C.c_int()
        st = self.lib.ref_simulate_store(slot, int(dwdp), layers, h, E, k, f, fs, wb, peak, mem_bw,
                                         link_bw, N, iters, warmup, kind, length, ratio, sd, mnt,
                                         bpr, seed, int(tdm), slice_size, int(merge_elim),
                                         C.byref(n))
        assert st == 0, self.lib.ref_last_error()
        ne = n.value
        i32a = np.zeros((max(ne, 1), 6), np.int32)
        i64a = np.zeros((max(ne, 1), 2), np.int64)
        by = np.zeros(max(ne, 1), np.float64)
        isa = np.zeros(N * iters, np.int64)
        iea = np.zeros(N * iters, np.int64)
        tka = np.zeros(N * iters, np.int64)
        dims = np.zeros(3, np.int32)
        st = self.lib.ref_report_events(slot, _ptr(i32a), _ptr(i64a), _ptr(by), _ptr(isa),
                                        _ptr(iea), _ptr(tka), _ptr(dims))
        assert st == 0, self.lib.ref_last_error()
        bd = np.zeros(35, np.float64)
        csv = C.create_string_buffer(8192)
        st = self.lib.ref_report_breakdown(slot, _ptr(bd), csv, 8192)
        assert st == 0, self.lib.ref_last_error()
        return {"events": (i32a[:ne], i64a[:ne], by[:ne]), "iter_start": isa, "iter_end": iea,
                "iter_tokens": tka, "dims": dims.tolist(), "breakdown": bd,
                "csv": csv.value.decode()}

    def simulate_report_cal(self, slot: int, dwdp: bool, layers, h, E, k, f, fs, wb, cal: dict, N,
                            iters, warmup, kind, length, ratio, sd, mnt, bpr, seed, tdm=True,
                            slice_size=1 << 20, merge_elim=True):
        """simulate_dwdp / simulate_dep with calibrated GpuSpec + CostCalibration
        (cal: peak_flops, mem_bw, link_bw, ce_inflight, grouped_gemm, dense_gemm,
        others_bytes_factor, mem_interference) into report slot `slot`; returns
        the same dict as simulate_report."""
        keys = ("peak_flops", "mem_bw", "link_bw", "ce_inflight", "grouped_gemm", "dense_gemm",
                "others_bytes_factor", "mem_interference")
        c = np.array([float(cal[k]) for k in keys], np.float64)
        n = C.c_int()
        st = self.lib.ref_simulate_store_cal(slot, int(dwdp), layers, h, E, k, f, fs, wb, _ptr(c), N,
                                             iters, warmup, kind, length, ratio, sd, mnt, bpr, seed,
                                             int(tdm), slice_size, int(merge_elim), C.byref(n))
        assert st == 0, self.lib.ref_last_error()
        return self._report(slot, n.value, N, iters)

    def _report(self, slot: int, ne: int, N: int, iters: int):
        i32a = np.zeros((max(ne, 1), 6), np.int32)
        i64a = np.zeros((max(ne, 1), 2), np.int64)
        by = np.zeros(max(ne, 1), np.float64)
        isa = np.zeros(N * iters, np.int64)
        iea = np.zeros(N * iters, np.int64)
        tka = np.zeros(N * iters, np.int64)
        dims = np.zeros(3, np.int32)
        st = self.lib.ref_report_events(slot, _ptr(i32a), _ptr(i64a), _ptr(by), _ptr(isa),
                                        _ptr(iea), _ptr(tka), _ptr(dims))
        assert st == 0, self.lib.ref_last_error()
        bd = np.zeros(35, np.float64)
        csv = C.create_string_buffer(8192)
        st = self.lib.ref_report_breakdown(slot, _ptr(bd), csv, 8192)
        assert st == 0, self.lib.ref_last_error()
        return {"events": (i32a[:ne], i64a[:ne], by[:ne]), "iter_start": isa, "iter_end": iea,
                "iter_tokens": tka, "dims": dims.tolist(), "breakdown": bd,
                "csv": csv.value.decode()}

    def compare(self, a35: np.ndarray, b35: np.ndarray):
        out = np.zeros(36, np.float64)
        csv = C.create_string_buffer(8192)
        st = self.lib.ref_compare(_ptr(np.ascontiguousarray(a35, np.float64)),
                                  _ptr(np.ascontiguousarray(b35, np.float64)), _ptr(out), csv, 8192)
        assert st == 0, self.lib.ref_last_error()
        return out, csv.value.decode()

    def analytic(self, h, E, k, f, fs, wb, peak, mem_bw, link_bw, N, tokens):
        out = np.zeros(4, np.float64)
        st = self.lib.ref_analytic(h, E, k, f, fs, wb, peak, mem_bw, link_bw, N, tokens, _ptr(out))
        assert st == 0, self.lib.ref_last_error()
        return {"t_compute_s": out[0], "t_prefetch_s": out[1], "t_all2all_s": out[2],
                "dep_dwdp_speedup": out[3]}


def oracle() -> _Oracle:
    if not os.path.exists(_LIB):
        build()
    return _Oracle()


def ref() -> _Ref | None:
    if not os.path.exists(_REF):
        try:
            build()
        except Exception:  # noqa: BLE001
            return None
    return _Ref() if os.path.exists(_REF) else None


def bf16_round(a: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns (uint16), round to nearest even."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(u16, np.uint16).astype(np.uint32) << 16).view(np.float32)
