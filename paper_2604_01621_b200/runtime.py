"""Python handle over the per-GPU DWDP runtime (dwdp_ctx in include/dwdp.h).

torch is used only as plumbing (device buffers, streams); every computation
runs in libdwdp.so's sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import asdict, dataclass

import numpy as np

from ._lib import (ENGINE_COPY, IPC_BLOB_BYTES, WEIGHT_FP8, WEIGHT_NVFP4, CtxConfigC, LayerRecordC, SliceC, check, lib)
from .planning import Slice


@dataclass
class DwdpConfig:
    """dwdp_ctx_config. Defaults: one DeepSeek-R1-shaped MoE layer group
    (h 7168, E 256 top-8, f 2048, 1 shared expert, sigmoid + noaux_tc
    group-limited routing n_group 8 / topk_group 4, norm_topk, scale 2.5)."""
    num_layers: int = 8
    num_experts: int = 256
    hidden: int = 7168
    ffn: int = 2048
    shared_ffn: int = 2048
    top_k: int = 8
    scoring: int = 1          # 0 softmax, 1 sigmoid
    n_group: int = 8
    topk_group: int = 4
    norm_topk: int = 1
    routed_scale: float = 2.5
    rank: int = 0
    group_size: int = 1
    extra_redundancy: int = 0
    device: int = 0
    merge_elim: int = 1
    tdm: int = 1
    slice_size: int = 1 << 20
    engine: int = ENGINE_COPY
    pull_ctas: int = 148      # pull-kernel CTAs (one per SM, co-resident with the GEMM)
    ce_inflight: int = 2      # copy-engine transfers in flight (reference GpuSpec default 2)
    weight_dtype: int = 0     # 0 bf16, 1 fp8 e4m3 (W8A8, per-channel weight scales)
    weight_seed: int = 2604_01621
    weight_layers: int = 0    # 0 = num_layers
    kernel_timing: int = 0    # CUDA events between the layer's kernels
    max_tokens: int = 32768

    @staticmethod
    def tiny(**kw) -> "DwdpConfig":
        """BASELINE config 1: hidden 512, 16 experts top-2 (softmax), f 1024."""
        d = dict(num_layers=1, num_experts=16, hidden=512, ffn=1024, shared_ffn=0, top_k=2,
                 scoring=0, n_group=1, topk_group=1, norm_topk=1, routed_scale=1.0,
                 max_tokens=1024)
        d.update(kw)
        return DwdpConfig(**d)

    def c(self) -> CtxConfigC:
        d = asdict(self)
        return CtxConfigC(**{k: d[k] for k, _ in CtxConfigC._fields_})


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class DwdpContext:
    def __init__(self, cfg: DwdpConfig):
        self.cfg = cfg
        h = C.c_void_p()
        check(lib().dwdp_ctx_create(C.byref(cfg.c()), C.byref(h)))
        self.h = h

    # -- lifecycle -----------------------------------------------------------
    def close(self) -> None:
        if self.h:
            check(lib().dwdp_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def memory(self) -> dict:
        w, r, ws = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().dwdp_ctx_memory(self.h, C.byref(w), C.byref(r), C.byref(ws)))
        return {"weights": w.value, "recv": r.value, "workspace": ws.value}

    # -- peers ---------------------------------------------------------------
    def export_ipc(self) -> bytes:
        buf = C.create_string_buffer(IPC_BLOB_BYTES)
        check(lib().dwdp_ctx_export_ipc(self.h, buf))
        return buf.raw

    def open_peers(self, blobs: bytes) -> None:
        assert len(blobs) == IPC_BLOB_BYTES * self.cfg.group_size
        check(lib().dwdp_ctx_open_peers(self.h, C.create_string_buffer(blobs, len(blobs))))

    @staticmethod
    def link_local(ctxs: list["DwdpContext"]) -> None:
        arr = (C.c_void_p * len(ctxs))(*[c.h for c in ctxs])
        check(lib().dwdp_ctx_link_local(arr, len(ctxs)))

    # -- weights -------------------------------------------------------------
    def init_weights(self, bias_scale: float = 0.0) -> None:
        check(lib().dwdp_ctx_init_weights(self.h, bias_scale))

    def set_bias(self, bias: np.ndarray) -> None:
        b = np.ascontiguousarray(bias, np.float32)
        assert b.shape == (self.cfg.num_experts,)
        check(lib().dwdp_ctx_set_bias(self.h, b.ctypes.data))

    def read_expert(self, layer: int, expert: int, t: int) -> np.ndarray:
        """Resident copy of tensor t (0 gate, 1 up, 2 down: bf16 bits, e4m3
        bytes for fp8, packed e2m1 codes [rows][K/2] for nvfp4; fp8/nvfp4:
        3/4/5 = per-row fp32 scales; nvfp4: 6/7/8 = e4m3 block scales in the
        512-byte atom layout, flat [rows*K/16])."""
        rows, cols = (self.cfg.ffn, self.cfg.hidden) if t % 3 < 2 else (self.cfg.hidden, self.cfg.ffn)
        if t >= 6:
            out = np.zeros(rows * cols // 16, np.uint8)
        elif t >= 3:
            out = np.zeros(rows, np.float32)
        elif self.cfg.weight_dtype == WEIGHT_NVFP4:
            out = np.zeros(rows * cols // 2, np.uint8)
            cols //= 2
        else:
            out = np.zeros(rows * cols, np.uint8 if self.cfg.weight_dtype == WEIGHT_FP8 else np.uint16)
        check(lib().dwdp_ctx_read_expert(self.h, layer, expert, t, out.ctypes.data))
        return out if t >= 3 else out.reshape(rows, cols)

    # -- prefetch handles (CopyEngineSim API) -------------------------------
    def prefetch_issue(self, global_layer: int) -> int:
        h = C.c_int64()
        check(lib().dwdp_prefetch_issue(self.h, global_layer, C.byref(h)))
        return h.value

    def prefetch_query(self, handle: int) -> bool:
        d = C.c_int32()
        check(lib().dwdp_prefetch_query(self.h, handle, C.byref(d)))
        return bool(d.value)

    def prefetch_wait(self, handle: int, stream=None) -> None:
        check(lib().dwdp_prefetch_wait(self.h, handle, _stream(stream)))

    def prefetch_times(self, handle: int) -> tuple[int, int, float]:
        s, e, b = C.c_int64(), C.c_int64(), C.c_double()
        check(lib().dwdp_prefetch_times(self.h, handle, C.byref(s), C.byref(e), C.byref(b)))
        return s.value, e.value, b.value

    def set_engine(self, engine: int) -> None:
        check(lib().dwdp_ctx_set_engine(self.h, engine))
        self.cfg.engine = engine

    def copy_plan(self) -> list[Slice]:
        n = C.c_size_t(0)
        check(lib().dwdp_ctx_copy_plan(self.h, None, C.byref(n)))
        arr = (SliceC * max(n.value, 1))()
        check(lib().dwdp_ctx_copy_plan(self.h, arr, C.byref(n)))
        return [Slice(arr[i].param_id, arr[i].src_rank, arr[i].src_offset, arr[i].dst_offset,
                      arr[i].length) for i in range(n.value)]

    # -- forward -------------------------------------------------------------
    def _out(self, x, y):
        import torch
        return torch.empty_like(x) if y is None else y

    def moe_forward(self, layer: int, x, y=None, stream=None):
        y = self._out(x, y)
        check(lib().dwdp_moe_forward(self.h, layer, _ptr(x), x.shape[0], _ptr(y), _stream(stream)))
        return y

    def layer_forward(self, global_layer: int, x, y=None, residual: bool = True, stream=None):
        y = self._out(x, y)
        check(lib().dwdp_layer_forward(self.h, global_layer, _ptr(x), x.shape[0], _ptr(y),
                                       int(residual), _stream(stream)))
        return y

    def stack_forward(self, x, y=None, stream=None):
        y = self._out(x, y)
        check(lib().dwdp_stack_forward(self.h, _ptr(x), x.shape[0], _ptr(y), _stream(stream)))
        return y

    def route(self, layer: int, x, stream=None):
        import torch
        T, k, E = x.shape[0], self.cfg.top_k, self.cfg.num_experts
        dev = x.device
        idx = torch.empty((T, k), dtype=torch.int32, device=dev)
        wts = torch.empty((T, k), dtype=torch.float32, device=dev)
        counts = torch.empty((E,), dtype=torch.int32, device=dev)
        row_of = torch.empty((T, k), dtype=torch.int32, device=dev)
        rows = C.c_int64()
        check(lib().dwdp_route(self.h, layer, _ptr(x), T, _ptr(idx), _ptr(wts), _ptr(counts),
                               _ptr(row_of), C.byref(rows), _stream(stream)))
        return idx, wts, counts, row_of, rows.value

    # -- DEP baseline (same kernels + NCCL all-to-alls) ----------------------
    def dep_init(self, nccl_id: bytes) -> None:
        assert len(nccl_id) == 128
        check(lib().dwdp_dep_init(self.h, C.create_string_buffer(nccl_id, 128)))

    def dep_set_mode(self, mode: int) -> None:
        """0: per-pair dispatch (reference semantics); 1: each token row once to
        every peer; 2: only to the ranks owning one of its experts; 1 and 2
        merge on the receive side and return one partial row per (token,
        rank) (dwdp_dep_set_mode)."""
        check(lib().dwdp_dep_set_mode(self.h, mode))

    def dep_layer_forward(self, layer: int, x, y=None, residual: bool = True, stream=None):
        y = self._out(x, y)
        check(lib().dwdp_dep_layer_forward(self.h, layer, _ptr(x), x.shape[0], _ptr(y),
                                           int(residual), _stream(stream)))
        return y

    def dep_stack_forward(self, x, y=None, stream=None):
        y = self._out(x, y)
        check(lib().dwdp_dep_stack_forward(self.h, _ptr(x), x.shape[0], _ptr(y), _stream(stream)))
        return y

    # -- accounting ----------------------------------------------------------
    def records(self) -> list[dict]:
        out = []
        while True:
            arr = (LayerRecordC * 256)()
            n = C.c_size_t(256)
            check(lib().dwdp_ctx_records(self.h, arr, C.byref(n)))
            out += [{k: getattr(arr[i], k) for k, _ in LayerRecordC._fields_} for i in range(n.value)]
            if n.value < 256:
                return out

    def launch_count(self) -> int:
        n = C.c_int64()
        check(lib().dwdp_ctx_launch_count(self.h, C.byref(n)))
        return n.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().dwdp_nccl_unique_id(buf))
    return buf.raw


def gemm_bf16(A, B, D=None, stream=None):
    """D = A @ B^T on the tcgen05 grouped-GEMM kernel (one group)."""
    import torch
    M, K = A.shape
    N = B.shape[0]
    D = torch.empty((M, N), dtype=torch.bfloat16, device=A.device) if D is None else D
    check(lib().dwdp_gemm_bf16(_ptr(A), _ptr(B), _ptr(D), M, N, K, _stream(stream)))
    return D


def quant_nvfp4(x, stream=None):
    """NVFP4 rows of a bf16 [R][K] matrix (the activation recipe): codes
    [R][K/2] uint8, block scales in the 512-byte atom layout, fp32 row scales."""
    import torch
    R, K = x.shape
    codes = torch.empty((R, K // 2), dtype=torch.uint8, device=x.device)
    sf = torch.zeros(((R + 127) // 128 * 128) * (K // 16), dtype=torch.uint8, device=x.device)
    s = torch.empty(R, dtype=torch.float32, device=x.device)
    check(lib().dwdp_quant_nvfp4(_ptr(x), R, K, _ptr(codes), _ptr(sf), _ptr(s), _stream(stream)))
    return codes, sf, s


def gemm_nvfp4(A, B, D=None, stream=None):
    """D = (A . B^T) * sa * sb over quant_nvfp4 outputs A = (codes, sf, s),
    B likewise, on the kind::mxf4nvf4 grouped-GEMM kernel (one group)."""
    import torch
    (a, asf, as_), (b, bsf, bs) = A, B
    M, N, K = a.shape[0], b.shape[0], 2 * a.shape[1]
    D = torch.empty((M, N), dtype=torch.bfloat16, device=a.device) if D is None else D
    check(lib().dwdp_gemm_nvfp4(_ptr(a), _ptr(asf), _ptr(as_), _ptr(b), _ptr(bsf), _ptr(bs), _ptr(D),
                                M, N, K, _stream(stream)))
    return D


def fill_bf16(t, seed: int, scale: float, stream=None):
    """Counter-hash fill, bit-identical to oracle_fill_bf16."""
    check(lib().dwdp_fill_bf16(_ptr(t), t.numel(), seed, scale, _stream(stream)))
    return t
