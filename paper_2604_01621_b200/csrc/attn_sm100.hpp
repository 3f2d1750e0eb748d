// MLA prefill attention on sm_100a (attn_sm100.cu): kernel launchers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "gemm_sm100.hpp"

namespace dwdp {

// One 128-query tile of one sequence: tokens [start, start + len) of the
// packed batch, queries [q0, min(q0 + 128, len)); vstart: the sequence's
// first column in V^T (a multiple of 64: TMA boxes of V^T start aligned).
struct AttnTile {
  int32_t start, len, q0, vstart;
};

// Causal attention per sequence and head: q, k [T][H][192] (128 nope + 64
// rope), vt [H][128][ldv] (V transposed, columns per AttnTile::vstart,
// ldv a multiple of 8) -> out
// [T][H][128], bf16, fp32 softmax; grid = tiles x heads.
void launch_mla_attention(const uint16_t* q, const uint16_t* k, const uint16_t* vt, int64_t T, int64_t ldv,
                          int H, const AttnTile* tiles, int ntiles, float softmax_scale, uint16_t* out,
                          cudaStream_t st);
// Query rows per AttnTile the attention kernel expects: 128, or 256 for the
// two-tile kernel (DWDP_ATTN_PAIR=1).
int mla_attention_query_step();
// y[r] = x[r] * rsqrt(mean(x[r]^2) + eps), rows of D elements (bf16, fp32 math).
void launch_rmsnorm(const uint16_t* in, int64_t ld_in, uint16_t* out, int64_t ld_out, int64_t rows, int D,
                    float eps, cudaStream_t st);
// RoPE (interleaved pairs, base theta) of q's 64 rope dims, in place.
void launch_q_rope(uint16_t* q, const int32_t* pos, int64_t T, int H, float theta, cudaStream_t st);
// K = (k_nope | RoPE(k_rope)) per head, V^T from kv [T][H][256] and kva
// [T][ld_kva]; token t's V^T column is vcol[t] (sequences start 64-aligned).
void launch_kv_assemble(const uint16_t* kv, const uint16_t* kva, int64_t ld_kva, int kv_lora, const int32_t* pos,
                        const int32_t* vcol, int64_t T, int H, float theta, uint16_t* K, uint16_t* Vt,
                        int64_t ldv, cudaStream_t st);

}  // namespace dwdp
