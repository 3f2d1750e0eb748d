// Grouped tcgen05 GEMM launch interface (see gemm_sm100.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace dwdp {

struct GemmArgs {
  int K;                        // reduction length (multiple of 64)
  int n_out;                    // output columns (SwiGLU: multiple of 128, else of 256)
  int rows_per_slot;            // B rows per arena slot
  int E;                        // expert id of the shared-expert group
  const int32_t* mblock_expert; // [m-blocks] expert of each 128-row block
  const int32_t* slot_of;       // [E + 1] expert -> arena slot
  const int32_t* meta;          // {total m-blocks, routed m-blocks, routed rows, T}
  uint16_t* D;                  // bf16 output (int32 in GEMM_INT8 mode), row-major
  int64_t ldd;                  // elements per output row
  int64_t m_limit;              // rows >= m_limit are not stored
  int shared_a2;                // shared-expert blocks read A from `a2` (GEMM1)
  // Optional [m-blocks] {first m-block, m-block count} of the expert segment
  // each m-block belongs to: tiles are then rastered n-block-major inside a
  // segment so the concurrently running CTAs share B tiles (the expert's
  // weights) and only the segment's A rows stay live in L2.
  const int2* mb_seg;
  // Optional [routed rows] source row of every padded expert-major row: the
  // routed A rows are then gathered straight from the token matrix a_src
  // (row stride a_ld elements) by the producer warp with cp.async into the
  // swizzled smem tile, so no permuted copy is materialised (bf16 GEMM1).
  const int32_t* a_rows;
  // fp8 modes: D = (A_q . B_q^T) * a_scale[row] * b_scale[B row]; SwiGLU uses
  // b_scale0 for the gate rows and b_scale1 for the up rows.
  const float* a_scale;
  const float* b_scale0;
  const float* b_scale1;
  // 0: 1-SM kernel. 1: CTA-pair kernel (cta_group::2, 256 x 256 tiles): needs
  // every expert segment (and the shared block) padded to 256 rows and, for
  // GEMM_PLAIN / GEMM_INT8, B maps with 128-row boxes.
  int pair;
  // segment raster: 0 auto (n-block-major while the segment's A rows <= its
  // B rows), 1 always m-block-major, 2 always n-block-major (experiments)
  int raster;
  // Optional [m-blocks] real rows of each m-block: the epilogue does not
  // store the padding rows (decode batches are mostly padding).
  const int32_t* mb_rows;
  const uint16_t* a_src;  // gather source (a_rows != nullptr)
  int64_t a_ld;
  // NVFP4 modes: e4m3 block scales of A ([m-blocks][K/64][512 B] atoms) and
  // of the B arenas ([slot][rows/128][K/64][512 B]; b_sf1: up rows of
  // GEMM1); a_scale / b_scale* hold the fp32 row scales.
  const uint8_t* a_sf;
  const uint8_t* b_sf0;
  const uint8_t* b_sf1;
  // Optional [m-blocks] first output row of each m-block (default mb * 128):
  // the split layout writes GEMM1's H into 256-row expert segments and GEMM2's
  // O back into 128-row segments (launch_split_layout). A rows stay mb * 128.
  const int32_t* d_row0;
  // > 0: one dense group of dense_m A rows (no tables, meta or slot map;
  // mblock_expert / slot_of / meta may be null; set m_limit = dense_m)
  int64_t dense_m;
};

// 2-D bf16 TMA map over a row-major [rows][cols] matrix, box = 64 x box_rows,
// SWIZZLE_128B (the UMMA K-major operand layout).
CUtensorMap make_tmap_bf16(const void* base, int64_t rows, int64_t cols, int box_rows);
// Same for an int8 matrix (box = 128 x box_rows).
CUtensorMap make_tmap_i8(const void* base, int64_t rows, int64_t cols, int box_rows);

// NVFP4 block-scale atoms viewed as [bytes/128][128] uint8 rows, box 16 rows
// (2 KB = the 4 atoms of one 256-deep k-block and 128 data rows), no swizzle:
// the CTA-pair NVFP4 GEMM loads scales with TMA.
CUtensorMap make_tmap_sf(const void* base, int64_t bytes);
// 3-D bf16 map (dims innermost first, strides in bytes of dims 1 and 2),
// SWIZZLE_128B (box[0] * 2 must be 128 bytes): the attention's per-head tiles.
CUtensorMap make_tmap_3d_bf16(const void* base, const int64_t dims[3], const int64_t strides[2],
                              const int box[3]);
// bf16 [rows][cols] output map, 32 x 32 boxes, SWIZZLE_64B: the TMA-store
// epilogue of the NVFP4 GEMM2.
CUtensorMap make_tmap_out(const void* base, int64_t rows, int64_t cols);

constexpr int GEMM_SWIGLU = 0, GEMM_PLAIN = 1, GEMM_INT8 = 2, GEMM_SWIGLU_FP8 = 3,
              GEMM_PLAIN_FP8 = 4, GEMM_SWIGLU_FP4 = 5, GEMM_PLAIN_FP4 = 6;

// Router logits [T][E] (fp32) from the int8 digit planes of x ([3][T][K],
// 128-row boxes) and of the router weights ([3][E][K], 64-row boxes) with
// the exact recombination fused into the epilogue (E % 64 == 0, K % 128 == 0).
void launch_router_gemm(const CUtensorMap& planes_x, const CUtensorMap& planes_w, const int32_t* xe,
                        const int32_t* we, float* logits, int64_t T, int E, int64_t K, cudaStream_t st);
// The same on CTA pairs (256 tokens per tile; weight planes as 32-row boxes).
void launch_router_gemm_pair(const CUtensorMap& planes_x, const CUtensorMap& planes_w32, const int32_t* xe,
                             const int32_t* we, float* logits, int64_t T, int E, int64_t K, cudaStream_t st);

// a: routed A rows (permuted tokens or H); a2: shared-expert A rows (x);
// b0: gate (SwiGLU) or down arena; b1: up arena (SwiGLU only).
// sf: NVFP4 maps {A scales, B0 scales, B1 scales, D output}; the CTA-pair
// kernel reads the first three, the plain (GEMM2) kernel the output map.
void launch_grouped_gemm(int mode, const CUtensorMap& a, const CUtensorMap& a2,
                         const CUtensorMap& b0, const CUtensorMap& b1, const GemmArgs& args,
                         int max_tiles, cudaStream_t st, const CUtensorMap* sf = nullptr);

}  // namespace dwdp
