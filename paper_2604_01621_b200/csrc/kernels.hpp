// Launch wrappers of the DWDP sm_100a kernels (host-callable, plain types).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dwdp {

struct RouterCfg {
  int E, k, scoring, n_group, topk_group, norm_topk;
  float routed_scale;
};

// Counter-hash bf16 fill (bit-identical to oracle_fill_bf16): slot s of
// `nslots` consecutive slots of `slot_elems` elements uses seeds[s].
void launch_fill_slots(uint16_t* dst, const uint64_t* seeds_dev, int nslots,
                       int64_t slot_elems, float scale, cudaStream_t st);
void launch_fill(uint16_t* dst, int64_t n, uint64_t seed, float scale, cudaStream_t st);
void launch_fill_f32(float* dst, int64_t n, uint64_t seed, float scale, cudaStream_t st);

// logits[T][E] = sum_i x[t][i] * w[e][i], fp32 fused multiply-adds in
// ascending i (SIMT reference kernel, kept for microbenchmarks).
void launch_router_logits(const uint16_t* x, const uint16_t* w, float* logits, int64_t T,
                          int E, int64_t K, cudaStream_t st);

// Exact router (the production path). Each bf16 row is mapped to 22-bit
// fixed point relative to its largest exponent (Q_i = mant_i << (e_i - emax +
// 14), truncated below the grid) and split into three balanced int8 digit
// planes dst[p][r][k] (Q = d0 + 2^8 d1 + 2^16 d2); emax[r] is the row
// exponent. The logits are then the int8 tensor-core products of the planes,
// recombined exactly in int64 and rounded once: bit-identical to the oracle.
// If meta != nullptr, writes the single-group GEMM table {mb, mb, 0, 0} for
// 3R rows.
void launch_router_quant(const uint16_t* src, int64_t R, int64_t K, int8_t* dst, int32_t* emax,
                         int32_t* meta, cudaStream_t st);
// Scoring + group-limited top-k + weights; idx/wts [T][k]. Logits come from
// the 9 int32 digit-plane products C[3T][3E] and the row exponents.
// C == nullptr: `logits` already holds the fp32 logits (launch_router_gemm;
// E = 256 contiguous-lane path only).
void launch_topk(const int32_t* C, const int32_t* ex, const int32_t* ew, const float* bias,
                 float* logits, int32_t* idx, float* wts, int64_t T, const RouterCfg& c,
                 cudaStream_t st);

// Stable expert-major permutation + gather of x rows.
//  counts[E]            tokens per expert
//  row_of[T*k]          destination row of pair (t, j)
//  mblock_expert[...]   expert of each 128-row block (routed then shared = E)
//  meta[4]              {total m-blocks, routed m-blocks, routed rows, T}
// scratch: >= permute_scratch_ints(T, E) int32.
int64_t permute_scratch_ints(int64_t T, int E);
//  mb_seg[...]          {first m-block, m-blocks} of each m-block's expert
//  src_row[routed rows] source token of every expert-major row (nullable)
//  xperm                expert-major copy of the rows (nullable: GEMM1 gathers)
// Returns the number of kernels launched.
int launch_permute(const int32_t* idx, const uint16_t* x, int64_t T, int E, int k, int64_t h,
                    int shared, int32_t* counts, int32_t* row_of, int32_t* mblock_expert,
                    int2* mb_seg, int32_t* src_row, int32_t* meta, uint16_t* xperm,
                    int32_t* scratch, cudaStream_t st, uint8_t* xperm8 = nullptr,
                    float* xscale = nullptr, int row_align = 128, int32_t* mb_rows = nullptr,
                    uint8_t* xsf = nullptr, int64_t shared_T = -1, int64_t cap_rows = 0);
// idx entries < 0 are pairs not computed on this rank (row_of = -1, no copy;
// combine_kernel skips them). shared_T (default T): rows of the shared-expert
// block (the DEP receive side permutes all ranks' tokens but runs the shared
// expert on its own). cap_rows > 0: if the padded rows would exceed it, the
// layer computes nothing and meta[4] = 1 (the caller raises).
// DEP receive side: idx -> idx with every expert outside [lo, hi) set to -1.
void launch_localize_idx(const int32_t* in, int64_t n, int lo, int hi, int32_t* out, cudaStream_t st);
// DEP mode 2 send side: idx2 [T][k + 1] = {self, then the rank of each
// expert at its first occurrence in the token's list if it is not self, else
// -1}: one row per (token, destination rank), the own rank always first.
void launch_dest_ranks(const int32_t* idx, int64_t T, int k, int per, int self, int32_t* idx2, cudaStream_t st);
// DEP mode 2: copy each token's routing (k ids, k weights) to every send row
// of that token (row_of2 [T][k2], -1 = no row).
void launch_scatter_routing(const int32_t* idx, const float* wts, const int32_t* row_of2, int64_t T, int k, int k2,
                            int32_t* sidx, float* swts, cudaStream_t st);
void launch_fill_f32(float* p, int64_t n, float v, cudaStream_t st);
// DEP modes 1/2 with quantised rows on the wire: for every row r = row_of[t][j]
// >= 0 copy token t's row scale xs[t] (and its sfb-byte linear block-scale
// row sfl[t], nvfp4) to xs_out[r] / sfl_out[r]. With meta (receive side):
// tokens t < shared_T also get the shared-expert row R = meta[2] + t (scale,
// block scales and the qrow-byte code row codes[t] -> codes_out[R]); nothing
// is written after a receive overflow (meta[4]).
void launch_qrow_meta(const int32_t* row_of, int64_t T, int k, const float* xs, const uint8_t* sfl, int sfb,
                      float* xs_out, uint8_t* sfl_out, const int32_t* meta, int64_t shared_T, const uint8_t* codes,
                      int64_t qrow, uint8_t* codes_out, cudaStream_t st);
// row_of[t][r] = r*T + t and weights 1 for the DEP final combine over N ranks.
void launch_rank_rows(int32_t* row_of, float* w, int64_t T, int N, cudaStream_t st);
// Split layout: the permuted rows stay in 128-row expert segments (X_perm, O,
// GEMM1's m-blocks), while H is laid out in 256-row segments so GEMM2 runs on
// CTA pairs. From the permute's counts this writes the 256-row layout's
// m-block tables (mblock2, mb_seg2, mb_rows2, meta2) and the per-m-block
// output row bases that move rows between the two layouts: d1 [128-layout
// m-blocks] = H row of GEMM1's output block, d2 [256-layout m-blocks] = O row
// (128 layout) of GEMM2's output block. One launch, one CTA.
void launch_split_layout(const int32_t* counts, int E, int64_t T, int shared, int32_t* mblock2,
                         int2* mb_seg2, int32_t* mb_rows2, int32_t* meta2, int32_t* d1, int32_t* d2,
                         cudaStream_t st);
// mb_rows [m-blocks] (nullable): real rows of each m-block (the GEMM epilogues
// skip the padding rows' stores).
// row_align (128 or 256): every expert segment, and the shared-expert block,
// is padded to a multiple of row_align rows (256 for the CTA-pair GEMM).
// W8A8 (weight_dtype fp8): xperm8 [rows][h] e4m3 copies of the token rows
// (routed rows + shared rows from meta[2]) with per-row scales xscale.

// fp8 expert weights: per (slot, row) scale = absmax/448, q = e4m3(v/scale)
// over the bf16 counter-hash values (bit-identical to the oracle).
void launch_fp8_fill_rows(uint8_t* dst, float* scales, const uint64_t* seeds, int nslots, int rows,
                          int64_t K, float scale, cudaStream_t st);
// NVFP4 (weight_dtype nvfp4): with xsf != nullptr the permute writes packed
// e2m1 rows (h/2 bytes) to xperm8, their e4m3 block scales LINEARLY to xsf
// ([rows][h/16]; launch_nvfp4_sf_relayout builds the GEMM's atoms) and fp32
// row scales to xscale.
//
// Block-scale layout of an NVFP4 matrix with K columns: for every 128-row
// block and every 64-column chunk, one 512-byte atom holding the 4 block
// scales of each row at (row % 32) * 16 + (row % 128 / 32) * 4 + block % 4 --
// the layout tcgen05.cp 32x128b.warpx4 expects in shared memory, so the
// GEMM moves it with plain bulk copies.
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int64_t nvfp4_sf_offset(int64_t row, int64_t block, int64_t K) {
  return ((row >> 7) * (K >> 6) + (block >> 2)) * 512 + (row & 31) * 16 + ((row >> 5) & 3) * 4 +
         (block & 3);
}
// NVFP4 expert weights over the bf16 counter-hash values (bit-identical to
// oracle_nvfp4_quant_row): codes [slot][rows][K/2], block scales
// [slot][rows*K/16] (atom layout per slot), row scales [slot][rows].
void launch_nvfp4_fill_rows(uint8_t* dst, uint8_t* sf, float* scales, const uint64_t* seeds,
                            int nslots, int rows, int64_t K, float scale, cudaStream_t st);
// Linear block scales [rows][K/16] -> the atom layout (rows < meta[0]*128;
// meta == nullptr: all max_rows rows, padded to 128 with zeros).
void launch_nvfp4_sf_relayout(const uint8_t* lin, uint8_t* atoms, int64_t max_rows, int64_t K,
                              const int32_t* meta, cudaStream_t st);
// bf16 rows (rows < meta[0]*128) -> NVFP4 codes + block scales (through the
// linear scratch sf_lin, [rows][K/16]) + row scales.
void launch_quant_rows_nvfp4(const uint16_t* src, int64_t max_rows, int64_t K, const int32_t* meta,
                             uint8_t* dst, uint8_t* sf_lin, uint8_t* sf, float* scales, cudaStream_t st);
// bf16 rows (rows < meta[0]*128) -> e4m3 + per-row scale.
void launch_quant_rows_fp8(const uint16_t* src, int64_t max_rows, int64_t K, const int32_t* meta,
                           uint8_t* dst, float* scales, cudaStream_t st);

// y[t] = sum_j w[t,j] * O[row_of[t,j]] (+ S[s_off + t]) (+ x[t]); the shared
// expert rows start at S + s_off*h with s_off = s_meta ? s_meta[2] : 0
// (S == nullptr: no shared expert).
void launch_combine(const uint16_t* O, const int32_t* row_of, const float* wts,
                    const uint16_t* S, const int32_t* s_meta, const uint16_t* resid, uint16_t* y,
                    int64_t T, int k, int64_t h, cudaStream_t st);
// row_of < 0 entries skipped (DEP mode 2's final combine over destination ranks)
void launch_combine_sparse(const uint16_t* O, const int32_t* row_of, const float* wts, const uint16_t* S,
                           const int32_t* s_meta, const uint16_t* resid, uint16_t* y, int64_t T, int k, int64_t h,
                           cudaStream_t st);
// y[t] = sum_j w[t,j] O[row_of[t,j]] over the pairs with row_of >= 0 only
// (the DEP receive side's partial rows; no shared expert, no residual).
void launch_combine_partial(const uint16_t* O, const int32_t* row_of, const float* wts, uint16_t* y, int64_t T,
                            int k, int64_t h, cudaStream_t st);

// One-launch P2P pull of a slice list over NVLink: work[i] = {src, dst, len}.
struct PullItem {
  const void* src;
  void* dst;
  uint64_t len;
};
// max_len: the longest item (bytes); chunks are interleaved across items.
void launch_pull(const PullItem* items_dev, int n_items, uint64_t max_len, int ctas, cudaStream_t st);

// Grouped GEMM on tcgen05 (gemm_sm100.cu). See GemmArgs there.
struct GroupedGemm;

// Preferred shared-memory carveout of this file's layer-path kernels: maximal
// for all of them (`all`: an SM pull engine runs beside the layer, so a GEMM
// CTA must always be able to join an SM holding a pull CTA), else maximal for
// the pull kernel only.
void configure_max_shared_carveout_kernels(bool all);

}  // namespace dwdp
