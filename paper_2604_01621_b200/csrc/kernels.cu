// DWDP sm_100a kernels except the grouped GEMM (gemm_sm100.cu):
// counter-hash init, router logits + scoring/top-k, stable permute/gather,
// weighted combine and the NVLink pull kernel.
//
// Numerical contract with the oracle (oracle/dwdp_oracle.c): the router
// logits are sequential fused multiply-adds over i = 0..h-1, the scoring
// exponent is a fixed IEEE sequence (det_expf), and the permutation is the
// stable expert-major order of (t, j) pairs — so expert indices, routing
// weights and row positions are bit-identical to the CPU restatement.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <stdexcept>
#include <cstdlib>
#include <cstdint>

#include "kernels.hpp"

namespace dwdp {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float hash_val(uint64_t seed, int64_t i, float scale) {
  const uint32_t u = static_cast<uint32_t>(mix64(seed, static_cast<uint64_t>(i)) >> 40);
  const float v = __fsub_rn(__fmul_rn(static_cast<float>(u), 0x1.0p-23f), 1.0f);
  return __fmul_rn(v, scale);
}

__device__ __forceinline__ uint16_t bf16_bits(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

__device__ __forceinline__ float bf16_f(uint16_t b) {
  return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

// ---------------------------------------------------------------- init
__global__ void fill_slots_kernel(uint16_t* __restrict__ dst, const uint64_t* __restrict__ seeds,
                                  int nslots, int64_t slot_elems, float scale) {
  const int64_t groups_per_slot = slot_elems / 8;
  const int64_t total = groups_per_slot * nslots;
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < total;
       g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = g / groups_per_slot;
    const int64_t e0 = (g - s * groups_per_slot) * 8;
    const uint64_t seed = seeds[s];
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      w[q] = uint32_t(bf16_bits(hash_val(seed, e0 + 2 * q, scale))) |
             (uint32_t(bf16_bits(hash_val(seed, e0 + 2 * q + 1, scale))) << 16);
    *reinterpret_cast<uint4*>(dst + s * slot_elems + e0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__global__ void fill_kernel(uint16_t* __restrict__ dst, int64_t n, uint64_t seed, float scale) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = bf16_bits(hash_val(seed, i, scale));
}

__global__ void fill_f32_kernel(float* __restrict__ dst, int64_t n, uint64_t seed, float scale) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = hash_val(seed, i, scale);
}

// ---------------------------------------------------------------- fp8 (e4m3)
// fp32 -> e4m3 (OCP E4M3, no inf): round to nearest even on the integer
// mantissa, saturate to +-448. Same integer recipe as oracle_f32_to_e4m3.
__device__ __forceinline__ uint8_t f32_to_e4m3(float x) {
  const uint32_t u = __float_as_uint(x);
  const uint32_t s = (u >> 24) & 0x80u;
  const uint32_t a = u & 0x7fffffffu;
  if (a > 0x7f800000u) return uint8_t(s | 0x7f);  // NaN
  if (a >= 0x43e00000u) return uint8_t(s | 0x7e);  // >= 448: saturate
  const int e = int(a >> 23) - 127;
  if (e < -6) {  // subnormal: multiple of 2^-9, RNE
    const float q = rintf(__fmul_rn(__uint_as_float(a), 512.0f));
    return uint8_t(s | uint32_t(q));  // q == 8 encodes the min normal 0x08
  }
  const uint32_t m = a & 0x7fffffu;
  uint32_t m3 = m >> 20;
  const uint32_t rem = m & 0xfffffu;
  if (rem > 0x80000u || (rem == 0x80000u && (m3 & 1u))) ++m3;
  uint32_t code = (uint32_t(e + 7) << 3) + m3;  // mantissa carry bumps the exponent
  if (code > 0x7e) code = 0x7e;
  return uint8_t(s | code);
}

// Quantised synthetic expert weights: one warp per (slot, row); the row's
// bf16 values come from the same counter hash as the bf16 init; scale =
// absmax / 448 (1 if the row is zero), q = e4m3(v / scale).
__global__ void __launch_bounds__(256) fp8_fill_rows_kernel(uint8_t* __restrict__ dst,
                                                            float* __restrict__ scales,
                                                            const uint64_t* __restrict__ seeds,
                                                            int nslots, int rows, int64_t K,
                                                            float scale) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= int64_t(nslots) * rows) return;
  const int64_t slot = wid / rows, r = wid - slot * rows;
  const uint64_t seed = seeds[slot];
  auto val = [&](int64_t k) { return bf16_f(bf16_bits(hash_val(seed, r * K + k, scale))); };
  float amax = 0.0f;
  for (int64_t k = lane; k < K; k += 32) amax = fmaxf(amax, fabsf(val(k)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float s = amax > 0.0f ? __fdiv_rn(amax, 448.0f) : 1.0f;
  uint8_t* out = dst + (slot * rows + r) * K;
  for (int64_t k = lane * 4; k < K; k += 128) {
    uint32_t w = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) w |= uint32_t(f32_to_e4m3(__fdiv_rn(val(k + q), s))) << (8 * q);
    *reinterpret_cast<uint32_t*>(out + k) = w;
  }
  if (lane == 0) scales[slot * rows + r] = s;
}

// One warp per bf16 row: per-row e4m3 quantisation (scale = absmax / 448).
__device__ __forceinline__ float row_absmax_bf16(const uint4* row, int64_t nch, int lane) {
  float amax = 0.0f;
#pragma unroll 4
  for (int64_t c = lane; c < nch; c += 32) {
    const uint4 v = __ldg(row + c);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
      amax = fmaxf(amax, fmaxf(fabsf(__uint_as_float(w[q] << 16)),
                               fabsf(__uint_as_float(w[q] & 0xffff0000u))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  return amax;
}

__device__ __forceinline__ uint2 quant8(uint4 v, float s) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t o[2] = {0, 0};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    o[q >> 1] |= uint32_t(f32_to_e4m3(__fdiv_rn(__uint_as_float(w[q] << 16), s))) << (16 * (q & 1));
    o[q >> 1] |= uint32_t(f32_to_e4m3(__fdiv_rn(__uint_as_float(w[q] & 0xffff0000u), s)))
                 << (16 * (q & 1) + 8);
  }
  return make_uint2(o[0], o[1]);
}

// ---------------------------------------------------------------- NVFP4
// Two-level NVFP4 (W4A4, tcgen05 kind::mxf4nvf4 block16): per row an fp32
// scale s = absmax / (448 * 6); per 16-element block an e4m3 scale code
// sf = e4m3(block_absmax / (6 s)); elements q = e2m1(v * rcp(e4m3(sf) * s))
// with the hardware conversion (cvt.rn.satfinite.e2m1x2.f32: round to
// nearest even on {0, .5, 1, 1.5, 2, 3, 4, 6}, saturating, sign kept) and a
// correctly rounded reciprocal. Same float sequence as oracle_nvfp4_quant_row.
// Work unit: one lane quantises a 64-element group (4 blocks) -> 32 bytes of
// codes (element 2i in the low nibble of byte i) + one 32-bit word of the 4
// block scales, which nvfp4_sf_offset keeps contiguous.
__device__ __forceinline__ float e4m3_to_f32(uint32_t b) {
  const uint32_t e = (b >> 3) & 0xfu, m = b & 7u;
  const float v = e ? __uint_as_float(((e + 120u) << 23) | (m << 20)) : float(m) * 0.001953125f;
  return (b & 0x80u) ? -v : v;
}
// 8 values -> 8 e2m1 codes, element i in nibble i
__device__ __forceinline__ uint32_t e2m1x8(const float* v, float inv) {
  uint32_t out;
  asm("{\n.reg .b8 b0, b1, b2, b3;\n"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n"
      "cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n"
      "cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n"
      "mov.b32 %0, {b0, b1, b2, b3};\n}"
      : "=r"(out)
      : "f"(__fmul_rn(v[0], inv)), "f"(__fmul_rn(v[1], inv)), "f"(__fmul_rn(v[2], inv)),
        "f"(__fmul_rn(v[3], inv)), "f"(__fmul_rn(v[4], inv)), "f"(__fmul_rn(v[5], inv)),
        "f"(__fmul_rn(v[6], inv)), "f"(__fmul_rn(v[7], inv)));
  return out;
}
// 64 values (4 blocks) -> codes c[0..7] (32 bytes) and the 4 block-scale codes.
__device__ __forceinline__ uint32_t nvfp4_group(const float* v, float s, uint32_t* c) {
  const float s6 = __fmul_rn(6.0f, s);
  uint32_t sfw = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    float bmax = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) bmax = fmaxf(bmax, fabsf(v[16 * b + i]));
    const uint32_t sf = f32_to_e4m3(__fdiv_rn(bmax, s6));
    const float ds = __fmul_rn(e4m3_to_f32(sf), s);
    const float inv = ds > 0.0f ? __frcp_rn(ds) : 0.0f;
    c[2 * b] = e2m1x8(v + 16 * b, inv);
    c[2 * b + 1] = e2m1x8(v + 16 * b + 8, inv);
    sfw |= sf << (8 * b);
  }
  return sfw;
}
__device__ __forceinline__ float nvfp4_row_scale(float amax) {
  return amax > 0.0f ? __fdiv_rn(amax, 2688.0f) : 1.0f;
}
// 8 uint4 of bf16 (64 elements) -> floats
__device__ __forceinline__ void unpack_bf16x64(const uint4* q, float* v) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t w[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[8 * j + 2 * i] = __uint_as_float(w[i] << 16);
      v[8 * j + 2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
}
// Block scales go to the atom layout directly (init-time weights) or, on
// the per-step paths, to a linear [row][K/16] buffer: 4-byte atom stores
// from scattered rows are partial-sector writes that HBM turns into
// read-modify-writes; nvfp4_sf_relayout_kernel then builds whole atoms.
__device__ __forceinline__ void store_group(uint8_t* codes_row, uint8_t* sf, int64_t r, int64_t g, int64_t K,
                                            const uint32_t* c, uint32_t sfw, bool linear) {
  uint4* o = reinterpret_cast<uint4*>(codes_row + g * 32);
  o[0] = make_uint4(c[0], c[1], c[2], c[3]);
  o[1] = make_uint4(c[4], c[5], c[6], c[7]);
  *reinterpret_cast<uint32_t*>(sf + (linear ? r * (K / 16) + 4 * g : nvfp4_sf_offset(r, 4 * g, K))) = sfw;
}

// Linear block scales [rows][K/16] -> 512-byte atoms (rows < meta[0]*128, or
// all max_rows rows padded to 128 when meta is null); one thread per
// destination word (the 4 scales of one row and 64-column chunk).
__global__ void __launch_bounds__(256) nvfp4_sf_relayout_kernel(const uint32_t* __restrict__ lin,
                                                                uint32_t* __restrict__ atoms,
                                                                int64_t max_rows, int64_t K,
                                                                const int32_t* __restrict__ meta) {
  const int64_t nc = K / 64;
  const int64_t rows = meta ? int64_t(meta[0]) * 128 : (max_rows + 127) / 128 * 128;
  const int64_t words = rows * nc;
  for (int64_t d = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; d < words;
       d += int64_t(gridDim.x) * blockDim.x) {
    const int64_t mb = d / (nc * 128), rem = d - mb * nc * 128;
    const int64_t c = rem >> 7, w = rem & 127;
    const int64_t r = mb * 128 + (w >> 2) + 32 * (w & 3);
    atoms[d] = r < max_rows ? __ldg(lin + r * nc + c) : 0u;
  }
}

// Synthetic NVFP4 expert weights: one warp per (slot, row) over the same
// bf16 counter-hash values as the bf16 init.
__global__ void __launch_bounds__(256) nvfp4_fill_rows_kernel(uint8_t* __restrict__ dst,
                                                              uint8_t* __restrict__ sfa,
                                                              float* __restrict__ scales,
                                                              const uint64_t* __restrict__ seeds,
                                                              int nslots, int rows, int64_t K,
                                                              float scale) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= int64_t(nslots) * rows) return;
  const int64_t slot = wid / rows, r = wid - slot * rows;
  const uint64_t seed = seeds[slot];
  auto val = [&](int64_t k) { return bf16_f(bf16_bits(hash_val(seed, r * K + k, scale))); };
  float amax = 0.0f;
  for (int64_t k = lane; k < K; k += 32) amax = fmaxf(amax, fabsf(val(k)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float s = nvfp4_row_scale(amax);
  uint8_t* sf_slot = sfa + slot * int64_t(rows) * (K / 16);
  for (int64_t g = lane; g < K / 64; g += 32) {
    float v[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = val(g * 64 + i);
    uint32_t c[8];
    const uint32_t sfw = nvfp4_group(v, s, c);
    store_group(dst + (slot * rows + r) * (K / 2), sf_slot, r, g, K, c, sfw, false);
  }
  if (lane == 0) scales[slot * rows + r] = s;
}

// bf16 rows (rows < meta[0]*128) -> NVFP4 codes + block scales + row scale.
__global__ void __launch_bounds__(256) quant_rows_nvfp4_kernel(const uint16_t* __restrict__ src,
                                                               int64_t max_rows, int64_t K,
                                                               const int32_t* __restrict__ meta,
                                                               uint8_t* __restrict__ dst,
                                                               uint8_t* __restrict__ sfl,
                                                               float* __restrict__ scales) {
  const int lane = threadIdx.x & 31;
  const int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t rows = meta ? int64_t(meta[0]) * 128 : max_rows;
  if (r >= rows) return;
  const uint4* row = reinterpret_cast<const uint4*>(src + r * K);
  const int64_t ng = K / 64;
  if (ng <= 32) {  // one group per lane: the row is read once, into registers
    uint4 q[8];
    float amax = 0.0f;
    if (lane < ng) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        q[j] = __ldg(row + 8 * lane + j);
        const uint32_t w[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          amax = fmaxf(amax, fmaxf(fabsf(__uint_as_float(w[i] << 16)),
                                   fabsf(__uint_as_float(w[i] & 0xffff0000u))));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const float s = nvfp4_row_scale(amax);
    if (lane < ng) {
      float v[64];
      unpack_bf16x64(q, v);
      uint32_t c[8];
      const uint32_t sfw = nvfp4_group(v, s, c);
      store_group(dst + r * (K / 2), sfl, r, lane, K, c, sfw, true);
    }
    if (lane == 0) scales[r] = s;
    return;
  }
  const float s = nvfp4_row_scale(row_absmax_bf16(row, K / 8, lane));
  for (int64_t g = lane; g < ng; g += 32) {
    uint4 q[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) q[j] = __ldg(row + 8 * g + j);
    float v[64];
    unpack_bf16x64(q, v);
    uint32_t c[8];
    const uint32_t sfw = nvfp4_group(v, s, c);
    store_group(dst + r * (K / 2), sfl, r, g, K, c, sfw, true);
  }
  if (lane == 0) scales[r] = s;
}

// Short rows (K <= 2048, K % 256 == 0; GEMM2's H): lane-interleaved, so every
// load and code store of the warp is one contiguous 512 / 128-byte run (the
// group-per-lane layout above reads 16 B from each of 32 lines per
// instruction). A 16-element block spans a lane pair (block max by one
// shuffle); lanes 8c..8c+7 hold the four blocks of one 64-column chunk, whose
// scale word lane 8c writes. Same float sequence per element as nvfp4_group.
template <int NJ>
__global__ void __launch_bounds__(256) quant_rows_nvfp4_il_kernel(const uint16_t* __restrict__ src,
                                                                  int64_t max_rows,
                                                                  const int32_t* __restrict__ meta,
                                                                  uint8_t* __restrict__ dst,
                                                                  uint8_t* __restrict__ sfl,
                                                                  float* __restrict__ scales) {
  constexpr int64_t K = int64_t(NJ) * 256;
  const int lane = threadIdx.x & 31;
  const int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t rows = meta ? int64_t(meta[0]) * 128 : max_rows;
  if (r >= rows) return;
  const uint4* row = reinterpret_cast<const uint4*>(src + r * K);
  uint4 q[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) q[j] = __ldg(row + j * 32 + lane);
  float amax = 0.0f;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const uint32_t w[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      amax = fmaxf(amax, fmaxf(fabsf(__uint_as_float(w[i] << 16)), fabsf(__uint_as_float(w[i] & 0xffff0000u))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float s = nvfp4_row_scale(amax);
  const float s6 = __fmul_rn(6.0f, s);
  uint32_t* codes = reinterpret_cast<uint32_t*>(dst + r * (K / 2));
  uint32_t* sfw = reinterpret_cast<uint32_t*>(sfl + r * (K / 16));
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    float v[8];
    const uint32_t w[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
    float bmax = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) bmax = fmaxf(bmax, fabsf(v[i]));
    bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, 1));
    const uint32_t sf = f32_to_e4m3(__fdiv_rn(bmax, s6));
    const float ds = __fmul_rn(e4m3_to_f32(sf), s);
    const float inv = ds > 0.0f ? __frcp_rn(ds) : 0.0f;
    codes[j * 32 + lane] = e2m1x8(v, inv);
    // scale bytes of blocks 2m (lane 2m) -> word of chunk lane/8
    uint32_t word = sf << (8 * ((lane >> 1) & 3));
    word |= __shfl_xor_sync(0xffffffffu, word, 2);
    word |= __shfl_xor_sync(0xffffffffu, word, 4);
    if ((lane & 7) == 0) sfw[j * 4 + (lane >> 3)] = word;
  }
  if (lane == 0) scales[r] = s;
}

// H (bf16, rows < meta[0]*128) -> e4m3 + per-row scale (GEMM2's A operand).
__global__ void __launch_bounds__(256) quant_rows_fp8_kernel(const uint16_t* __restrict__ src,
                                                             int64_t max_rows, int64_t K,
                                                             const int32_t* __restrict__ meta,
                                                             uint8_t* __restrict__ dst,
                                                             float* __restrict__ scales) {
  const int lane = threadIdx.x & 31;
  const int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t rows = meta ? int64_t(meta[0]) * 128 : max_rows;
  if (r >= rows) return;
  const uint4* row = reinterpret_cast<const uint4*>(src + r * K);
  const int64_t nch = K / 8;
  const float amax = row_absmax_bf16(row, nch, lane);
  const float s = amax > 0.0f ? __fdiv_rn(amax, 448.0f) : 1.0f;
  uint2* out = reinterpret_cast<uint2*>(dst + r * K);
  for (int64_t c = lane; c < nch; c += 32) out[c] = quant8(__ldg(row + c), s);
  if (lane == 0) scales[r] = s;
}

// ---------------------------------------------------------------- router
// SIMT fp32 GEMM, 128 tokens x 128 experts per CTA, 8x8 outputs per thread.
// Every output accumulates fma(x[t][i], w[e][i], acc) for i ascending.
constexpr int RB_M = 128, RB_N = 128, RB_K = 16;

__global__ void __launch_bounds__(256) router_logits_kernel(const uint16_t* __restrict__ x,
                                                            const uint16_t* __restrict__ w,
                                                            float* __restrict__ logits, int64_t T,
                                                            int E, int64_t K) {
  __shared__ __align__(16) float As[2][RB_K][RB_M];
  __shared__ __align__(16) float Bs[2][RB_K][RB_N];
  const int tid = threadIdx.x;
  const int64_t m0 = int64_t(blockIdx.x) * RB_M;
  const int n0 = blockIdx.y * RB_N;
  // loader: thread -> (row = tid / 2, 8 consecutive k at (tid % 2) * 8)
  const int lr = tid >> 1, lk = (tid & 1) * 8;
  const bool a_ok = m0 + lr < T, b_ok = n0 + lr < E;
  const uint16_t* ap = x + (m0 + lr) * K + lk;
  const uint16_t* bp = w + int64_t(n0 + lr) * K + lk;
  uint4 ra = make_uint4(0, 0, 0, 0), rb = make_uint4(0, 0, 0, 0);
  auto gload = [&](int64_t k0) {
    ra = a_ok ? *reinterpret_cast<const uint4*>(ap + k0) : make_uint4(0, 0, 0, 0);
    rb = b_ok ? *reinterpret_cast<const uint4*>(bp + k0) : make_uint4(0, 0, 0, 0);
  };
  auto sstore = [&](int buf) {
    const uint32_t av[4] = {ra.x, ra.y, ra.z, ra.w}, bv[4] = {rb.x, rb.y, rb.z, rb.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      As[buf][lk + 2 * q][lr] = __uint_as_float(av[q] << 16);
      As[buf][lk + 2 * q + 1][lr] = __uint_as_float(av[q] & 0xffff0000u);
      Bs[buf][lk + 2 * q][lr] = __uint_as_float(bv[q] << 16);
      Bs[buf][lk + 2 * q + 1][lr] = __uint_as_float(bv[q] & 0xffff0000u);
    }
  };
  // compute mapping: rows {ty*4 + i, 64 + ty*4 + i}, cols {tx*4 + j, 64 + tx*4 + j}
  const int tx = tid & 15, ty = tid >> 4;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

  const int64_t nk = K / RB_K;
  gload(0);
  sstore(0);
  __syncthreads();
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int buf = int(kt & 1);
    if (kt + 1 < nk) gload((kt + 1) * RB_K);
#pragma unroll
    for (int kk = 0; kk < RB_K; ++kk) {
      float a[8], b[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
    }
    if (kt + 1 < nk) sstore(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t t = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (t >= T) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (e < E) logits[t * E + e] = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------- top-k
__device__ __forceinline__ float det_expf(float x) {
  if (x < -87.0f) return 0.0f;
  if (x > 88.0f) return __int_as_float(0x7f800000);
  const float n = rintf(__fmul_rn(x, 1.44269504088896341f));
  float r = __fmaf_rn(n, -0.693145751953125f, x);
  r = __fmaf_rn(n, -1.428606765330187e-06f, r);
  float p = 1.38888889e-3f;
  p = __fmaf_rn(p, r, 8.33333333e-3f);
  p = __fmaf_rn(p, r, 4.16666667e-2f);
  p = __fmaf_rn(p, r, 1.66666667e-1f);
  p = __fmaf_rn(p, r, 0.5f);
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  // n in [-126, 127] and p in (0.7, 1.42): one correctly rounded multiply by
  // the exact power of two equals ldexpf(p, n) (the oracle's formulation).
  return __fmul_rn(p, __int_as_float((int(n) + 127) << 23));
}

__device__ __forceinline__ bool better(float a, int ia, float b, int ib) {
  return a > b || (a == b && ia < ib);
}

// Warp argmax over (value, index) pairs; lanes holding no candidate pass
// (-inf, INT_MAX). Returns the winner on all lanes.
__device__ __forceinline__ void warp_best(float& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (better(ov, oi, v, i)) {
      v = ov;
      i = oi;
    }
  }
}

constexpr int TOPK_MAXV = 16;  // E <= 512
constexpr int TOPK_MAXK = 16;

// Exact logit from the 9 digit-plane products: Z = sum_{a,b} 2^{8(a+b)} C_ab
// (int64, exact), rounded once to fp32, scaled by the row exponents.
__device__ __forceinline__ float exact_logit(const int32_t* __restrict__ C, int64_t T, int E,
                                             int64_t t, int e, int sx) {
  long long z = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      z += static_cast<long long>(C[(a * T + t) * (3 * E) + b * E + e]) * (1LL << (8 * (a + b)));
  const float f = __ll2float_rn(z);
  // exact power-of-two scaling == ldexpf whenever 2^sx is a normal float
  return (sx >= -126 && sx <= 127) ? __fmul_rn(f, __int_as_float((sx + 127) << 23)) : ldexpf(f, sx);
}

__global__ void __launch_bounds__(256) topk_kernel(const int32_t* __restrict__ C,
                                                   const int32_t* __restrict__ ex,
                                                   const int32_t* __restrict__ ew,
                                                   const float* __restrict__ bias,
                                                   float* __restrict__ logits,
                                                   int32_t* __restrict__ idx_out,
                                                   float* __restrict__ wts_out, int64_t T,
                                                   RouterCfg c) {
  const int lane = threadIdx.x & 31;
  const int64_t t = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  const int E = c.E;
  const int V = (E + 31) >> 5;
  const float NEG = __int_as_float(0xff800000);
  float lg[TOPK_MAXV], sc[TOPK_MAXV], ch[TOPK_MAXV];
  float* row = logits + t * E;
  const int xe = ex[t];
#pragma unroll
  for (int v = 0; v < TOPK_MAXV; ++v) {
    const int e = lane + 32 * v;
    if (v < V && e < E) {
      lg[v] = exact_logit(C, T, E, t, e, xe + ew[e] - 296);
      row[e] = lg[v];
      if (c.scoring == 1) {
        sc[v] = __fdiv_rn(1.0f, __fadd_rn(1.0f, det_expf(-lg[v])));
        ch[v] = __fadd_rn(sc[v], bias ? bias[e] : 0.0f);
      } else {
        sc[v] = lg[v];
        ch[v] = lg[v];
      }
    } else {
      lg[v] = sc[v] = ch[v] = NEG;
    }
  }
  const int G = c.n_group > 0 ? c.n_group : 1;
  if (G > 1 && c.topk_group < G) {
    const int gs = E / G;
    int grp[TOPK_MAXV];  // group of each of this lane's slots (one division per slot)
#pragma unroll
    for (int v = 0; v < TOPK_MAXV; ++v) {
      const int e = lane + 32 * v;
      grp[v] = (v < V && e < E) ? e / gs : -1;
    }
    uint32_t gsel = 0;        // bit g: group kept (G <= 32)
    float gscore_mine = NEG;  // lane g holds group g's score
    for (int g = 0; g < G; ++g) {
      // top-2 of the group: one lane-local pass keeping the best two, then
      // two warp reductions (the second excludes the first winner)
      float v1 = NEG, v2 = NEG;
      int i1 = 0x7fffffff, i2 = 0x7fffffff;
#pragma unroll
      for (int v = 0; v < TOPK_MAXV; ++v) {
        if (grp[v] != g) continue;
        const int e = lane + 32 * v;
        if (better(ch[v], e, v1, i1)) {
          v2 = v1;
          i2 = i1;
          v1 = ch[v];
          i1 = e;
        } else if (better(ch[v], e, v2, i2)) {
          v2 = ch[v];
          i2 = e;
        }
      }
      float w1 = v1;
      int j1 = i1;
      warp_best(w1, j1);
      // runner-up: this lane's best candidate other than the winner
      float w2 = (i1 == j1) ? v2 : v1;
      int j2 = (i1 == j1) ? i2 : i1;
      warp_best(w2, j2);
      const float gsc = gs >= 2 ? __fadd_rn(w1, w2) : w1;
      if (lane == g) gscore_mine = gsc;
    }
    for (int s = 0; s < c.topk_group; ++s) {
      float v = (lane < G && !((gsel >> lane) & 1u)) ? gscore_mine : NEG;
      int i = (lane < G && !((gsel >> lane) & 1u)) ? lane : 0x7fffffff;
      warp_best(v, i);
      gsel |= 1u << i;
    }
#pragma unroll
    for (int v = 0; v < TOPK_MAXV; ++v)
      if (grp[v] >= 0 && !((gsel >> grp[v]) & 1u)) ch[v] = 0.0f;  // HF masked_fill 0.0
  }
  // top-k over ch, ties to the lower index
  int sel[TOPK_MAXK];
  uint32_t taken_mask = 0;  // bit v of this lane's slots
  for (int j = 0; j < c.k; ++j) {
    float bv = NEG;
    int bi = 0x7fffffff;
#pragma unroll
    for (int v = 0; v < TOPK_MAXV; ++v) {
      const int e = lane + 32 * v;
      if (v < V && e < E && !((taken_mask >> v) & 1u) && better(ch[v], e, bv, bi)) {
        bv = ch[v];
        bi = e;
      }
    }
    warp_best(bv, bi);
    sel[j] = bi;
    if ((bi & 31) == lane) taken_mask |= 1u << (bi >> 5);
  }
  // weights: fetch the winners' score / logit from their owning lanes
  float wv[TOPK_MAXK];
  for (int j = 0; j < c.k; ++j) {
    const int e = sel[j];
    float mine = 0.0f;
#pragma unroll
    for (int v = 0; v < TOPK_MAXV; ++v)
      if (v == (e >> 5)) mine = (c.scoring == 1) ? sc[v] : lg[v];
    wv[j] = __shfl_sync(0xffffffffu, mine, e & 31);
  }
  __syncwarp();  // logits row written by all lanes is read by lane 0 below
  if (lane != 0) return;
  if (c.scoring == 1) {
    if (c.norm_topk) {
      float s = 0.0f;
      for (int j = 0; j < c.k; ++j) s = __fadd_rn(s, wv[j]);
      s = __fadd_rn(s, 1e-20f);
      for (int j = 0; j < c.k; ++j) wv[j] = __fdiv_rn(wv[j], s);
    }
  } else {
    const float m = wv[0];
    float s = 0.0f;
    for (int j = 0; j < c.k; ++j) {
      wv[j] = det_expf(__fsub_rn(wv[j], m));
      if (c.norm_topk) s = __fadd_rn(s, wv[j]);
    }
    if (!c.norm_topk)
      for (int e = 0; e < E; ++e) s = __fadd_rn(s, det_expf(__fsub_rn(row[e], m)));
    for (int j = 0; j < c.k; ++j) wv[j] = __fdiv_rn(wv[j], s);
  }
  for (int j = 0; j < c.k; ++j) {
    idx_out[t * c.k + j] = sel[j];
    wts_out[t * c.k + j] = __fmul_rn(wv[j], c.routed_scale);
  }
}

// Same contract as topk_kernel for E = 32*V with every lane's V experts in
// one routing group (E % 32 == 0, (E / n_group) % V == 0): lane l owns the
// contiguous experts [V*l, V*l + V), so the 9 plane products are read as int4
// vectors, a group's top-2 is a lane-local top-2 merged over the group's
// E/(n_group*V) lanes (two xor shuffles for R1) and the kept groups are
// ranked from G broadcast scores. Results are bit-identical to topk_kernel.
// FROM_LOGITS: the logits were already formed (router GEMM with the
// recombination fused, launch_router_gemm); read them instead of C.
template <int V, bool FROM_LOGITS>
__global__ void __launch_bounds__(256) topk_contig_kernel(const int32_t* __restrict__ C,
                                                          const int32_t* __restrict__ ex,
                                                          const int32_t* __restrict__ ew,
                                                          const float* __restrict__ bias,
                                                          float* __restrict__ logits,
                                                          int32_t* __restrict__ idx_out,
                                                          float* __restrict__ wts_out, int64_t T,
                                                          RouterCfg c) {
  const int lane = threadIdx.x & 31;
  const int64_t t = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  const int E = c.E;
  const int e0 = V * lane;
  const float NEG = __int_as_float(0xff800000);
  long long z[V];
#pragma unroll
  for (int i = 0; i < V; ++i) z[i] = 0;
#pragma unroll
  for (int a = 0; a < (FROM_LOGITS ? 0 : 3); ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const int32_t* src = C + (a * T + t) * (3 * E) + b * E + e0;
      int32_t w[V];
      if (V % 4 == 0) {
#pragma unroll
        for (int i = 0; i < V; i += 4) {
          const int4 q = __ldg(reinterpret_cast<const int4*>(src + i));
          w[i] = q.x;
          w[i + 1] = q.y;
          w[i + 2] = q.z;
          w[i + 3] = q.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) w[i] = __ldg(src + i);
      }
#pragma unroll
      for (int i = 0; i < V; ++i) z[i] += static_cast<long long>(w[i]) * (1LL << (8 * (a + b)));
    }
  const int xe = ex[t];
  float lg[V], sc[V], ch[V];
  float* row = logits + t * E;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    if (FROM_LOGITS) {
      lg[i] = row[e0 + i];
    } else {
      const int sx = xe + ew[e0 + i] - 296;
      const float f = __ll2float_rn(z[i]);
      lg[i] = (sx >= -126 && sx <= 127) ? __fmul_rn(f, __int_as_float((sx + 127) << 23)) : ldexpf(f, sx);
      row[e0 + i] = lg[i];
    }
    if (c.scoring == 1) {
      sc[i] = __fdiv_rn(1.0f, __fadd_rn(1.0f, det_expf(-lg[i])));
      ch[i] = __fadd_rn(sc[i], bias ? bias[e0 + i] : 0.0f);
    } else {
      sc[i] = lg[i];
      ch[i] = lg[i];
    }
  }
  const int G = c.n_group > 0 ? c.n_group : 1;
  if (G > 1 && c.topk_group < G) {
    const int gs = E / G, lpg = gs / V;  // experts and lanes per group
    // lane-local top-2 values, then merge across the group's lanes
    float v1 = NEG, v2 = NEG;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      if (ch[i] > v1) {
        v2 = v1;
        v1 = ch[i];
      } else if (ch[i] > v2) {
        v2 = ch[i];
      }
    }
    for (int o = 1; o < lpg; o <<= 1) {
      const float o1 = __shfl_xor_sync(0xffffffffu, v1, o);
      const float o2 = __shfl_xor_sync(0xffffffffu, v2, o);
      const float hi = fmaxf(v1, o1);
      const float lo = fmaxf(fminf(v1, o1), fmaxf(v2, o2));
      v1 = hi;
      v2 = lo;
    }
    const float gsc = gs >= 2 ? __fadd_rn(v1, v2) : v1;
    const int g = lane / lpg;
    int rank = 0;
    for (int h = 0; h < G; ++h) {
      const float sh = __shfl_sync(0xffffffffu, gsc, h * lpg);
      rank += (sh > gsc || (sh == gsc && h < g)) ? 1 : 0;
    }
    if (rank >= c.topk_group)
#pragma unroll
      for (int i = 0; i < V; ++i) ch[i] = 0.0f;  // HF masked_fill 0.0
  }
  int sel[TOPK_MAXK];
  uint32_t taken = 0;
  for (int j = 0; j < c.k; ++j) {
    float bv = NEG;
    int bi = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < V; ++i)
      if (!((taken >> i) & 1u) && better(ch[i], e0 + i, bv, bi)) {
        bv = ch[i];
        bi = e0 + i;
      }
    warp_best(bv, bi);
    sel[j] = bi;
    if (bi / V == lane) taken |= 1u << (bi - e0);
  }
  float wv[TOPK_MAXK];
  for (int j = 0; j < c.k; ++j) {
    const int e = sel[j];
    float mine = 0.0f;
#pragma unroll
    for (int i = 0; i < V; ++i)
      if (e0 + i == e) mine = (c.scoring == 1) ? sc[i] : lg[i];
    wv[j] = __shfl_sync(0xffffffffu, mine, e / V);
  }
  __syncwarp();
  if (lane != 0) return;
  if (c.scoring == 1) {
    if (c.norm_topk) {
      float s = 0.0f;
      for (int j = 0; j < c.k; ++j) s = __fadd_rn(s, wv[j]);
      s = __fadd_rn(s, 1e-20f);
      for (int j = 0; j < c.k; ++j) wv[j] = __fdiv_rn(wv[j], s);
    }
  } else {
    const float m = wv[0];
    float s = 0.0f;
    for (int j = 0; j < c.k; ++j) {
      wv[j] = det_expf(__fsub_rn(wv[j], m));
      if (c.norm_topk) s = __fadd_rn(s, wv[j]);
    }
    if (!c.norm_topk)
      for (int e = 0; e < E; ++e) s = __fadd_rn(s, det_expf(__fsub_rn(row[e], m)));
    for (int j = 0; j < c.k; ++j) wv[j] = __fdiv_rn(wv[j], s);
  }
  for (int j = 0; j < c.k; ++j) {
    idx_out[t * c.k + j] = sel[j];
    wts_out[t * c.k + j] = __fmul_rn(wv[j], c.routed_scale);
  }
}

// ---------------------------------------------------------------- router quant
// bf16 bits -> (mantissa incl. implicit bit, exponent field clamped to >= 1)
__device__ __forceinline__ void bf16_fields(uint32_t b, int& mant, int& eb) {
  const int E = int((b >> 7) & 0xFFu), M = int(b & 0x7Fu);
  mant = E ? (M | 0x80) : M;
  eb = E ? E : 1;
}

__device__ __forceinline__ int fixed22(uint32_t b, int emax) {
  int mant, eb;
  bf16_fields(b, mant, eb);
  const int sh = eb - emax + 14;
  int q = sh >= 0 ? (mant << sh) : (sh > -8 ? (mant >> -sh) : 0);
  return (b & 0x8000u) ? -q : q;
}

// One warp per row: pass 1 finds the row exponent, pass 2 writes the three
// balanced int8 digit planes (Q = d0 + 256 d1 + 65536 d2, |Q| < 2^22).
constexpr int RQ_WARPS = 2;   // rows (warps) per CTA when the rows are staged in smem
constexpr int RQ_UNROLL = 7;  // 16-byte loads in flight per lane (h = 7168: 4 x 7 x 32 chunks)

__global__ void __launch_bounds__(256) router_quant_kernel(const uint16_t* __restrict__ src,
                                                           int64_t R, int64_t K,
                                                           int8_t* __restrict__ dst,
                                                           int32_t* __restrict__ emax,
                                                           int32_t* __restrict__ meta, int staged) {
  if (meta && blockIdx.x == 0 && threadIdx.x == 0) {
    const int mb = int((3 * R + 255) / 256) * 2;  // even: whole CTA-pair tiles (rows >= 3R not stored)
    meta[0] = mb;
    meta[1] = mb;
    meta[2] = 0;
    meta[3] = 0;
  }
  const int lane = threadIdx.x & 31;
  const int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= R) return;
  const uint4* row = reinterpret_cast<const uint4*>(src + r * K);
  const int64_t nch = K / 8;
  extern __shared__ uint4 rq_rows[];  // [warps per block][nch] when staged
  if (staged) {  // one HBM read: pass 1 stages the row in smem, pass 2 quantises from it
    // Pass 1: the row's largest magnitude (sign-cleared bf16 bits order like
    // the values) gives the exponent field emax, two elements per __vmaxu2.
    uint4* srow = rq_rows + (threadIdx.x >> 5) * nch;
    uint32_t mx = 0;
    for (int64_t c0 = lane; c0 < nch; c0 += 32 * RQ_UNROLL) {
      uint4 v[RQ_UNROLL];
#pragma unroll
      for (int u = 0; u < RQ_UNROLL; ++u) {
        const int64_t c = c0 + 32 * u;
        v[u] = c < nch ? __ldg(row + c) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < RQ_UNROLL; ++u) {
        const int64_t c = c0 + 32 * u;
        if (c < nch) srow[c] = v[u];
        mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(v[u].x & 0x7FFF7FFFu, v[u].y & 0x7FFF7FFFu),
                                   __vmaxu2(v[u].z & 0x7FFF7FFFu, v[u].w & 0x7FFF7FFFu)));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = __vmaxu2(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const uint32_t top = max(mx & 0xFFFFu, mx >> 16);
    const int m = top ? max(int(top >> 7), 1) : 1;  // = max over nonzero elements of max(E, 1)
    // Pass 2: Q = trunc(x * 2^(148 - emax)) (exact: a bf16 times a power of
    // two; |Q| < 2^22), digits of Q = d0 + 2^8 d1 + 2^16 d2 in [-128, 127]:
    // Q1 = (Q + 128) >> 8, Q2 = (Q1 + 128) >> 8, digits = their low bytes.
    const int kx = 148 - m;  // in [-106, 147]: beyond 127 split into 2^64 * 2^(kx-64)
    const float s1 = __int_as_float(((kx > 127 ? 64 : kx) + 127) << 23);
    const float s2 = kx > 127 ? __int_as_float((kx - 64 + 127) << 23) : 1.0f;
    __syncwarp();
    for (int64_t c = lane; c < nch; c += 32) {
      const uint4 v = srow[c];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      uint32_t p[3][2];
#pragma unroll
      for (int hw = 0; hw < 2; ++hw) {  // two words = four elements per packed plane word
        int q0[4], q1[4], q2[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t word = w[2 * hw + (e >> 1)];
          const float f = __uint_as_float((e & 1) ? (word & 0xFFFF0000u) : (word << 16));
          q0[e] = __float2int_rz(__fmul_rn(__fmul_rn(f, s1), s2));
          q1[e] = (q0[e] + 128) >> 8;
          q2[e] = (q1[e] + 128) >> 8;
        }
        p[0][hw] = __byte_perm(__byte_perm(q0[0], q0[1], 0x40), __byte_perm(q0[2], q0[3], 0x40), 0x5410);
        p[1][hw] = __byte_perm(__byte_perm(q1[0], q1[1], 0x40), __byte_perm(q1[2], q1[3], 0x40), 0x5410);
        p[2][hw] = __byte_perm(__byte_perm(q2[0], q2[1], 0x40), __byte_perm(q2[2], q2[3], 0x40), 0x5410);
      }
      *reinterpret_cast<uint2*>(dst + (0 * R + r) * K + c * 8) = make_uint2(p[0][0], p[0][1]);
      *reinterpret_cast<uint2*>(dst + (1 * R + r) * K + c * 8) = make_uint2(p[1][0], p[1][1]);
      *reinterpret_cast<uint2*>(dst + (2 * R + r) * K + c * 8) = make_uint2(p[2][0], p[2][1]);
    }
    if (lane == 0) emax[r] = m;
    return;
  }
  int m = 0;
  for (int64_t c = lane; c < nch; c += 32) {
    const uint4 v = __ldg(row + c);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      int mant, eb;
      bf16_fields((w[q >> 1] >> (16 * (q & 1))) & 0xFFFFu, mant, eb);
      if (mant && eb > m) m = eb;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (m == 0) m = 1;
  for (int64_t c = lane; c < nch; c += 32) {
    const uint4 v = __ldg(row + c);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t p0[2] = {0, 0}, p1[2] = {0, 0}, p2[2] = {0, 0};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int Q = fixed22((w[q >> 1] >> (16 * (q & 1))) & 0xFFFFu, m);
      const int d0 = int(int8_t(uint8_t(Q & 0xFF)));
      const int Q1 = (Q - d0) >> 8;
      const int d1 = int(int8_t(uint8_t(Q1 & 0xFF)));
      const int d2 = (Q1 - d1) >> 8;
      p0[q >> 2] |= uint32_t(uint8_t(d0)) << (8 * (q & 3));
      p1[q >> 2] |= uint32_t(uint8_t(d1)) << (8 * (q & 3));
      p2[q >> 2] |= uint32_t(uint8_t(d2)) << (8 * (q & 3));
    }
    *reinterpret_cast<uint2*>(dst + (0 * R + r) * K + c * 8) = make_uint2(p0[0], p0[1]);
    *reinterpret_cast<uint2*>(dst + (1 * R + r) * K + c * 8) = make_uint2(p1[0], p1[1]);
    *reinterpret_cast<uint2*>(dst + (2 * R + r) * K + c * 8) = make_uint2(p2[0], p2[1]);
  }
  if (lane == 0) emax[r] = m;
}

// ---------------------------------------------------------------- permute
// Tokens per chunk: 128, halved (down to 8) while that leaves fewer than two
// chunks per SM, so small (decode) batches still spread the row copies over
// the whole GPU. Pairs are ranked chunk by chunk, so the permutation is the
// same stable expert-major order for every chunk size.
constexpr int PCH_MAX = 128, PCH_MIN = 8;
constexpr int MB_ROWS = 128;  // rows per GEMM m-block
inline int permute_chunk(int64_t T) {
  int pch = PCH_MAX;
  while (pch > PCH_MIN && (T + pch - 1) / pch < 2 * 148) pch >>= 1;
  return pch;
}

__global__ void __launch_bounds__(256) permute_count_kernel(const int32_t* __restrict__ idx,
                                                            int64_t T, int E, int k, int pch,
                                                            int32_t* __restrict__ chunk_counts) {
  extern __shared__ int32_t hist[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int64_t p0 = int64_t(blockIdx.x) * pch * k;
  const int64_t p1 = (p0 + int64_t(pch) * k < T * k) ? p0 + int64_t(pch) * k : T * k;
  for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    const int e = idx[p];
    if (e >= 0) atomicAdd(&hist[e], 1);  // e < 0: pair not computed here (DEP: remote expert)
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    chunk_counts[int64_t(blockIdx.x) * E + e] = hist[e];
}

// One CTA: per-expert exclusive prefix over chunks, padded expert offsets,
// m-block -> expert table.
__global__ void __launch_bounds__(1024) permute_scan_kernel(int32_t* __restrict__ chunk_counts,
                                                            int nchunks, int E, int64_t T,
                                                            int shared, int align,
                                                            int32_t* __restrict__ counts,
                                                            int32_t* __restrict__ expert_off,
                                                            int32_t* __restrict__ mblock_expert,
                                                            int2* __restrict__ mb_seg,
                                                            int32_t* __restrict__ src_row,
                                                            int32_t* __restrict__ meta,
                                                            int32_t* __restrict__ mb_rows,
                                                            int64_t shared_T, int64_t cap_rows) {
  extern __shared__ int32_t sh[];  // [E] padded sizes, then [E] offsets
  int32_t* pad = sh;
  int32_t* off = sh + E;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t run = 0;
    int c = 0;
    for (; c + 8 <= nchunks; c += 8) {  // 8 independent loads in flight
      int32_t n[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) n[u] = chunk_counts[int64_t(c + u) * E + e];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        chunk_counts[int64_t(c + u) * E + e] = run;
        run += n[u];
      }
    }
    for (; c < nchunks; ++c) {
      const int32_t n = chunk_counts[int64_t(c) * E + e];
      chunk_counts[int64_t(c) * E + e] = run;
      run += n;
    }
    counts[e] = run;
    pad[e] = (run + align - 1) / align * align;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t acc = 0;
    for (int e = 0; e < E; ++e) {
      off[e] = acc;
      acc += pad[e];
    }
    const int32_t routed_mb = acc / MB_ROWS;
    const int32_t shared_mb =
        shared ? int32_t((shared_T + align - 1) / align * (align / MB_ROWS)) : 0;
    // capacity guard (callers whose row count is data-dependent, e.g. the DEP
    // receive side): an overflowing layer computes nothing and raises meta[4]
    const bool over = cap_rows > 0 && int64_t(acc) + int64_t(shared_mb) * MB_ROWS > cap_rows;
    meta[0] = over ? 0 : routed_mb + shared_mb;
    meta[1] = over ? 0 : routed_mb;
    meta[2] = over ? 0 : acc;
    meta[3] = int32_t(shared_T);
    meta[4] = over ? 1 : 0;
  }
  __syncthreads();
  if (meta[4]) return;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    expert_off[e] = off[e];
    const int2 seg = make_int2(off[e] / MB_ROWS, pad[e] / MB_ROWS);
    for (int32_t b = seg.x; b < seg.x + seg.y; ++b) {
      mblock_expert[b] = e;
      mb_seg[b] = seg;
      if (mb_rows) {  // real (non-padding) rows of the m-block
        const int32_t v = counts[e] - (b - seg.x) * MB_ROWS;
        mb_rows[b] = v < 0 ? 0 : (v > MB_ROWS ? MB_ROWS : v);
      }
    }
    if (src_row)  // padding rows gather token 0 (computed, never read)
      for (int32_t r = off[e] + counts[e]; r < off[e] + pad[e]; ++r) src_row[r] = 0;
  }
  if (shared) {
    const int32_t rmb = meta[1];
    const int2 seg = make_int2(rmb, meta[0] - rmb);
    for (int32_t b = threadIdx.x; b < seg.y; b += blockDim.x) {
      mblock_expert[rmb + b] = E;
      mb_seg[rmb + b] = seg;
      if (mb_rows) {
        const int64_t v = shared_T - int64_t(b) * MB_ROWS;
        mb_rows[rmb + b] = v < 0 ? 0 : (v > MB_ROWS ? MB_ROWS : int32_t(v));
      }
    }
  }
}

__global__ void __launch_bounds__(256) permute_scatter_kernel(
    const int32_t* __restrict__ idx, const uint16_t* __restrict__ x, int64_t T, int E, int k,
    int64_t h, const int32_t* __restrict__ chunk_base, const int32_t* __restrict__ expert_off,
    int32_t* __restrict__ row_of, int32_t* __restrict__ src_row, uint16_t* __restrict__ xperm,
    uint8_t* __restrict__ xperm8, float* __restrict__ xscale, const int32_t* __restrict__ meta,
    int shared, int pch, uint8_t* __restrict__ xsf) {
  extern __shared__ int32_t sm[];  // cursor[E], rows[pch * k]
  int32_t* cursor = sm;
  int32_t* rows = sm + E;
  for (int e = threadIdx.x; e < E; e += blockDim.x) cursor[e] = 0;
  __syncthreads();
  const int64_t t0 = int64_t(blockIdx.x) * pch;
  const int ntok = int(T - t0 < pch ? T - t0 : pch);
  const int npairs = ntok * k;
  if (threadIdx.x < 32) {  // warp 0 ranks pairs in (t, j) order
    const int lane = threadIdx.x;
    for (int s = 0; s < npairs; s += 32) {
      const int pl = s + lane;
      const bool act = pl < npairs;
      const int e = act ? idx[t0 * k + pl] : -1;
      // pairs with e < 0 are not computed on this rank (DEP receive side),
      // and none are after a capacity overflow (meta[4])
      const bool live = act && e >= 0 && !(meta && meta[4]);
      const unsigned lm = __ballot_sync(0xffffffffu, live);
      if (live) {
        const unsigned peers = __match_any_sync(lm, e);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        const int before = cursor[e];
        const int pos = expert_off[e] + chunk_base[int64_t(blockIdx.x) * E + e] + before + rank;
        rows[pl] = pos;
        row_of[t0 * k + pl] = pos;
        if (src_row) src_row[pos] = int32_t(t0 + pl / k);
        __syncwarp(lm);
        if (lane == 31 - __clz(peers)) cursor[e] = before + __popc(peers);
      } else if (act) {
        rows[pl] = -1;
        row_of[t0 * k + pl] = -1;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (xperm8 && xsf) {  // NVFP4: quantise each token row once, write k + shared copies
    // row scales first (warp per token), then one thread per (token,
    // 64-element group): 8 independent 16-byte loads per thread and
    // coalesced 32-byte code stores across the CTA
    float* rs = reinterpret_cast<float*>(rows + pch * k);
    const int32_t shared_row0 = shared ? meta[2] : 0;
    const int64_t shared_T = shared ? meta[3] : 0;  // tokens [0, shared_T) have a shared-expert row
    for (int tl = warp; tl < ntok; tl += blockDim.x >> 5) {
      const float sc = nvfp4_row_scale(row_absmax_bf16(reinterpret_cast<const uint4*>(x + (t0 + tl) * h),
                                                       h / 8, lane));
      if (lane == 0) rs[tl] = sc;
      if (lane < k && rows[tl * k + lane] >= 0) xscale[rows[tl * k + lane]] = sc;
      if (t0 + tl < shared_T && lane == 0) xscale[shared_row0 + t0 + tl] = sc;
    }
    __syncthreads();
    const int ng = int(h / 64);
    for (int it = threadIdx.x; it < ntok * ng; it += blockDim.x) {
      const int tl = it / ng, g = it - tl * ng;
      const uint4* src = reinterpret_cast<const uint4*>(x + (t0 + tl) * h) + 8 * g;
      uint4 q[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = __ldg(src + j);
      float v[64];
      unpack_bf16x64(q, v);
      uint32_t c[8];
      const uint32_t sfw = nvfp4_group(v, rs[tl], c);
      for (int j = 0; j < k; ++j) {
        const int64_t r = rows[tl * k + j];
        if (r >= 0) store_group(xperm8 + r * (h / 2), xsf, r, g, h, c, sfw, true);
      }
      if (t0 + tl < shared_T) {
        const int64_t r = shared_row0 + t0 + tl;
        store_group(xperm8 + r * (h / 2), xsf, r, g, h, c, sfw, true);
      }
    }
    return;
  }
  if (xperm8) {  // W8A8: quantise each token row once (per-row scale), write k + shared copies
    const int64_t nch = h / 8;
    const int32_t shared_row0 = shared ? meta[2] : 0;
    const int64_t shared_T = shared ? meta[3] : 0;
    for (int tl = warp; tl < ntok; tl += blockDim.x >> 5) {
      const uint4* src = reinterpret_cast<const uint4*>(x + (t0 + tl) * h);
      const bool sh = t0 + tl < shared_T;
      const float amax = row_absmax_bf16(src, nch, lane);
      const float s = amax > 0.0f ? __fdiv_rn(amax, 448.0f) : 1.0f;
      // four 16-byte loads in flight per lane before the quantise + k stores
      int64_t c0 = lane;
      for (; c0 + 96 < nch; c0 += 128) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(src + c0 + 32 * u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t c = c0 + 32 * u;
          const uint2 q = quant8(v[u], s);
          for (int j = 0; j < k; ++j)
            if (rows[tl * k + j] >= 0) reinterpret_cast<uint2*>(xperm8 + int64_t(rows[tl * k + j]) * h)[c] = q;
          if (sh) reinterpret_cast<uint2*>(xperm8 + int64_t(shared_row0 + t0 + tl) * h)[c] = q;
        }
      }
      for (int64_t c = c0; c < nch; c += 32) {
        const uint2 q = quant8(__ldg(src + c), s);
        for (int j = 0; j < k; ++j)
          if (rows[tl * k + j] >= 0) reinterpret_cast<uint2*>(xperm8 + int64_t(rows[tl * k + j]) * h)[c] = q;
        if (sh) reinterpret_cast<uint2*>(xperm8 + int64_t(shared_row0 + t0 + tl) * h)[c] = q;
      }
      if (lane < k && rows[tl * k + lane] >= 0) xscale[rows[tl * k + lane]] = s;
      if (sh && lane == 0) xscale[shared_row0 + t0 + tl] = s;
    }
    return;
  }
  if (!xperm) return;  // GEMM1 gathers the rows itself (TMA tile::gather4)
  // gather: each warp copies whole token rows to their k destinations, four
  // 16-byte loads in flight per lane before the 4k stores (latency hiding)
  const int64_t segs = h / 8;
  for (int tl = warp; tl < ntok; tl += blockDim.x >> 5) {
    const uint4* src = reinterpret_cast<const uint4*>(x + (t0 + tl) * h);
    const int32_t* dst = rows + tl * k;
    int64_t s = lane;
    for (; s + 96 < segs; s += 128) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(src + s + 32 * u);
      for (int j = 0; j < k; ++j) {
        if (dst[j] < 0) continue;
        uint4* d = reinterpret_cast<uint4*>(xperm + int64_t(dst[j]) * h) + s;
#pragma unroll
        for (int u = 0; u < 4; ++u) d[32 * u] = v[u];
      }
    }
    for (; s < segs; s += 32) {
      const uint4 v = __ldg(src + s);
      for (int j = 0; j < k; ++j)
        if (dst[j] >= 0) reinterpret_cast<uint4*>(xperm + int64_t(dst[j]) * h)[s] = v;
    }
  }
}

// Row replication with the bulk-copy (TMA) engine: one thread per CTA loads
// each token row (h*2 bytes) into shared memory with cp.async.bulk and writes
// it to its k expert-major destinations with k bulk stores, so the 8x write
// amplification of the permute costs no per-16-byte instructions (the warp
// copy above is issue-bound at the power-capped SM clock). A ring of PB_BUFS
// rows keeps the next loads in flight while the stores of a row drain.
constexpr int PB_BUFS = 3;

__device__ __forceinline__ uint32_t pb_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(32) permute_copy_bulk_kernel(const uint16_t* __restrict__ x,
                                                               int64_t T, int k, int64_t h,
                                                               const int32_t* __restrict__ row_of,
                                                               uint16_t* __restrict__ xperm,
                                                               int tpc) {
  extern __shared__ __align__(128) uint8_t pbuf[];
  __shared__ __align__(8) uint64_t bar[PB_BUFS];
  if (threadIdx.x != 0) return;
  const uint32_t bytes = uint32_t(h * 2);
  const int64_t t0 = int64_t(blockIdx.x) * tpc;
  const int n = int(T - t0 < tpc ? T - t0 : tpc);
  if (n <= 0) return;
  for (int b = 0; b < PB_BUFS; ++b)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(pb_smem(&bar[b])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto load = [&](int i) {
    const int b = i % PB_BUFS;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(pb_smem(&bar[b])),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            pb_smem(pbuf + size_t(b) * bytes)),
        "l"(x + (t0 + i) * h), "r"(bytes), "r"(pb_smem(&bar[b]))
        : "memory");
  };
  for (int i = 0; i < PB_BUFS && i < n; ++i) load(i);
  for (int i = 0; i < n; ++i) {
    const int b = i % PB_BUFS;
    const uint32_t parity = uint32_t(i / PB_BUFS) & 1u;
    uint32_t ok = 0;
    do {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          "selp.u32 %0, 1, 0, p;\n}"
          : "=r"(ok)
          : "r"(pb_smem(&bar[b])), "r"(parity)
          : "memory");
    } while (!ok);
    const int32_t* dst = row_of + (t0 + i) * k;
    for (int j = 0; j < k; ++j)
      if (dst[j] >= 0)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         xperm + int64_t(dst[j]) * h),
                     "r"(pb_smem(pbuf + size_t(b) * bytes)), "r"(bytes)
                     : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (i + PB_BUFS < n) {  // buffer b is refilled once its stores have read it
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load(i + PB_BUFS);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------- combine
// resid never aliases y: the stacks ping-pong between two buffers
// (Ctx::stack_forward), so every input is read through the non-coherent path.
// SKIP_NEG: rows < 0 are pairs computed on another rank (DEP partial combine).
template <bool SKIP_NEG>
__global__ void __launch_bounds__(128) combine_kernel(const uint16_t* __restrict__ O,
                                                      const int32_t* __restrict__ row_of,
                                                      const float* __restrict__ wts,
                                                      const uint16_t* __restrict__ S,
                                                      const int32_t* __restrict__ s_meta,
                                                      const uint16_t* __restrict__ resid,
                                                      uint16_t* __restrict__ y, int64_t T, int k, int64_t h) {
  const int64_t t = blockIdx.x;
  if (t >= T) return;
  __shared__ int32_t srow[TOPK_MAXK + 1];
  __shared__ float sw[TOPK_MAXK];
  if (threadIdx.x < k) {
    srow[threadIdx.x] = row_of[t * k + threadIdx.x];
    sw[threadIdx.x] = wts[t * k + threadIdx.x];
  }
  if (threadIdx.x == 0) srow[TOPK_MAXK] = (s_meta ? s_meta[2] : 0) + int32_t(t);
  __syncthreads();
  const bool shared = S != nullptr;
  const int64_t segs = h / 8;
  // Every row's 16-byte load of a batch (up to 8 routed rows, the shared row
  // and the residual) is issued before the first FMA: one load in flight per
  // thread left the kernel latency-bound below the HBM rate. The FMA order
  // (routed rows in j order, then shared, then residual) is unchanged.
  constexpr int CB = 8;
  for (int64_t s = threadIdx.x; s < segs; s += blockDim.x) {
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
    uint4 vs = make_uint4(0, 0, 0, 0), vr = make_uint4(0, 0, 0, 0);
    if (shared) vs = __ldg(reinterpret_cast<const uint4*>(S + int64_t(srow[TOPK_MAXK]) * h) + s);
    if (resid) vr = __ldg(reinterpret_cast<const uint4*>(resid + t * h) + s);
    for (int j0 = 0; j0 < k; j0 += CB) {
      uint4 v[CB];
#pragma unroll
      for (int jj = 0; jj < CB; ++jj)
        if (j0 + jj < k) {
          if (SKIP_NEG && srow[j0 + jj] < 0)
            v[jj] = make_uint4(0, 0, 0, 0);
          else
            v[jj] = __ldg(reinterpret_cast<const uint4*>(O + int64_t(srow[j0 + jj]) * h) + s);
        }
#pragma unroll
      for (int jj = 0; jj < CB; ++jj) {
        if (j0 + jj >= k) break;
        const uint32_t u[4] = {v[jj].x, v[jj].y, v[jj].z, v[jj].w};
        const float wj = sw[j0 + jj];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[2 * q] = __fmaf_rn(wj, __uint_as_float(u[q] << 16), acc[2 * q]);
          acc[2 * q + 1] = __fmaf_rn(wj, __uint_as_float(u[q] & 0xffff0000u), acc[2 * q + 1]);
        }
      }
    }
    if (shared) {
      const uint4 v = vs;
      const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[2 * q] += __uint_as_float(u[q] << 16);
        acc[2 * q + 1] += __uint_as_float(u[q] & 0xffff0000u);
      }
    }
    if (resid) {
      const uint4 v = vr;
      const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[2 * q] += __uint_as_float(u[q] << 16);
        acc[2 * q + 1] += __uint_as_float(u[q] & 0xffff0000u);
      }
    }
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      o[q] = uint32_t(bf16_bits(acc[2 * q])) | (uint32_t(bf16_bits(acc[2 * q + 1])) << 16);
    reinterpret_cast<uint4*>(y + t * h)[s] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// ---------------------------------------------------------------- pull
// TMA bulk pull: one elected thread per CTA streams 8 KB chunks of the copy
// plan's slices (interleaved over slices, see PullCursor) from peer HBM over
// NVLink into a shared-memory ring (cp.async.bulk global->shared, mbarrier
// completion) and out to the local receive buffer (cp.async.bulk
// shared->global, bulk-group completion).
// 3 x 8 KB ring (26 KB with the barriers): fits next to a 194 KB grouped-GEMM
// CTA on every SM (228 KB per SM, 1 KB reserved per CTA), so the pull runs
// concurrently with the expert GEMMs instead of queueing behind them. The
// achieved GB/s was flat over 4-32 KB chunks x 2-8 buffers (the fabric sets it).
constexpr int PULL_CHUNK_DEFAULT = 8192, PULL_BUFS_DEFAULT = 3, PULL_BUFS_MAX = 8;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Chunk c of slice i has global index c * n + i (slice-interleaved), and CTA
// b takes indices b, b + grid, b + 2 grid, ...: every CTA gets the same number
// of chunks whatever the slice count and sizes, and the chunks in flight at
// any moment come from all slices -- i.e. from every peer of the TDM rotation
// at once -- instead of one CTA streaming a whole 64 MB slice from one peer.
// Indices past the end of a shorter slice are skipped.
struct PullCursor {
  uint32_t chunk;  // bytes per chunk
  uint64_t g;  // global chunk index
  int it;      // slice of g (n = done)
  uint64_t off;
  __device__ void seek(const PullItem* items, int n, uint64_t total) {
    while (g < total) {
      const int i = int(g % uint64_t(n));
      const uint64_t o = (g / uint64_t(n)) * chunk;
      if (o < items[i].len) {
        it = i;
        off = o;
        return;
      }
      g += gridDim.x;
    }
    it = n;
  }
  __device__ void advance(const PullItem* items, int n, uint64_t total) {
    g += gridDim.x;
    seek(items, n, total);
  }
};

__global__ void __launch_bounds__(32) tma_pull_kernel(const PullItem* __restrict__ items, int n,
                                                      uint64_t total, uint32_t chunk, int nbufs) {
  extern __shared__ __align__(128) uint8_t pull_smem[];  // nbufs chunks (dynamic)
  __shared__ __align__(8) uint64_t bar[PULL_BUFS_MAX];
  auto buf = [&](int b) { return pull_smem + size_t(b) * chunk; };
  if (threadIdx.x != 0) return;
  for (int b = 0; b < nbufs; ++b)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[b])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase = 0;  // bit b: parity of buffer b's next completion
  auto load = [&](int b, const PullCursor& c) {
    const PullItem& w = items[c.it];
    const uint32_t len = uint32_t(w.len - c.off < chunk ? w.len - c.off : chunk);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[b])),
                 "r"(len)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(buf(b))),
        "l"(static_cast<const uint8_t*>(w.src) + c.off), "r"(len), "r"(smem_addr(&bar[b]))
        : "memory");
  };
  PullCursor prod{chunk, blockIdx.x, 0, 0};
  prod.seek(items, n, total);
  PullCursor cons = prod;
  int issued = 0, done = 0;
  while (issued < nbufs && prod.it < n) {  // prologue: fill the ring
    load(issued, prod);
    prod.advance(items, n, total);
    ++issued;
  }
  while (done < issued) {
    const int b = done % nbufs;
    uint32_t ok = 0;
    do {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          "selp.u32 %0, 1, 0, p;\n}"
          : "=r"(ok)
          : "r"(smem_addr(&bar[b])), "r"((phase >> b) & 1u)
          : "memory");
    } while (!ok);
    phase ^= 1u << b;
    const PullItem& w = items[cons.it];
    const uint32_t len = uint32_t(w.len - cons.off < chunk ? w.len - cons.off : chunk);
    // streamed into the receive buffer: evict-first so the 17-20 GB per layer
    // does not push the running GEMM's expert weights out of L2
    asm volatile(
        "{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
        "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, pol;\n}" ::"l"(
            static_cast<uint8_t*>(w.dst) + cons.off),
        "r"(smem_addr(buf(b))), "r"(len)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    cons.advance(items, n, total);
    ++done;
    if (prod.it < n) {  // refill buffer b once its store has read shared memory
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load(b, prod);
      prod.advance(items, n, total);
      ++issued;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int grid_for(int64_t work, int block) {
  int64_t g = (work + block - 1) / block;
  if (g > 148 * 16) g = 148 * 16;
  return int(g < 1 ? 1 : g);
}

}  // namespace

void launch_fill_slots(uint16_t* dst, const uint64_t* seeds, int nslots, int64_t slot_elems,
                       float scale, cudaStream_t st) {
  if (nslots <= 0) return;
  fill_slots_kernel<<<grid_for(nslots * (slot_elems / 8), 256), 256, 0, st>>>(dst, seeds, nslots,
                                                                             slot_elems, scale);
}

void launch_fill(uint16_t* dst, int64_t n, uint64_t seed, float scale, cudaStream_t st) {
  if (n > 0) fill_kernel<<<grid_for(n, 256), 256, 0, st>>>(dst, n, seed, scale);
}

void launch_fill_f32(float* dst, int64_t n, uint64_t seed, float scale, cudaStream_t st) {
  if (n > 0) fill_f32_kernel<<<grid_for(n, 256), 256, 0, st>>>(dst, n, seed, scale);
}

void launch_router_logits(const uint16_t* x, const uint16_t* w, float* logits, int64_t T, int E,
                          int64_t K, cudaStream_t st) {
  if (T <= 0) return;
  dim3 grid(unsigned((T + RB_M - 1) / RB_M), unsigned((E + RB_N - 1) / RB_N));
  router_logits_kernel<<<grid, 256, 0, st>>>(x, w, logits, T, E, K);
}

void launch_topk(const int32_t* C, const int32_t* ex, const int32_t* ew, const float* bias,
                 float* logits, int32_t* idx, float* wts, int64_t T, const RouterCfg& c,
                 cudaStream_t st) {
  if (T <= 0) return;
  const unsigned grid = unsigned((T + 7) / 8);
  const int G = c.n_group > 0 ? c.n_group : 1;
  const int V = c.E / 32;
  const bool contig = c.E % 32 == 0 && (V == 1 || V == 2 || V == 4 || V == 8) &&
                      (G == 1 || ((c.E / G) % V == 0 && (c.E / G) / V <= 32 &&
                                  (((c.E / G) / V) & ((c.E / G) / V - 1)) == 0));
  if (contig && V == 8 && C == nullptr)  // logits formed by the fused router GEMM
    topk_contig_kernel<8, true><<<grid, 256, 0, st>>>(C, ex, ew, bias, logits, idx, wts, T, c);
  else if (contig && V == 8)
    topk_contig_kernel<8, false><<<grid, 256, 0, st>>>(C, ex, ew, bias, logits, idx, wts, T, c);
  else if (contig && V == 4)
    topk_contig_kernel<4, false><<<grid, 256, 0, st>>>(C, ex, ew, bias, logits, idx, wts, T, c);
  else if (contig && V == 2)
    topk_contig_kernel<2, false><<<grid, 256, 0, st>>>(C, ex, ew, bias, logits, idx, wts, T, c);
  else if (contig && V == 1)
    topk_contig_kernel<1, false><<<grid, 256, 0, st>>>(C, ex, ew, bias, logits, idx, wts, T, c);
  else
    topk_kernel<<<grid, 256, 0, st>>>(C, ex, ew, bias, logits, idx, wts, T, c);
}

void launch_router_quant(const uint16_t* src, int64_t R, int64_t K, int8_t* dst, int32_t* emax,
                         int32_t* meta, cudaStream_t st) {
  if (R <= 0) return;
  const size_t smem = size_t(RQ_WARPS) * size_t(K) * 2;
  if (smem <= 48 * 1024)
    router_quant_kernel<<<unsigned((R + RQ_WARPS - 1) / RQ_WARPS), 32 * RQ_WARPS, smem, st>>>(
        src, R, K, dst, emax, meta, 1);
  else
    router_quant_kernel<<<unsigned((R + 7) / 8), 256, 0, st>>>(src, R, K, dst, emax, meta, 0);
}

int64_t permute_scratch_ints(int64_t T, int E) {
  // chunks <= max(T / 128, 2 * (2 * 148)) + 1 (permute_chunk halves only below 296)
  const int64_t nch = std::max<int64_t>((T + PCH_MAX - 1) / PCH_MAX, 4 * 148 + 1);
  return nch * E + E;
}

// Two layouts of the same expert-major rows (see launch_split_layout): per
// expert e with c rows, segment 128-layout [o1, o1 + ceil(c/128)*128) and
// 256-layout [o2, o2 + ceil(c/256)*256); m-block j of e holds rows
// [j*128, j*128+128) of e's rows in both. The shared-expert block (T rows)
// follows the routed segments in each layout.
__global__ void __launch_bounds__(1024) split_layout_kernel(const int32_t* __restrict__ counts,
                                                            int E, int64_t T, int shared,
                                                            int32_t* __restrict__ mblock2,
                                                            int2* __restrict__ mb_seg2,
                                                            int32_t* __restrict__ mb_rows2,
                                                            int32_t* __restrict__ meta2,
                                                            int32_t* __restrict__ d1,
                                                            int32_t* __restrict__ d2) {
  extern __shared__ int32_t sm[];  // [E] 128-layout offsets, [E] 256-layout offsets, [2] totals
  int32_t* o1 = sm;
  int32_t* o2 = sm + E;
  if (threadIdx.x == 0) {
    int32_t a1 = 0, a2 = 0;
    for (int e = 0; e < E; ++e) {
      const int32_t c = counts[e];
      o1[e] = a1;
      o2[e] = a2;
      a1 += (c + 127) / 128 * 128;
      a2 += (c + 255) / 256 * 256;
    }
    sm[2 * E] = a1;
    sm[2 * E + 1] = a2;
    const int32_t smb2 = shared ? int32_t((T + 255) / 256 * 2) : 0;
    meta2[0] = a2 / MB_ROWS + smb2;
    meta2[1] = a2 / MB_ROWS;
    meta2[2] = a2;
    meta2[3] = int32_t(T);
  }
  __syncthreads();
  const int32_t R1 = sm[2 * E], R2 = sm[2 * E + 1];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int32_t c = counts[e];
    const int32_t n1 = (c + 127) / 128, n2 = (c + 255) / 256 * 2;
    const int32_t b1 = o1[e] / MB_ROWS, b2 = o2[e] / MB_ROWS;
    for (int32_t j = 0; j < n1; ++j) d1[b1 + j] = o2[e] + j * MB_ROWS;
    for (int32_t j = 0; j < n2; ++j) {
      mblock2[b2 + j] = e;
      mb_seg2[b2 + j] = make_int2(b2, n2);
      const int32_t v = c - j * MB_ROWS;
      mb_rows2[b2 + j] = v < 0 ? 0 : (v > MB_ROWS ? MB_ROWS : v);
      d2[b2 + j] = j < n1 ? o1[e] + j * MB_ROWS : 0;
    }
  }
  if (shared) {
    const int32_t n1 = int32_t((T + 127) / 128), n2 = int32_t((T + 255) / 256 * 2);
    const int32_t b1 = R1 / MB_ROWS, b2 = R2 / MB_ROWS;
    for (int32_t j = threadIdx.x; j < n2; j += blockDim.x) {
      if (j < n1) d1[b1 + j] = R2 + j * MB_ROWS;
      mblock2[b2 + j] = E;
      mb_seg2[b2 + j] = make_int2(b2, n2);
      const int64_t v = T - int64_t(j) * MB_ROWS;
      mb_rows2[b2 + j] = v < 0 ? 0 : (v > MB_ROWS ? MB_ROWS : int32_t(v));
      d2[b2 + j] = j < n1 ? R1 + j * MB_ROWS : 0;
    }
  }
}

void launch_split_layout(const int32_t* counts, int E, int64_t T, int shared, int32_t* mblock2,
                         int2* mb_seg2, int32_t* mb_rows2, int32_t* meta2, int32_t* d1, int32_t* d2,
                         cudaStream_t st) {
  split_layout_kernel<<<1, 1024, (2 * E + 2) * sizeof(int32_t), st>>>(counts, E, T, shared, mblock2,
                                                                      mb_seg2, mb_rows2, meta2, d1, d2);
}

// DEP receive side: pairs whose expert lies outside this rank's block
// [lo, hi) are marked -1 (not computed here); local ones keep their global id.
__global__ void localize_idx_kernel(const int32_t* __restrict__ in, int64_t n, int lo, int hi,
                                    int32_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int e = in[i];
    out[i] = (e >= lo && e < hi) ? e : -1;
  }
}

void launch_localize_idx(const int32_t* in, int64_t n, int lo, int hi, int32_t* out, cudaStream_t st) {
  if (n > 0)
    localize_idx_kernel<<<unsigned(std::min<int64_t>((n + 255) / 256, 148 * 8)), 256, 0, st>>>(in, n, lo,
                                                                                               hi, out);
}

// row_of[t][r] = r * T + t, w = 1: the DEP final combine sums the N ranks'
// partial rows of token t with combine_kernel (fma(1, v, acc) = v + acc).
__global__ void rank_rows_kernel(int32_t* __restrict__ row_of, float* __restrict__ w, int64_t T,
                                 int N) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < T * N; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / N, r = i - t * N;
    row_of[i] = int32_t(r * T + t);
    w[i] = 1.0f;
  }
}

namespace {
__global__ void dest_ranks_kernel(const int32_t* __restrict__ idx, int64_t T, int k, int per, int self,
                                  int32_t* __restrict__ idx2) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < T; t += int64_t(gridDim.x) * blockDim.x) {
    int32_t* o = idx2 + t * (k + 1);
    o[0] = self;
    for (int j = 0; j < k; ++j) {
      const int r = idx[t * k + j] / per;
      bool first = r != self;
      for (int i = 0; i < j && first; ++i) first = idx[t * k + i] / per != r;
      o[1 + j] = first ? r : -1;
    }
  }
}
__global__ void scatter_routing_kernel(const int32_t* __restrict__ idx, const float* __restrict__ wts,
                                       const int32_t* __restrict__ row_of2, int64_t T, int k, int k2,
                                       int32_t* __restrict__ sidx, float* __restrict__ swts) {
  const int64_t n = T * k2;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t r = row_of2[i];
    if (r < 0) continue;
    const int64_t t = i / k2;
    for (int j = 0; j < k; ++j) {
      sidx[int64_t(r) * k + j] = idx[t * k + j];
      swts[int64_t(r) * k + j] = wts[t * k + j];
    }
  }
}
__device__ __forceinline__ void copy_row_warp(uint8_t* dst, const uint8_t* src, int64_t bytes, int lane) {
  for (int64_t c = lane; c < bytes / 16; c += 32)
    reinterpret_cast<uint4*>(dst)[c] = __ldg(reinterpret_cast<const uint4*>(src) + c);
}
__global__ void __launch_bounds__(256) qrow_meta_kernel(const int32_t* __restrict__ row_of, int64_t T, int k,
                                                        const float* __restrict__ xs,
                                                        const uint8_t* __restrict__ sfl, int sfb,
                                                        float* __restrict__ xs_out, uint8_t* __restrict__ sfl_out,
                                                        const int32_t* __restrict__ meta, int64_t shared_T,
                                                        const uint8_t* __restrict__ codes, int64_t qrow,
                                                        uint8_t* __restrict__ codes_out) {
  if (meta && meta[4]) return;
  const int lane = threadIdx.x & 31;
  const int64_t shared_row0 = meta ? meta[2] : 0;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); t < T;
       t += int64_t(gridDim.x) * (blockDim.x >> 5)) {
    const float s = xs[t];
    for (int j = 0; j < k; ++j) {
      const int32_t r = row_of[t * k + j];
      if (r < 0) continue;
      if (lane == 0) xs_out[r] = s;
      if (sfl) copy_row_warp(sfl_out + int64_t(r) * sfb, sfl + t * sfb, sfb, lane);
    }
    if (meta && t < shared_T) {
      const int64_t R = shared_row0 + t;
      if (lane == 0) xs_out[R] = s;
      if (sfl) copy_row_warp(sfl_out + R * sfb, sfl + t * sfb, sfb, lane);
      copy_row_warp(codes_out + R * qrow, codes + t * qrow, qrow, lane);
    }
  }
}
__global__ void fill_f32_kernel(float* p, int64_t n, float v) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = v;
}
}  // namespace

void launch_dest_ranks(const int32_t* idx, int64_t T, int k, int per, int self, int32_t* idx2, cudaStream_t st) {
  if (T > 0)
    dest_ranks_kernel<<<unsigned(std::min<int64_t>((T + 255) / 256, 148 * 8)), 256, 0, st>>>(idx, T, k, per, self,
                                                                                            idx2);
}
void launch_scatter_routing(const int32_t* idx, const float* wts, const int32_t* row_of2, int64_t T, int k, int k2,
                            int32_t* sidx, float* swts, cudaStream_t st) {
  if (T > 0)
    scatter_routing_kernel<<<unsigned(std::min<int64_t>((T * k2 + 255) / 256, 148 * 8)), 256, 0, st>>>(
        idx, wts, row_of2, T, k, k2, sidx, swts);
}
void launch_qrow_meta(const int32_t* row_of, int64_t T, int k, const float* xs, const uint8_t* sfl, int sfb,
                      float* xs_out, uint8_t* sfl_out, const int32_t* meta, int64_t shared_T, const uint8_t* codes,
                      int64_t qrow, uint8_t* codes_out, cudaStream_t st) {
  if (T > 0)
    qrow_meta_kernel<<<unsigned(std::min<int64_t>((T + 7) / 8, 148 * 16)), 256, 0, st>>>(
        row_of, T, k, xs, sfl, sfb, xs_out, sfl_out, meta, shared_T, codes, qrow, codes_out);
}
void launch_fill_f32(float* p, int64_t n, float v, cudaStream_t st) {
  if (n > 0) fill_f32_kernel<<<unsigned(std::min<int64_t>((n + 255) / 256, 148 * 8)), 256, 0, st>>>(p, n, v);
}

void launch_rank_rows(int32_t* row_of, float* w, int64_t T, int N, cudaStream_t st) {
  if (T > 0)
    rank_rows_kernel<<<unsigned(std::min<int64_t>((T * N + 255) / 256, 148 * 8)), 256, 0, st>>>(row_of, w, T,
                                                                                              N);
}

int launch_permute(const int32_t* idx, const uint16_t* x, int64_t T, int E, int k, int64_t h,
                    int shared, int32_t* counts, int32_t* row_of, int32_t* mblock_expert,
                    int2* mb_seg, int32_t* src_row, int32_t* meta, uint16_t* xperm,
                    int32_t* scratch, cudaStream_t st, uint8_t* xperm8, float* xscale,
                    int row_align, int32_t* mb_rows, uint8_t* xsf, int64_t shared_T,
                    int64_t cap_rows) {
  const int pch = permute_chunk(T);
  const int nch = int((T + pch - 1) / pch);
  int32_t* chunk_counts = scratch;
  int32_t* expert_off = scratch + int64_t(nch) * E;
  if (nch > 0)
    permute_count_kernel<<<nch, 256, E * sizeof(int32_t), st>>>(idx, T, E, k, pch, chunk_counts);
  permute_scan_kernel<<<1, 1024, 2 * E * sizeof(int32_t), st>>>(
      chunk_counts, nch, E, T, shared, row_align, counts, expert_off, mblock_expert, mb_seg, src_row,
      meta, mb_rows, shared_T < 0 ? T : shared_T, cap_rows);
  // bf16 rows: rank in the scatter kernel, replicate with the bulk-copy kernel
  const bool bulk = xperm != nullptr && xperm8 == nullptr && h % 8 == 0 &&
                    size_t(PB_BUFS) * size_t(h) * 2 <= 48 * 1024;
  if (nch > 0)
    permute_scatter_kernel<<<nch, 256, (E + pch * k + (xsf ? pch : 0)) * sizeof(int32_t), st>>>(
        idx, x, T, E, k, h, chunk_counts, expert_off, row_of, src_row, bulk ? nullptr : xperm,
        xperm8, xscale, meta, shared, pch, xsf);
  if (bulk && T > 0) {
    const int per_sm = 5;  // 43 KB of row buffers per CTA
    const int tpc = int(std::max<int64_t>(1, (T + 148 * per_sm - 1) / (148 * per_sm)));
    permute_copy_bulk_kernel<<<unsigned((T + tpc - 1) / tpc), 32, size_t(PB_BUFS) * h * 2, st>>>(
        x, T, k, h, row_of, xperm, tpc);
  }
  return (nch > 0 ? 2 : 0) + 1 + (bulk && T > 0 ? 1 : 0);
}

void launch_fp8_fill_rows(uint8_t* dst, float* scales, const uint64_t* seeds, int nslots, int rows,
                          int64_t K, float scale, cudaStream_t st) {
  const int64_t warps = int64_t(nslots) * rows;
  if (warps > 0)
    fp8_fill_rows_kernel<<<unsigned((warps + 7) / 8), 256, 0, st>>>(dst, scales, seeds, nslots, rows,
                                                                   K, scale);
}

void launch_nvfp4_fill_rows(uint8_t* dst, uint8_t* sf, float* scales, const uint64_t* seeds,
                            int nslots, int rows, int64_t K, float scale, cudaStream_t st) {
  const int64_t warps = int64_t(nslots) * rows;
  if (warps > 0)
    nvfp4_fill_rows_kernel<<<unsigned((warps + 7) / 8), 256, 0, st>>>(dst, sf, scales, seeds, nslots,
                                                                     rows, K, scale);
}

void launch_nvfp4_sf_relayout(const uint8_t* lin, uint8_t* atoms, int64_t max_rows, int64_t K,
                              const int32_t* meta, cudaStream_t st) {
  const int64_t words = (max_rows + 127) / 128 * 128 * (K / 64);
  const int64_t blocks = std::min<int64_t>((words + 255) / 256, 148 * 16);
  if (blocks > 0)
    nvfp4_sf_relayout_kernel<<<unsigned(blocks), 256, 0, st>>>(reinterpret_cast<const uint32_t*>(lin),
                                                               reinterpret_cast<uint32_t*>(atoms),
                                                               max_rows, K, meta);
}

void launch_quant_rows_nvfp4(const uint16_t* src, int64_t max_rows, int64_t K, const int32_t* meta,
                             uint8_t* dst, uint8_t* sf_lin, uint8_t* sf, float* scales, cudaStream_t st) {
  if (max_rows <= 0) return;
  const unsigned grid = unsigned((max_rows + 7) / 8);
  if (K == 2048)
    quant_rows_nvfp4_il_kernel<8><<<grid, 256, 0, st>>>(src, max_rows, meta, dst, sf_lin, scales);
  else if (K == 1024)
    quant_rows_nvfp4_il_kernel<4><<<grid, 256, 0, st>>>(src, max_rows, meta, dst, sf_lin, scales);
  else if (K == 256)
    quant_rows_nvfp4_il_kernel<1><<<grid, 256, 0, st>>>(src, max_rows, meta, dst, sf_lin, scales);
  else
    quant_rows_nvfp4_kernel<<<grid, 256, 0, st>>>(src, max_rows, K, meta, dst, sf_lin, scales);
  launch_nvfp4_sf_relayout(sf_lin, sf, max_rows, K, meta, st);
}

void launch_quant_rows_fp8(const uint16_t* src, int64_t max_rows, int64_t K, const int32_t* meta,
                           uint8_t* dst, float* scales, cudaStream_t st) {
  if (max_rows > 0)
    quant_rows_fp8_kernel<<<unsigned((max_rows + 7) / 8), 256, 0, st>>>(src, max_rows, K, meta, dst,
                                                                        scales);
}

void launch_combine(const uint16_t* O, const int32_t* row_of, const float* wts,
                    const uint16_t* S, const int32_t* s_meta, const uint16_t* resid, uint16_t* y,
                    int64_t T, int k, int64_t h, cudaStream_t st) {
  if (T <= 0) return;
  if (resid == y) throw std::runtime_error("combine: resid must not alias y");
  combine_kernel<false><<<unsigned(T), 128, 0, st>>>(O, row_of, wts, S, s_meta, resid, y, T, k, h);
}

void launch_combine_sparse(const uint16_t* O, const int32_t* row_of, const float* wts, const uint16_t* S,
                           const int32_t* s_meta, const uint16_t* resid, uint16_t* y, int64_t T, int k, int64_t h,
                           cudaStream_t st) {
  if (T <= 0) return;
  if (resid == y) throw std::runtime_error("combine: resid must not alias y");
  combine_kernel<true><<<unsigned(T), 128, 0, st>>>(O, row_of, wts, S, s_meta, resid, y, T, k, h);
}

void launch_combine_partial(const uint16_t* O, const int32_t* row_of, const float* wts, uint16_t* y, int64_t T,
                            int k, int64_t h, cudaStream_t st) {
  if (T > 0)
    combine_kernel<true><<<unsigned(T), 128, 0, st>>>(O, row_of, wts, nullptr, nullptr, nullptr, y, T, k, h);
}

void launch_pull(const PullItem* items, int n, uint64_t max_len, int ctas, cudaStream_t st) {
  // chunk size and ring depth: 8 KB x 3 by default; DWDP_PULL_CHUNK /
  // DWDP_PULL_BUFS override them for experiments (the ring must stay small
  // enough to co-reside with a grouped-GEMM CTA). One host thread per GPU may
  // call concurrently: the settings are a thread-safe static, the smem
  // attribute is set once per device.
  struct PullCfg {
    int chunk, bufs;
  };
  static const PullCfg pc = [] {
    const char* c = std::getenv("DWDP_PULL_CHUNK");
    const char* b = std::getenv("DWDP_PULL_BUFS");
    return PullCfg{c ? std::max(1024, std::min(65536, std::atoi(c))) / 16 * 16 : PULL_CHUNK_DEFAULT,
                   b ? std::max(1, std::min(PULL_BUFS_MAX, std::atoi(b))) : PULL_BUFS_DEFAULT};
  }();
  static std::once_flag attr_once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(attr_once[dev & 63], [] {
    cudaFuncSetAttribute(tma_pull_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         PULL_BUFS_MAX * 65536 > 200 * 1024 ? 200 * 1024 : PULL_BUFS_MAX * 65536);
  });
  const uint64_t total = (max_len + pc.chunk - 1) / pc.chunk * uint64_t(n);
  if (n > 0)
    tma_pull_kernel<<<ctas, 32, size_t(pc.bufs) * pc.chunk, st>>>(items, n, total, uint32_t(pc.chunk),
                                                                  pc.bufs);
}

// Shared-memory carveout of the layer-path kernels. An SM's L1 / shared split
// is set by the first CTA that lands on it while it is idle; CTAs needing
// more shared memory cannot join until it drains. With an SM pull engine
// running beside the layer (N > 1, pull / hybrid), a pull CTA resident on an
// SM configured by a small kernel kept the 194 KB grouped-GEMM CTAs off it
// for the whole pull (GEMM1 11 -> 35 ms per layer at N = 4): then every
// layer-path kernel asks for the maximal carveout. Otherwise only the pull
// kernel does, and the small kernels keep the driver's choice -- the maximal
// carveout shrinks L1 and slowed the combine 1.47 -> 1.87 ms per layer
// (profiles/r2_ab_carveout.jsonl).
void configure_max_shared_carveout_kernels(bool all) {
  const int c = all ? int(cudaSharedmemCarveoutMaxShared) : int(cudaSharedmemCarveoutDefault);
  auto set = [&](const void* f) { cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, c); };
  cudaFuncSetAttribute(reinterpret_cast<const void*>(tma_pull_kernel),
                       cudaFuncAttributePreferredSharedMemoryCarveout, int(cudaSharedmemCarveoutMaxShared));
  set(reinterpret_cast<const void*>(router_quant_kernel));
  set(reinterpret_cast<const void*>(topk_kernel));
  set(reinterpret_cast<const void*>(topk_contig_kernel<8, true>));
  set(reinterpret_cast<const void*>(topk_contig_kernel<8, false>));
  set(reinterpret_cast<const void*>(topk_contig_kernel<4, false>));
  set(reinterpret_cast<const void*>(topk_contig_kernel<2, false>));
  set(reinterpret_cast<const void*>(topk_contig_kernel<1, false>));
  set(reinterpret_cast<const void*>(permute_count_kernel));
  set(reinterpret_cast<const void*>(permute_scan_kernel));
  set(reinterpret_cast<const void*>(permute_scatter_kernel));
  set(reinterpret_cast<const void*>(permute_copy_bulk_kernel));
  set(reinterpret_cast<const void*>(combine_kernel<false>));
  set(reinterpret_cast<const void*>(combine_kernel<true>));
  set(reinterpret_cast<const void*>(quant_rows_fp8_kernel));
  set(reinterpret_cast<const void*>(quant_rows_nvfp4_kernel));
  set(reinterpret_cast<const void*>(quant_rows_nvfp4_il_kernel<8>));
  set(reinterpret_cast<const void*>(nvfp4_sf_relayout_kernel));
  set(reinterpret_cast<const void*>(split_layout_kernel));
  set(reinterpret_cast<const void*>(localize_idx_kernel));
  set(reinterpret_cast<const void*>(rank_rows_kernel));
  cudaGetLastError();
}

}  // namespace dwdp
