// Grouped expert GEMM on Blackwell 5th-gen tensor cores (sm_100a).
//
//   GEMM1 (SWIGLU = true):  H[m, n] = silu(X[m,:] . Wg[e][n,:]) * (X[m,:] . Wu[e][n,:])
//   GEMM2 (SWIGLU = false): O[m, n] = H[m,:] . Wd[e][n,:]
//
// Rows m are the expert-major permuted tokens, padded per expert to 128-row
// m-blocks; m-block b belongs to expert mblock_expert[b] (device table written
// by the permute kernel, so group sizes never touch the host). Expert weights
// live in per-tensor arenas [slot][rows][K] (K-major) that hold the owned
// experts AND the DWDP receive buffers, so remote experts are consumed in
// place (split-weight layout, no merge copy); slot_of[e] maps expert -> slot.
// The shared expert is group E: its A rows are read straight from x.
//
// Structure (one CTA per SM, persistent, 256 threads):
//   warp 0      TMA producer  (cp.async.bulk.tensor -> 4-stage smem ring)
//   warp 1      MMA issuer    (tcgen05.mma kind::f16, M128 x N256 x K16, fp32 in TMEM)
//   warp 2      TMEM allocator (512 columns = 2 accumulator buffers)
//   warps 4-7   epilogue      (tcgen05.ld -> SwiGLU / cast -> bf16 stores)
// The two TMEM accumulators let the epilogue of tile i overlap the MMAs of
// tile i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "gemm_sm100.hpp"

namespace dwdp {
namespace {

constexpr int BM = 128;
constexpr int BN = 256;  // accumulator columns per tile
constexpr int BK = 64;   // 128 B of bf16 = one SWIZZLE_128B atom row
// 4 stages (194 KB): the 1-SM kernel (router int8 GEMM) must also fit beside a
// 26 KB prefetch pull CTA, or it queues behind the whole pull (measured: the
// router GEMM waited 24 ms per layer next to a 49 KB pull CTA at N = 4).
constexpr int STAGES = 4;
constexpr int A_STAGE = BM * BK * 2;  // 16 KB
constexpr int B_STAGE = BN * BK * 2;  // 32 KB
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) + 1024 /*align*/ + 256 /*barriers*/;
// scaled (fp8 / nvfp4) modes add the tiles' weight-row scales (2 x 256 fp32)
constexpr int SMEM_BYTES8 = SMEM_BYTES + 2048;
constexpr uint32_t TMEM_COLS = 512;
// NVFP4 modes (kind::mxf4nvf4 block16): a 128-byte smem row holds 256 e2m1
// elements, so one stage carries 4x the K of a bf16 stage; 3 stages plus the
// e4m3 block scales (A: 128 rows x 16 = 2 KB, B: 256 rows x 16 = 4 KB).
// TMEM: two overlapping accumulators (columns [0,256) and [192,448)) and the
// block scales of one k-block at [448,512); the epilogue drains the 64
// shared columns first and releases them early (tpart), so the next tile's
// MMAs start while the rest of the tile is still being stored.
constexpr int FP4_STAGES = 3;
constexpr int SFA_STAGE = 2048, SFB_STAGE = 4096;
constexpr int SMEM_BYTES4 =
    FP4_STAGES * (A_STAGE + B_STAGE + SFA_STAGE + SFB_STAGE) + 1024 + 256 + 2048 + 4 * 4096;
constexpr uint32_t FP4_ACC1 = 192, TM_SFA = 448, TM_SFB = 464;

// ---------------------------------------------------------------- PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// 16-byte cp.async global -> shared (L2 only), and the arrive-on-completion
// of the calling thread's cp.asyncs on an mbarrier (counts as one arrival).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Split form for software pipelining: the registers of an issued load must
// not be read before tcgen05.wait::ld.
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms 1024 B
// apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// Kernel modes: SwiGLU-fused bf16 (GEMM1), plain bf16 (GEMM2), the exact
// int8 x int8 -> int32 mode of the router (kind::i8, order-free accumulation),
// and the W8A8 e4m3 modes (kind::f8f6f4, scales applied in the epilogue).
constexpr int kSwiGLU = 0, kPlain = 1, kInt8 = 2, kSwiGLU8 = 3, kPlain8 = 4, kSwiGLU4 = 5,
              kPlain4 = 6;
template <int MODE>
__host__ __device__ constexpr bool is_fp4() {
  return MODE == kSwiGLU4 || MODE == kPlain4;
}
// Instruction descriptor, both operands K-major, M=128, N=256:
//   f16 kind:    bf16 x bf16 -> fp32 (c_format 1, a/b_format 1 = BF16)
//   i8 kind:     s8 x s8 -> s32      (c_format 2, a/b_format 1 = signed)
//   f8f6f4 kind: e4m3 x e4m3 -> fp32 (c_format 1, a/b_format 0 = E4M3)
//   mxf4nvf4:    e2m1 x e2m1 -> fp32 with e4m3 block scales (block-scaled
//                descriptor: a/b_format 1 = E2M1, scale_format 0 = UE4M3,
//                no c_format field, scale-factor ids 0)
template <int MODE>
__host__ __device__ constexpr uint32_t idesc() {
  if (is_fp4<MODE>())
    return (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
  return (MODE == kInt8 ? (2u << 4) : (1u << 4)) |
         (MODE == kSwiGLU8 || MODE == kPlain8 ? 0u : (1u << 7) | (1u << 10)) |
         (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}
__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc_v, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc_v), "r"(accum));
}
__device__ __forceinline__ void tc_mma_f8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc_v, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc_v), "r"(accum));
}

__device__ __forceinline__ void tc_mma_fp4(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc_v, uint32_t accum, uint32_t sfa,
                                           uint32_t sfb) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc_v), "r"(accum), "r"(sfa), "r"(sfb));
}
// smem -> TMEM copy of one 512-byte block-scale atom: 32 rows x 128 bit,
// replicated into the four lane quarters (each lane of quarter q then holds
// rows lane + 32 j in column j, the layout the block-scaled MMA reads).
// Its smem descriptor: no-swizzle K-major, 8-row core matrices 128 B apart
// (SBO), version 1.
__device__ __forceinline__ uint64_t sf_desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(128 >> 4) << 32) | (uint64_t(1) << 46);
}
__device__ __forceinline__ void tc_cp_sf_d(uint32_t taddr, uint64_t d) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(d) : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile(
      "{\n.reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, e;\n}"
      : "=r"(p));
  return p != 0;
}
// 1-D bulk copy global -> shared, completion on an mbarrier.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  return uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(a))) |
         (uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(b))) << 16);
}

// Group tables, or a single dense group (GemmArgs::dense_m > 0: expert 0 in
// slot 0, no device tables or meta; rows >= dense_m are not stored).
__device__ __forceinline__ int g_expert(const GemmArgs& p, int mb) {
  return p.mblock_expert ? p.mblock_expert[mb] : 0;
}
__device__ __forceinline__ int g_slot(const GemmArgs& p, int e) { return p.slot_of ? p.slot_of[e] : 0; }
__device__ __forceinline__ int g_total_mb(const GemmArgs& p) {
  return p.dense_m > 0 ? int((p.dense_m + 127) / 128) : p.meta[0];
}
__device__ __forceinline__ int g_routed_mb(const GemmArgs& p) {
  return p.dense_m > 0 ? int((p.dense_m + 127) / 128) : p.meta[1];
}

// Linear tile id -> (m-block, n-block). Tiles of a segment (consecutive
// m-blocks of one expert) occupy the id range [start*NB, (start+len)*NB), so
// the segment is found from the m-block tile/NB falls in. Inside a segment the
// raster keeps the smaller operand set live in L2 while the ~148 concurrent
// tiles sweep the other: n-block-major (all of the segment's A rows live, B
// n-blocks streamed once) while the segment's A rows (len*128 per K) are at
// most its B rows (NB*256 per K) -- every routed expert -- and m-block-major
// (B live, A streamed once) for long segments such as the shared expert's
// T rows, which n-major would re-read from HBM once per n-block.
__device__ __forceinline__ void tile_coords(int tile, int nb_count, const int2* __restrict__ seg,
                                            int raster, int& mb, int& nb) {
  mb = tile / nb_count;
  nb = tile - mb * nb_count;
  if (seg && raster != 1) {
    const int2 s = seg[mb];
    if (raster == 2 || s.y <= 2 * nb_count) {
      const int local = tile - s.x * nb_count;
      nb = local / s.y;
      mb = s.x + (local - nb * s.y);
    }
  }
}

// Epilogue of one 128 x BN accumulator tile: warp q of the epilogue group
// owns TMEM lanes (rows) 32q..32q+31; tbase addresses this warp's lanes and
// the tile's accumulator columns.
// TMA store of one epilogue chunk: the warp's 32 rows x 32 bf16 columns
// (2 KB) go through a double-buffered SWIZZLE_64B smem box; 16-byte stores of
// 32 different rows straight from registers cost one L1 wavefront each and
// were the NVFP4 GEMM2's bottleneck (6.8 -> 4.5 ms without them).
__device__ __forceinline__ void tma_store_box(uint8_t* stage, int* nstore, const CUtensorMap* tmD,
                                              const uint32_t* pk, int lane, bool store, int col, int row) {
  uint8_t* sb = stage + (*nstore & 1) * 2048;
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  __syncwarp();
#pragma unroll
  for (int w = 0; w < 4; ++w)
    *reinterpret_cast<uint4*>(sb + lane * 64 + ((w ^ ((lane >> 1) & 3)) << 4)) =
        make_uint4(pk[4 * w], pk[4 * w + 1], pk[4 * w + 2], pk[4 * w + 3]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const bool any = __any_sync(0xffffffffu, store);
  if (lane == 0 && any) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(tmD)),
                 "r"(col), "r"(row), "r"(smem_u32(sb))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  ++*nstore;
}

// NVFP4 tiles start at column `start` (mod the tile width) and arrive on
// `part` after the first two 32-column chunks: those cover the columns the
// other accumulator overlaps.
// Scaled modes: `ssc` (optional) holds the tile's weight-row scales in
// shared memory (SwiGLU: 128 gate then 128 up; plain: 256) and sa_in the
// row's activation scale, both fetched before the accumulator wait.
template <int MODE>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& p, int mb, int nb, uint32_t tbase, int q,
                                              int lane, int start = 0, uint64_t* part = nullptr,
                                              const float* ssc = nullptr, float sa_in = 1.0f,
                                              uint32_t part_cl = 0, uint8_t* stage = nullptr,
                                              int* nstore = nullptr, const CUtensorMap* tmD = nullptr) {
  constexpr bool SWIGLU = MODE == kSwiGLU || MODE == kSwiGLU8 || MODE == kSwiGLU4;
  constexpr bool FP8 = MODE == kSwiGLU8 || MODE == kPlain8 || is_fp4<MODE>();  // scaled epilogue
  auto release = [&](int i) {  // local barrier, or the CTA-pair leader's (cluster address)
    if ((part != nullptr || part_cl != 0) && i == 1) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (part_cl != 0)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(part_cl)
                       : "memory");
        else
          mbar_arrive(part);
      }
    }
  };
  const int64_t arow = int64_t(mb) * BM + q * 32 + lane;  // A row (activation scale)
  const int64_t drow0 = p.d_row0 != nullptr ? int64_t(p.d_row0[mb]) : int64_t(mb) * BM;
  const int64_t row = drow0 + q * 32 + lane;                // output row
  const bool store = arow < p.m_limit && (p.mb_rows == nullptr || q * 32 + lane < p.mb_rows[mb]);
  // fp8: per-row activation scale x per-output-channel weight scale
  float sa = 1.0f;
  const float* sb0 = nullptr;
  const float* sb1 = nullptr;
  if (FP8 && ssc != nullptr) {
    sa = sa_in;
    sb0 = ssc;
    sb1 = ssc + 128;
  } else if (FP8) {
    sa = p.a_scale[arow];
    const int64_t b0 = int64_t(g_slot(p, g_expert(p, mb))) * p.rows_per_slot +
                       int64_t(nb) * (SWIGLU ? 128 : BN);
    sb0 = p.b_scale0 + b0;
    sb1 = SWIGLU ? p.b_scale1 + b0 : nullptr;
  }
  // 16-byte scale loads: shared (broadcast) or read-only global
  auto ld4 = [&](const float* ptr) {
    return ssc != nullptr ? *reinterpret_cast<const float4*>(ptr)
                          : __ldg(reinterpret_cast<const float4*>(ptr));
  };
  if (MODE == kInt8) {
    int32_t* out = reinterpret_cast<int32_t*>(p.D) + row * p.ldd + nb * BN;
    const int cols = p.n_out - nb * BN < BN ? p.n_out - nb * BN : BN;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      tmem_ld32(tbase + c, v);
      if (store && c < cols) {
        if (c + 32 <= cols) {
          int4* o4 = reinterpret_cast<int4*>(out + c);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            o4[i] = make_int4(__float_as_int(v[4 * i]), __float_as_int(v[4 * i + 1]),
                              __float_as_int(v[4 * i + 2]), __float_as_int(v[4 * i + 3]));
        } else {
          for (int i = 0; i < cols - c; ++i) out[c + i] = __float_as_int(v[i]);
        }
      }
    }
  } else if (SWIGLU) {
    // the gate/up columns of chunks 0 and 1 (NVFP4: the overlapped ones) are
    // read and released before processing; afterwards chunk i+1 loads while
    // chunk i is processed
    uint16_t* out = p.D + row * p.ldd + nb * 128;
    uint32_t gb[2][32], ub[2][32];
    tmem_ld32_issue(tbase + (start & 127), gb[0]);
    tmem_ld32_issue(tbase + 128 + (start & 127), ub[0]);
    tmem_ld32_issue(tbase + ((start + 32) & 127), gb[1]);
    tmem_ld32_issue(tbase + 128 + ((start + 32) & 127), ub[1]);
    tmem_ld_wait();
    release(1);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = (start + 32 * i) & 127;
      if (i >= 1 && i + 1 < 4) {
        tmem_ld32_issue(tbase + ((start + 32 * (i + 1)) & 127), gb[(i + 1) & 1]);
        tmem_ld32_issue(tbase + 128 + ((start + 32 * (i + 1)) & 127), ub[(i + 1) & 1]);
      }
      float g[32], u[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        g[j] = __uint_as_float(gb[i & 1][j]);
        u[j] = __uint_as_float(ub[i & 1][j]);
      }
      if (FP8) {  // weight-row scales: 16-byte broadcast loads
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 s0 = ld4(sb0 + c + j);
          const float4 s1 = ld4(sb1 + c + j);
          g[j] *= sa * s0.x;
          g[j + 1] *= sa * s0.y;
          g[j + 2] *= sa * s0.z;
          g[j + 3] *= sa * s0.w;
          u[j] *= sa * s1.x;
          u[j + 1] *= sa * s1.y;
          u[j + 2] *= sa * s1.z;
          u[j + 3] *= sa * s1.w;
        }
      }
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float g0 = g[2 * j], g1 = g[2 * j + 1];
        const float h0 = __fdividef(g0, 1.0f + __expf(-g0)) * u[2 * j];
        const float h1 = __fdividef(g1, 1.0f + __expf(-g1)) * u[2 * j + 1];
        pk[j] = pack_bf16(h0, h1);
      }
      if (stage != nullptr)
        tma_store_box(stage, nstore, tmD, pk, lane, store, nb * 128 + c, int(drow0 + q * 32));
      else if (store) {
        uint4* o4 = reinterpret_cast<uint4*>(out + c);
#pragma unroll
        for (int w = 0; w < 4; ++w)
          o4[w] = make_uint4(pk[4 * w], pk[4 * w + 1], pk[4 * w + 2], pk[4 * w + 3]);
      }
      if (i >= 1 && i + 1 < 4) tmem_ld_wait();  // chunk i+1 landed
    }
  } else {
    // plain: chunks 0 and 1 (the columns the other accumulator overlaps, for
    // NVFP4) are read first and released before any processing; afterwards
    // the TMEM load of chunk i+2 is in flight while chunk i is scaled, packed
    // and stored (GEMM2's short K leaves the drain on the critical path)
    uint16_t* out = p.D + row * p.ldd + nb * BN;
    constexpr int NCH = BN / 32;
    uint32_t buf[3][32];
    tmem_ld32_issue(tbase + (start & (BN - 1)), buf[0]);
    tmem_ld32_issue(tbase + ((start + 32) & (BN - 1)), buf[1]);
    tmem_ld_wait();
    release(1);
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const int c = (start + 32 * i) & (BN - 1);
      if (i + 2 < NCH) tmem_ld32_issue(tbase + ((start + 32 * (i + 2)) & (BN - 1)), buf[(i + 2) % 3]);
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(buf[i % 3][j]);
      if (FP8) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 s0 = ld4(sb0 + c + j);
          v[j] *= sa * s0.x;
          v[j + 1] *= sa * s0.y;
          v[j + 2] *= sa * s0.z;
          v[j + 3] *= sa * s0.w;
        }
      }
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
      if (stage != nullptr) {
        tma_store_box(stage, nstore, tmD, pk, lane, store, nb * BN + c, int(drow0 + q * 32));
      } else if (store) {
        uint4* o4 = reinterpret_cast<uint4*>(out + c);
#pragma unroll
        for (int w = 0; w < 4; ++w)
          o4[w] = make_uint4(pk[4 * w], pk[4 * w + 1], pk[4 * w + 2], pk[4 * w + 3]);
      }
      if (i + 2 < NCH) tmem_ld_wait();  // chunk i+2 landed
    }
  }
}

// At most 232 registers per thread: two GEMM warps per SM sub-partition
// (2 x 32 x 232 of its 16K registers) leave room for the 32-thread pull
// kernel's warp (36 registers) beside the GEMM CTA. At 238 (the compiler's
// free choice) the pull CTAs and the GEMM could not co-reside and GEMM1 waited
// for the whole pull (11 -> 27-35 ms per layer with the pull engine).
template <int MODE>
__global__ void __maxnreg__(232)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmA2,
                        const __grid_constant__ CUtensorMap tmB0,
                        const __grid_constant__ CUtensorMap tmB1,
                        const __grid_constant__ CUtensorMap tmD, GemmArgs p) {
  constexpr bool FP4 = is_fp4<MODE>();
  constexpr int NST = FP4 ? FP4_STAGES : STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + NST * A_STAGE;
  uint8_t* sSFA = sB + NST * B_STAGE;                     // NVFP4 only
  uint8_t* sSFB = sSFA + (FP4 ? NST * SFA_STAGE : 0);
  constexpr bool TMA_ST = MODE == kPlain4;  // NVFP4 GEMM2: TMA-store epilogue
  uint8_t* sStage = sSFB + (FP4 ? NST * SFB_STAGE : 0);  // [4 warps][2][2 KB]
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + (TMA_ST ? 4 * 4096 : 0));
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 2;
  uint64_t* tpart = tempty + 2;  // NVFP4: overlapped accumulator columns drained
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tpart + 2);
  float* sscale = reinterpret_cast<float*>(tmem_holder + 4);  // [2][256] scaled modes (16-B aligned)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      // gathering: + one cp.async-completion arrival per producer lane
      mbar_init(&full[s], p.a_rows != nullptr ? 33 : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
      mbar_init(&tpart[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB0)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int total_mb = g_total_mb(p);
  const int routed_mb = g_routed_mb(p);
  constexpr bool SWIGLU = MODE == kSwiGLU || MODE == kSwiGLU8 || MODE == kSwiGLU4;
  constexpr bool FP8 = MODE == kSwiGLU8 || MODE == kPlain8;
  // K elements per 128-byte smem row, and the TMA column step (map elements)
  constexpr int BKE = FP4 ? 256 : (MODE == kInt8 || FP8) ? 128 : 64;
  constexpr int BKC = FP4 ? 128 : BKE;
  const int nb_count = SWIGLU ? p.n_out / 128 : (p.n_out + BN - 1) / BN;
  const int num_tiles = total_mb * nb_count;
  const int kb_count = p.K / BKE;
  const int64_t sf_chunks = p.K / 64;  // NVFP4: 512-byte scale atoms per 128 rows

  if (warp == 0) {  // ------------------ TMA producer (lane 0; all lanes when gathering)
    int s = 0;
    uint32_t ph = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int mb, nb;
      tile_coords(tile, nb_count, p.mb_seg, p.raster, mb, nb);
      const int e = g_expert(p, mb);
      const bool sh = p.shared_a2 && e == p.E;
      const bool gather = p.a_rows != nullptr && !sh;
      const CUtensorMap* am = sh ? &tmA2 : &tmA;
      const int arow = (sh ? mb - routed_mb : mb) * BM;
      const int brow = g_slot(p, e) * p.rows_per_slot + nb * (SWIGLU ? 128 : BN);
      // gather mode: lane l copies rows 4l..4l+3 of the m-block (8 x 16 B per
      // row and k-block) into the SWIZZLE_128B layout TMA would have produced
      const char* srow[4];
      if (gather)
        for (int i = 0; i < 4; ++i)
          srow[i] = reinterpret_cast<const char*>(
              p.a_src + int64_t(p.a_rows[int64_t(mb) * BM + 4 * lane + i]) * p.a_ld);
      // (L2 priority hints on these loads were measured and rejected: evict-first
      // on the streamed operand made GEMM1 read 210 GB from HBM instead of 37;
      // evict-last on the reused one cut the isolated kernel's HBM reads to
      // 26 GB but its lines outlive the kernel and slowed the full step 11%.)
      for (int kb = 0; kb < kb_count; ++kb) {
        if (lane == 0) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], (gather ? 0 : A_STAGE) + B_STAGE +
                                       (FP4 ? SFA_STAGE + SFB_STAGE : 0));
          if (!gather) tma_load_2d(sA + s * A_STAGE, am, &full[s], kb * BKC, arow);
          if (SWIGLU) {
            tma_load_2d(sB + s * B_STAGE, &tmB0, &full[s], kb * BKC, brow);
            tma_load_2d(sB + s * B_STAGE + B_STAGE / 2, &tmB1, &full[s], kb * BKC, brow);
          } else {
            tma_load_2d(sB + s * B_STAGE, &tmB0, &full[s], kb * BKC, brow);
          }
          if (FP4) {  // block scales: 4 atoms (one per 64-deep MMA) per 128 rows
            const int64_t ko = int64_t(4 * kb) * 512;
            bulk_load(sSFA + s * SFA_STAGE, p.a_sf + (int64_t(arow >> 7) * sf_chunks) * 512 + ko,
                      SFA_STAGE, &full[s]);
            const int64_t rb = brow >> 7;  // B row block (gate / down rows)
            if (SWIGLU) {
              bulk_load(sSFB + s * SFB_STAGE, p.b_sf0 + rb * sf_chunks * 512 + ko, 2048, &full[s]);
              bulk_load(sSFB + s * SFB_STAGE + 2048, p.b_sf1 + rb * sf_chunks * 512 + ko, 2048,
                        &full[s]);
            } else {
              bulk_load(sSFB + s * SFB_STAGE, p.b_sf0 + rb * sf_chunks * 512 + ko, 2048, &full[s]);
              bulk_load(sSFB + s * SFB_STAGE + 2048, p.b_sf0 + (rb + 1) * sf_chunks * 512 + ko, 2048,
                        &full[s]);
            }
          }
        }
        if (p.a_rows != nullptr) {
          __syncwarp();  // slot s is free (lane 0 waited on it)
          if (gather) {
            const uint32_t base = smem_u32(sA + s * A_STAGE);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int r = 4 * lane + i;
              const char* src = srow[i] + int64_t(kb) * 128;
#pragma unroll
              for (int c = 0; c < 8; ++c)
                cp_async16(base + uint32_t(r * 128 + ((c ^ (r & 7)) << 4)), src + c * 16);
            }
          }
          cp_async_arrive_noinc(&full[s]);  // every lane, every stage (count 33)
        }
        if (++s == NST) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1 && FP4) {  // ---------- NVFP4 MMA issuer (whole warp, one elected lane)
    // Per k-block: 12 smem->TMEM scale copies and 4 block-scaled MMAs. The
    // warp stays converged and elects once per k-block, and descriptors are
    // a per-stage base plus immediates, so the issue loop stays shorter than
    // the 4 MMAs it feeds.
    int s = 0;
    uint32_t ph = 0;
    int local = 0;
    const uint64_t sfa0 = sf_desc(smem_u32(sSFA)), sfb0 = sf_desc(smem_u32(sSFB));
    const uint64_t ad0 = sw128_desc(smem_u32(sA)), bd0 = sw128_desc(smem_u32(sB));
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int a = local & 1;
      mbar_wait(&tempty[a], ((local >> 1) & 1) ^ 1);
      // the accumulators overlap: the previous tile's epilogue must have
      // drained the shared columns
      if (local > 0) mbar_wait(&tpart[a ^ 1], ((local - 1) >> 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem_base + uint32_t(a) * FP4_ACC1;
      for (int kb = 0; kb < kb_count; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          // descriptor start addresses are in 16-byte units
          const uint64_t sfa = sfa0 + uint64_t(s * (SFA_STAGE >> 4));
          const uint64_t sfb = sfb0 + uint64_t(s * (SFB_STAGE >> 4));
          const uint64_t ad = ad0 + uint64_t(s * (A_STAGE >> 4));
          const uint64_t bd = bd0 + uint64_t(s * (B_STAGE >> 4));
          // tcgen05.cp and tcgen05.mma execute in issue order, so one TMEM
          // copy of the scales suffices
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            tc_cp_sf_d(tmem_base + TM_SFA + 4 * k, sfa + 32 * k);
            tc_cp_sf_d(tmem_base + TM_SFB + 8 * k, sfb + 32 * k);
            tc_cp_sf_d(tmem_base + TM_SFB + 8 * k + 4, sfb + 128 + 32 * k);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k)  // 64 e2m1 (32 B) along K per MMA
            tc_mma_fp4(d, ad + 2 * k, bd + 2 * k, idesc<MODE>(), (kb | k) != 0,
                       tmem_base + TM_SFA + 4 * k, tmem_base + TM_SFB + 8 * k);
          tc_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == NST) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) tc_commit(&tfull[a]);
      __syncwarp();
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      int s = 0;
      uint32_t ph = 0;
      int local = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
        const int a = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&tempty[a], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(a * BN);
        for (int kb = 0; kb < kb_count; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (p.a_rows != nullptr)  // cp.async (generic proxy) writes -> tcgen05 (async proxy) reads
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          const uint64_t ad = sw128_desc(smem_u32(sA + s * A_STAGE));
          const uint64_t bd = sw128_desc(smem_u32(sB + s * B_STAGE));
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // +32 B along K per MMA (16 bf16 or 32 int8)
            if (MODE == kInt8)
              tc_mma_i8(d, ad + 2 * k, bd + 2 * k, idesc<MODE>(), (kb | k) != 0);
            else if (FP8)
              tc_mma_f8(d, ad + 2 * k, bd + 2 * k, idesc<MODE>(), (kb | k) != 0);
            else
              tc_mma(d, ad + 2 * k, bd + 2 * k, idesc<MODE>(), (kb | k) != 0);
          }
          tc_commit(&empty[s]);
          if (++s == NST) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit(&tfull[a]);
      }
    }
  } else if (warp >= 4) {  // ------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int local = 0;
    constexpr bool SCALED = FP8 || FP4;
    const int et = q * 32 + lane;  // 0..127: this thread's row of the tile
    // scaled modes: the scales of tile i+1 are loaded into registers while
    // tile i drains, so no global-load latency sits inside a drain; they are
    // staged in a double-buffered smem copy (one named barrier per tile)
    float n0 = 0.0f, n1 = 0.0f, nsa = 1.0f;
    auto fetch_scales = [&](int t) {
      int m, n;
      tile_coords(t, nb_count, p.mb_seg, p.raster, m, n);
      const int64_t b0 = int64_t(g_slot(p, g_expert(p, m))) * p.rows_per_slot +
                         int64_t(n) * (SWIGLU ? 128 : BN);
      n0 = __ldg(p.b_scale0 + b0 + et);
      n1 = SWIGLU ? __ldg(p.b_scale1 + b0 + et) : __ldg(p.b_scale0 + b0 + 128 + et);
      nsa = int64_t(m) * BM + et < p.m_limit ? __ldg(p.a_scale + int64_t(m) * BM + et) : 1.0f;
    };
    if (SCALED && blockIdx.x < num_tiles) fetch_scales(blockIdx.x);
    int nstore = 0;  // TMA-store boxes issued by this warp (buffer parity)
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      int mb, nb;
      tile_coords(tile, nb_count, p.mb_seg, p.raster, mb, nb);
      const int a = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      const float pre0 = n0, pre1 = n1, sa = nsa;
      if (SCALED && tile + int(gridDim.x) < num_tiles) fetch_scales(tile + gridDim.x);
      mbar_wait(&tfull[a], aph);
      tc_fence_after();
      float* ssc = sscale + (local & 1) * 256;
      if (SCALED) {
        // buffer local&1 was last read in tile local-2, before every thread
        // passed the barrier of tile local-1
        ssc[et] = pre0;
        ssc[128 + et] = pre1;
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      const uint32_t lanes = uint32_t(q * 32) << 16;
      if (FP4)  // accumulator 0 overlaps accumulator 1 in its last 64 columns
        epilogue_tile<MODE>(p, mb, nb, tmem_base + lanes + uint32_t(a) * FP4_ACC1, q, lane,
                            a == 0 ? (SWIGLU ? 64 : 192) : 0, &tpart[a], ssc, sa, 0,
                            TMA_ST ? sStage + q * 4096 : nullptr, &nstore, &tmD);
      else if (SCALED)
        epilogue_tile<MODE>(p, mb, nb, tmem_base + lanes + uint32_t(a * BN), q, lane, 0, nullptr,
                            ssc, sa);
      else
        epilogue_tile<MODE>(p, mb, nb, tmem_base + lanes + uint32_t(a * BN), q, lane);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
    }
    // the staged boxes must be read out before the CTA's smem goes away
    if (TMA_ST && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- CTA pair
// 2-SM variant (cta_group::2) for the bf16 expert GEMMs. A cluster of two
// CTAs on one TPC computes a 256 x 256 tile: CTA r loads A rows of m-block
// 2*pair + r and half of B (SwiGLU: r = 0 the 128 gate rows, r = 1 the 128 up
// rows; plain: B rows [128r, 128r + 128) of the n-block), and the leader's
// single thread issues M256 x N256 x K16 MMAs that read A and B from both
// CTAs' shared memory and accumulate each CTA's 128 rows in its own TMEM. Per
// CTA this halves the B bytes moved from L2 and read from shared memory per
// MMA flop (32 KB per 64-deep k-block instead of 48 KB). Requires expert
// segments padded to 256 rows (permute row_align 256), so both m-blocks of a
// pair always belong to the same expert.
constexpr int P_STAGE = 2 * BM * BK * 2;  // A (16 KB) + half of B (16 KB) per CTA
// 6 stages (194 KB) leave room on every SM for one prefetch pull CTA (26 KB):
// with 7 the pull kernel could not co-reside and DWDP at N=4 fell 10-20%;
// with 5 GEMM2's tensor pipe dropped from 94% to 86% active.
constexpr int P_STAGES = 6;
constexpr int P_SMEM_BYTES = P_STAGES * P_STAGE + 1024 + 256;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_rank(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// TMA tile load into this CTA's smem whose completion is signalled on the
// leader CTA's mbarrier (cluster address).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cl,
                                                 int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cl), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_mma_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc_v, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc_v), "r"(accum));
}
// Commit the leader's MMAs to the same-offset mbarrier in both CTAs.
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
// M = 256 (pair), N = 256, both operands K-major: bf16 x bf16 -> fp32 or
// e4m3 x e4m3 -> fp32 (a/b_format 0).
template <int MODE>
__host__ __device__ constexpr uint32_t pair_idesc() {
  return (MODE == kInt8 ? (2u << 4) : (1u << 4)) |
         (MODE == kSwiGLU8 || MODE == kPlain8 ? 0u : (1u << 7) | (1u << 10)) |
         (uint32_t(BN >> 3) << 17) | (uint32_t(256 >> 4) << 24);
}
__device__ __forceinline__ void tc_mma_pair_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc_v, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc_v), "r"(accum));
}
__device__ __forceinline__ void tc_mma_pair_f8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc_v, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc_v), "r"(accum));
}

// Pair tile id -> (pair index, n-block); segments in m-blocks are even.
__device__ __forceinline__ void pair_coords(int tile, int nb_count, const int2* __restrict__ seg,
                                            int raster, int& mp, int& nb) {
  mp = tile / nb_count;
  nb = tile - mp * nb_count;
  if (seg && raster != 1) {
    const int2 s = seg[2 * mp];
    const int px = s.x >> 1, py = s.y >> 1;
    if (raster == 2 || py <= nb_count) {  // A rows (256 per pair) <= B rows (256 per n-block): n-major
      const int local = tile - px * nb_count;
      nb = local / py;
      mp = px + (local - nb * py);
    }
  }
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    grouped_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                             const __grid_constant__ CUtensorMap tmA2,
                             const __grid_constant__ CUtensorMap tmB0,
                             const __grid_constant__ CUtensorMap tmB1, GemmArgs p) {
  constexpr bool SWIGLU = MODE == kSwiGLU || MODE == kSwiGLU8;
  constexpr bool FP8 = MODE == kSwiGLU8 || MODE == kPlain8;
  constexpr int BKE = (FP8 || MODE == kInt8) ? 128 : 64;  // K elements per 128-byte smem row
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P_STAGES * P_STAGE);
  uint64_t* empty = full + P_STAGES;
  uint64_t* tfull = empty + P_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  auto sA = [&](int st) { return smem + st * P_STAGE; };
  auto sB = [&](int st) { return smem + st * P_STAGE + BM * BK * 2; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) {
    for (int st = 0; st < P_STAGES; ++st) {
      mbar_init(&full[st], 1);   // leader: its expect_tx arrive (both CTAs' TMA bytes)
      mbar_init(&empty[st], 1);  // one multicast commit per stage use
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // leader: 4 local + 4 peer epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB0)) : "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int total_mb = g_total_mb(p);
  const int routed_mb = g_routed_mb(p);
  const int nb_count = SWIGLU ? p.n_out / 128 : (p.n_out + BN - 1) / BN;
  const int num_tiles = (total_mb >> 1) * nb_count;
  const int kb_count = p.K / BKE;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {  // ------------------ TMA producer (both CTAs)
      const uint32_t full_cl0 = map_to_rank(&full[0], 0);  // leader's full[0]
      int st = 0;
      uint32_t ph = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl) {
        int mp, nb;
        pair_coords(tile, nb_count, p.mb_seg, p.raster, mp, nb);
        const int mb = 2 * mp + int(rank);
        const int e = g_expert(p, mb);
        const bool sh = p.shared_a2 && e == p.E;
        const CUtensorMap* am = sh ? &tmA2 : &tmA;
        const int arow = (sh ? mb - routed_mb : mb) * BM;
        const CUtensorMap* bm = (SWIGLU && rank == 1) ? &tmB1 : &tmB0;
        const int brow = g_slot(p, e) * p.rows_per_slot +
                         (SWIGLU ? nb * 128 : nb * BN + int(rank) * 128);
        for (int kb = 0; kb < kb_count; ++kb) {
          mbar_wait(&empty[st], ph ^ 1);
          const uint32_t bar = full_cl0 + uint32_t(st) * 8u;
          // Only the leader arrives (expecting both CTAs' bytes). The peer's
          // complete_tx may land first (the phase cannot complete while the
          // leader's arrival is pending); a remote arrive from the peer would
          // put a cluster-scope release fence in front of every load.
          if (rank == 0) mbar_expect_tx(&full[st], 2 * P_STAGE);
          tma_load_2d_pair(sA(st), am, bar, kb * BKE, arow);
          tma_load_2d_pair(sB(st), bm, bar, kb * BKE, brow);
          if (++st == P_STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---------------- MMA issuer (leader only)
      int st = 0;
      uint32_t ph = 0;
      int local = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl, ++local) {
        const int a = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&tempty[a], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(a * BN);
        for (int kb = 0; kb < kb_count; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint64_t ad = sw128_desc(smem_u32(sA(st)));
          const uint64_t bd = sw128_desc(smem_u32(sB(st)));
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // +32 B along K per MMA (16 bf16 or 32 e4m3)
            if (MODE == kInt8)
              tc_mma_pair_i8(d, ad + 2 * k, bd + 2 * k, pair_idesc<MODE>(), (kb | k) != 0);
            else if (FP8)
              tc_mma_pair_f8(d, ad + 2 * k, bd + 2 * k, pair_idesc<MODE>(), (kb | k) != 0);
            else
              tc_mma_pair(d, ad + 2 * k, bd + 2 * k, pair_idesc<MODE>(), (kb | k) != 0);
          }
          tc_commit_pair(&empty[st]);
          if (++st == P_STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
        tc_commit_pair(&tfull[a]);
      }
    }
  } else if (warp >= 4) {  // ------------- epilogue (both CTAs, own 128 rows)
    const int q = warp & 3;
    const uint32_t tempty_cl0 = map_to_rank(&tempty[0], 0);
    int local = 0;
    for (int tile = cid; tile < num_tiles; tile += ncl, ++local) {
      int mp, nb;
      pair_coords(tile, nb_count, p.mb_seg, p.raster, mp, nb);
      const int a = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      mbar_wait(&tfull[a], aph);
      tc_fence_after();
      epilogue_tile<MODE>(p, 2 * mp + int(rank), nb,
                          tmem_base + (uint32_t(q * 32) << 16) + uint32_t(a * BN), q, lane);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_cl0 + uint32_t(a) * 8u);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- NVFP4 CTA pair
// kind::mxf4nvf4 on CTA pairs (cta_group::2, M256 x N256 x K64 per MMA). Per
// CTA and k-block it moves A (its 128 rows, 16 KB), half of B (16 KB), the
// scales of its A rows (2 KB) and the scales of ALL 256 B rows (4 KB): 38 KB
// instead of the 1-SM kernel's 54 KB, whose L2->SM traffic (~24 TB/s needed at
// the fp4 MMA rate) is what bounds it. The leader's tcgen05.cp.cta_group::2
// copies each CTA's scale atoms into that CTA's TMEM (same offsets); the
// accumulators overlap as in the 1-SM kernel. Scale atoms arrive by 2-D TMA
// (128-byte rows, 16 rows = 2 KB) so that every load of both CTAs completes
// on the leader's barrier.
constexpr int P4_STAGES = 4;  // + 16 KB of TMA-store boxes
constexpr int P4_A = BM * 128, P4_B = 128 * 128, P4_SFA = 2048, P4_SFB = 4096;
constexpr int P4_STAGE = P4_A + P4_B + P4_SFA + P4_SFB;
constexpr int P4_SMEM_BYTES = P4_STAGES * P4_STAGE + 4 * 4096 + 1024 + 256 + 2048;

__device__ __forceinline__ void tc_mma_pair_fp4(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                                uint32_t idesc_v, uint32_t accum, uint32_t sfa,
                                                uint32_t sfb) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc_v), "r"(accum), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void tc_cp_sf_pair(uint32_t taddr, uint64_t d) {
  asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(d) : "memory");
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    grouped_gemm_pair_fp4_kernel(const __grid_constant__ CUtensorMap tmA,
                                 const __grid_constant__ CUtensorMap tmB0,
                                 const __grid_constant__ CUtensorMap tmB1,
                                 const __grid_constant__ CUtensorMap tmSA,
                                 const __grid_constant__ CUtensorMap tmSB0,
                                 const __grid_constant__ CUtensorMap tmSB1,
                                 const __grid_constant__ CUtensorMap tmD, GemmArgs p) {
  constexpr bool SWIGLU = MODE == kSwiGLU4;
  constexpr uint32_t IDESC = (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(256 >> 4) << 24);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  auto sA = [&](int st) { return smem + st * P4_STAGE; };
  auto sB = [&](int st) { return smem + st * P4_STAGE + P4_A; };
  auto sSA = [&](int st) { return smem + st * P4_STAGE + P4_A + P4_B; };
  auto sSB = [&](int st) { return smem + st * P4_STAGE + P4_A + P4_B + P4_SFA; };
  uint8_t* sStage = smem + P4_STAGES * P4_STAGE;  // [4 warps][2][2 KB] TMA-store boxes
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + 4 * 4096);
  uint64_t* empty = full + P4_STAGES;
  uint64_t* tfull = empty + P4_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* tpart = tempty + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tpart + 2);
  float* sscale = reinterpret_cast<float*>(tmem_holder + 4);  // [2][256]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) {
    for (int st = 0; st < P4_STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // leader: 4 local + 4 peer epilogue warps
      mbar_init(&tpart[a], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int total_mb = g_total_mb(p);
  const int nb_count = SWIGLU ? p.n_out / 128 : p.n_out / BN;
  const int num_tiles = (total_mb >> 1) * nb_count;
  const int kb_count = p.K / 256;
  const int64_t sf_rows_per_rb = int64_t(p.K / 64) * 4;  // 128-byte rows of scales per 128 data rows
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {  // ------------------ TMA producer (both CTAs)
      const uint32_t full_cl0 = map_to_rank(&full[0], 0);
      int st = 0;
      uint32_t ph = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl) {
        int mp, nb;
        pair_coords(tile, nb_count, p.mb_seg, p.raster, mp, nb);
        const int mb = 2 * mp + int(rank);
        const int slot = g_slot(p, g_expert(p, mb));
        const int arow = mb * BM;
        // B rows of this CTA's half, and the 128-row blocks of the whole N tile
        const CUtensorMap* bm = (SWIGLU && rank == 1) ? &tmB1 : &tmB0;
        const int brow = slot * p.rows_per_slot + (SWIGLU ? nb * 128 : nb * BN + int(rank) * 128);
        const int64_t rb0 = (int64_t(slot) * p.rows_per_slot + int64_t(nb) * (SWIGLU ? 128 : BN)) >> 7;
        const CUtensorMap* sb1 = SWIGLU ? &tmSB1 : &tmSB0;
        const int64_t rb1 = SWIGLU ? rb0 : rb0 + 1;
        for (int kb = 0; kb < kb_count; ++kb) {
          mbar_wait(&empty[st], ph ^ 1);
          const uint32_t bar = full_cl0 + uint32_t(st) * 8u;
          if (rank == 0) mbar_expect_tx(&full[st], 2 * P4_STAGE);
          tma_load_2d_pair(sA(st), &tmA, bar, kb * 128, arow);
          tma_load_2d_pair(sB(st), bm, bar, kb * 128, brow);
          tma_load_2d_pair(sSA(st), &tmSA, bar, 0, int((arow >> 7) * sf_rows_per_rb + 16 * kb));
          tma_load_2d_pair(sSB(st), &tmSB0, bar, 0, int(rb0 * sf_rows_per_rb + 16 * kb));
          tma_load_2d_pair(sSB(st) + 2048, sb1, bar, 0, int(rb1 * sf_rows_per_rb + 16 * kb));
          if (++st == P4_STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // ---------------- MMA issuer (leader warp, one elected lane)
      int st = 0;
      uint32_t ph = 0;
      int local = 0;
      const uint64_t a0 = sw128_desc(smem_u32(sA(0))), b0 = sw128_desc(smem_u32(sB(0)));
      const uint64_t sa0 = sf_desc(smem_u32(sSA(0))), sb0 = sf_desc(smem_u32(sSB(0)));
      for (int tile = cid; tile < num_tiles; tile += ncl, ++local) {
        const int a = local & 1;
        mbar_wait(&tempty[a], ((local >> 1) & 1) ^ 1);
        if (local > 0) mbar_wait(&tpart[a ^ 1], ((local - 1) >> 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(a) * FP4_ACC1;
        for (int kb = 0; kb < kb_count; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t off = uint64_t(st * (P4_STAGE >> 4));
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              tc_cp_sf_pair(tmem_base + TM_SFA + 4 * k, sa0 + off + 32 * k);
              tc_cp_sf_pair(tmem_base + TM_SFB + 8 * k, sb0 + off + 32 * k);
              tc_cp_sf_pair(tmem_base + TM_SFB + 8 * k + 4, sb0 + off + 128 + 32 * k);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_pair_fp4(d, a0 + off + 2 * k, b0 + off + 2 * k, IDESC, (kb | k) != 0,
                              tmem_base + TM_SFA + 4 * k, tmem_base + TM_SFB + 8 * k);
            tc_commit_pair(&empty[st]);
          }
          __syncwarp();
          if (++st == P4_STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
        if (elect_one()) tc_commit_pair(&tfull[a]);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {  // ------------- epilogue (both CTAs, own 128 rows)
    const int q = warp & 3;
    const int et = q * 32 + lane;
    const uint32_t tempty_cl0 = map_to_rank(&tempty[0], 0);
    const uint32_t tpart_cl0 = map_to_rank(&tpart[0], 0);
    float n0 = 0.0f, n1 = 0.0f, nsa = 1.0f;
    auto fetch_scales = [&](int t) {
      int mp, n;
      pair_coords(t, nb_count, p.mb_seg, p.raster, mp, n);
      const int m = 2 * mp + int(rank);
      const int64_t b0 = int64_t(g_slot(p, g_expert(p, m))) * p.rows_per_slot +
                         int64_t(n) * (SWIGLU ? 128 : BN);
      n0 = __ldg(p.b_scale0 + b0 + et);
      n1 = SWIGLU ? __ldg(p.b_scale1 + b0 + et) : __ldg(p.b_scale0 + b0 + 128 + et);
      nsa = int64_t(m) * BM + et < p.m_limit ? __ldg(p.a_scale + int64_t(m) * BM + et) : 1.0f;
    };
    if (cid < num_tiles) fetch_scales(cid);
    int nstore = 0;  // TMA-store boxes issued by this warp (buffer parity)
    int local = 0;
    for (int tile = cid; tile < num_tiles; tile += ncl, ++local) {
      int mp, nb;
      pair_coords(tile, nb_count, p.mb_seg, p.raster, mp, nb);
      const int a = local & 1;
      const float pre0 = n0, pre1 = n1, sa = nsa;
      if (tile + ncl < num_tiles) fetch_scales(tile + ncl);
      mbar_wait(&tfull[a], (local >> 1) & 1);
      tc_fence_after();
      float* ssc = sscale + (local & 1) * 256;
      ssc[et] = pre0;
      ssc[128 + et] = pre1;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      epilogue_tile<MODE>(p, 2 * mp + int(rank), nb,
                          tmem_base + (uint32_t(q * 32) << 16) + uint32_t(a) * FP4_ACC1, q, lane,
                          a == 0 ? (SWIGLU ? 64 : 192) : 0, nullptr, ssc, sa, tpart_cl0 + uint32_t(a) * 8u,
                          sStage + q * 4096, &nstore, &tmD);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_cl0 + uint32_t(a) * 8u);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- router
// Router logits with the digit-plane recombination fused into the GEMM.
// A = the activations' three int8 digit planes [3][T][h] (plane a weighs
// 2^8a), B = the router weights' planes [3][E][h]. A tile (128 tokens x 64
// experts) issues all nine plane products per k-block, accumulating the
// products of equal weight a + b = s in one int32 TMEM accumulator D_s
// (|D_s| <= 3 * h * 2^14 < 2^31 for h <= 43690), five accumulators of 64
// columns. The epilogue forms the exact z = sum_s D_s 2^8s in int64 and the
// fp32 logit ldexp(fp32(z), e_x + e_w - 296) -- the same single rounding as
// the oracle (dwdp_oracle.c route_one) -- and writes fp32 logits [T][E]:
// 4 B per (token, expert) instead of 36 B of int32 plane products.
constexpr int R_BN = 64;
constexpr int R_STAGES = 2;               // 144 KB: fits beside a 26 KB pull CTA
constexpr int R_A = 3 * BM * 128;         // 48 KB: 3 planes x 128 rows x 128 B of K
constexpr int R_B = 3 * R_BN * 128;       // 24 KB
constexpr int R_SMEM = R_STAGES * (R_A + R_B) + 1024 + 256;
constexpr uint32_t R_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(R_BN >> 3) << 17) |
                             (uint32_t(BM >> 4) << 24);
constexpr uint32_t R_IDESC3 = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(3 * R_BN >> 3) << 17) |
                              (uint32_t(BM >> 4) << 24);  // N = the 3 stacked weight planes

__global__ void __launch_bounds__(256, 1)
    router_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const int32_t* __restrict__ xe, const int32_t* __restrict__ we,
                       float* __restrict__ logits, int T, int E, int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sA + R_STAGES * R_A;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + R_STAGES * R_B);
  uint64_t* empty = full + R_STAGES;
  uint64_t* tfull = empty + R_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < R_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int nb_count = E / R_BN;
  const int num_tiles = (T + BM - 1) / BM * nb_count;
  const int kb_count = K / 128;
  if (warp == 0) {
    if (lane == 0) {  // TMA producer: the m-block's 3 A planes and the n-block's 3 B planes
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int mb = tile / nb_count, nb = tile - mb * nb_count;
        for (int kb = 0; kb < kb_count; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], R_A + R_B);
#pragma unroll
          for (int a = 0; a < 3; ++a)
            tma_load_2d(sA + s * R_A + a * (BM * 128), &tmA, &full[s], kb * 128, a * T + mb * BM);
#pragma unroll
          for (int b = 0; b < 3; ++b)
            tma_load_2d(sB + s * R_B + b * (R_BN * 128), &tmB, &full[s], kb * 128, b * E + nb * R_BN);
          if (++s == R_STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer. The B stage holds the three weight planes as 192
    // contiguous rows, so one M128 N192 MMA with A plane a writes the
    // products (a, 0..2) into columns [64a, 64a + 192) = D_a, D_{a+1},
    // D_{a+2}: three MMAs per K32 step instead of nine N64 ones (an SS-mode
    // N64 MMA is bound by its 6 KB of smem operand reads, 57 cycles for 32
    // of math, scripts/micro/mma_rate.cu). The tile's first K32 step uses
    // the nine N64 products so each D_s is overwritten exactly once. The
    // whole warp runs the schedule (warp-uniform descriptors); one elected
    // lane issues.
    int s = 0;
    uint32_t ph = 0;
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      mbar_wait(tempty, (local & 1) ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < kb_count; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint64_t ad = sw128_desc(smem_u32(sA + s * R_A));
        const uint64_t bd = sw128_desc(smem_u32(sB + s * R_B));
        if (elect_one()) {
          int k0 = 0;
          if (kb == 0) {  // first K32 step: D_s = the first product of weight s, then accumulate
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int b = 0; b < 3; ++b)
                tc_mma_i8(tmem + uint32_t((a + b) * R_BN), ad + uint64_t(a * (BM * 128 >> 4)),
                          bd + uint64_t(b * (R_BN * 128 >> 4)), R_IDESC, !(a == 0 || b == 2));
            k0 = 1;
          }
          for (int k = k0; k < 4; ++k)
#pragma unroll
            for (int a = 0; a < 3; ++a)
              tc_mma_i8(tmem + uint32_t(a * R_BN), ad + uint64_t(a * (BM * 128 >> 4)) + 2 * k, bd + 2 * k,
                        R_IDESC3, 1);
          tc_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == R_STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) tc_commit(tfull);
      __syncwarp();
    }
  } else if (warp >= 4) {  // epilogue: exact recombination, one rounding, fp32 logits
    const int q = warp & 3;
    const uint32_t lb = uint32_t(q * 32) << 16;
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int mb = tile / nb_count, nb = tile - mb * nb_count;
      const int t = mb * BM + q * 32 + lane;
      const int sx0 = t < T ? xe[t] - 296 : 0;
      mbar_wait(tfull, local & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < R_BN; c += 32) {
        long long z[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) z[i] = 0;
#pragma unroll
        for (int sidx = 0; sidx < 5; ++sidx) {
          uint32_t r[32];
          tmem_ld32_issue(tmem + lb + uint32_t(sidx * R_BN + c), r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) z[i] += static_cast<long long>(int32_t(r[i])) * (1LL << (8 * sidx));
        }
        if (c + 32 >= R_BN) {  // accumulators drained: the next tile's MMAs may start
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty);
        }
        if (t < T) {
          const int e0 = nb * R_BN + c;
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int sx = sx0 + __ldg(we + e0 + i);
            const float f = __ll2float_rn(z[i]);
            v[i] = (sx >= -126 && sx <= 127) ? __fmul_rn(f, __int_as_float((sx + 127) << 23)) : ldexpf(f, sx);
          }
          float4* o = reinterpret_cast<float4*>(logits + int64_t(t) * E + e0);
#pragma unroll
          for (int i = 0; i < 8; ++i) o[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------- router, CTA pairs
// router_gemm_pair_kernel: the same product on CTA pairs (cta_group::2, M =
// 256 tokens). Each CTA stages its own 128 token rows of the three activation
// planes and half of the 192 stacked weight rows (32-row boxes: rank r holds
// stacked rows [96r, 96r + 96)), so one M256 N192 K32 MMA per activation
// plane and K32 step reads 7 KB of shared memory per SM instead of 10 KB and
// stays under the MMA time. The accumulators are zeroed by the epilogue
// (after each drain, and once at start), so every product accumulates.
constexpr int RP_STAGES = 3;
constexpr int RP_A = 3 * BM * 128;  // 48 KB
constexpr int RP_B = 96 * 128;      // 12 KB
constexpr int RP_SMEM = RP_STAGES * (RP_A + RP_B) + 1024 + 256;
constexpr uint32_t RP_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(3 * R_BN >> 3) << 17) |
                              (uint32_t(256 >> 4) << 24);

__device__ __forceinline__ void tmem_st32_zero(uint32_t taddr) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(0u)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    router_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                            const int32_t* __restrict__ xe, const int32_t* __restrict__ we,
                            float* __restrict__ logits, int T, int E, int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto sA = [&](int st) { return smem + st * (RP_A + RP_B); };
  auto sB = [&](int st) { return smem + st * (RP_A + RP_B) + RP_A; };
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RP_STAGES * (RP_A + RP_B));
  uint64_t* empty = full + RP_STAGES;
  uint64_t* tfull = empty + RP_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) {
    for (int st = 0; st < RP_STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 8);  // leader: 4 local + 4 peer epilogue warps
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int nb_count = E / R_BN;
  const int num_tiles = (T + 2 * BM - 1) / (2 * BM) * nb_count;
  const int kb_count = K / 128;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs): own A rows, own half of the stacked weight rows
      const uint32_t full_cl0 = map_to_rank(&full[0], 0);
      int st = 0;
      uint32_t ph = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl) {
        const int mp = tile / nb_count, nb = tile - mp * nb_count;
        const int mb = 2 * mp + int(rank);
        for (int kb = 0; kb < kb_count; ++kb) {
          mbar_wait(&empty[st], ph ^ 1);
          const uint32_t bar = full_cl0 + uint32_t(st) * 8u;
          if (rank == 0) mbar_expect_tx(&full[st], 2 * (RP_A + RP_B));
#pragma unroll
          for (int a = 0; a < 3; ++a)
            tma_load_2d_pair(sA(st) + a * (BM * 128), &tmA, bar, kb * 128, a * T + mb * BM);
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const int srow = 96 * int(rank) + 32 * i;  // stacked row: plane srow / 64, row srow % 64
            tma_load_2d_pair(sB(st) + i * (32 * 128), &tmB, bar, kb * 128, (srow / 64) * E + nb * R_BN + srow % 64);
          }
          if (++st == RP_STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // MMA issuer (leader; whole warp, one elected lane issues)
      int st = 0;
      uint32_t ph = 0;
      int local = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl, ++local) {
        mbar_wait(tempty, local & 1);  // accumulators drained and zeroed
        tc_fence_after();
        for (int kb = 0; kb < kb_count; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint64_t ad = sw128_desc(smem_u32(sA(st)));
          const uint64_t bd = sw128_desc(smem_u32(sB(st)));
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int a = 0; a < 3; ++a)
                tc_mma_pair_i8(tmem + uint32_t(a * R_BN), ad + uint64_t(a * (BM * 128 >> 4)) + 2 * k, bd + 2 * k,
                               RP_IDESC, 1);
            tc_commit_pair(&empty[st]);
          }
          __syncwarp();
          if (++st == RP_STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
        if (elect_one()) tc_commit_pair(tfull);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {  // epilogue (both CTAs, own 128 rows): exact recombination, one rounding
    const int q = warp & 3;
    const uint32_t lb = uint32_t(q * 32) << 16;
    const uint32_t tempty_cl0 = map_to_rank(tempty, 0);
    auto zero_and_release = [&]() {
#pragma unroll
      for (int c = 0; c < 5 * R_BN; c += 32) tmem_st32_zero(tmem + lb + uint32_t(c));
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_cl0);
    };
    zero_and_release();
    int local = 0;
    for (int tile = cid; tile < num_tiles; tile += ncl, ++local) {
      const int mp = tile / nb_count, nb = tile - mp * nb_count;
      const int t = (2 * mp + int(rank)) * BM + q * 32 + lane;
      const int sx0 = t < T ? xe[t] - 296 : 0;
      mbar_wait(tfull, local & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < R_BN; c += 32) {
        long long z[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) z[i] = 0;
#pragma unroll
        for (int sidx = 0; sidx < 5; ++sidx) {
          uint32_t r[32];
          tmem_ld32_issue(tmem + lb + uint32_t(sidx * R_BN + c), r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) z[i] += static_cast<long long>(int32_t(r[i])) * (1LL << (8 * sidx));
        }
        if (c + 32 >= R_BN) zero_and_release();  // every accumulator column read: the next tile may start
        if (t < T) {
          const int e0 = nb * R_BN + c;
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int sx = sx0 + __ldg(we + e0 + i);
            const float f = __ll2float_rn(z[i]);
            v[i] = (sx >= -126 && sx <= 127) ? __fmul_rn(f, __int_as_float((sx + 127) << 23)) : ldexpf(f, sx);
          }
          float4* o = reinterpret_cast<float4*>(logits + int64_t(t) * E + e0);
#pragma unroll
          for (int i = 0; i < 8; ++i) o[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}


// ---------------------------------------------------------------- host
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
  return fn;
}


}  // namespace

CUtensorMap make_tmap_2d(const void* base, int64_t rows, int64_t cols, int box_rows, bool int8) {
  CUtensorMap m;
  const int esz = int8 ? 1 : 2;
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(cols) * esz};
  const cuuint32_t box[2] = {cuuint32_t(128 / esz), cuuint32_t(box_rows)};  // 128-byte rows
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encoder()(&m, int8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                               2, const_cast<void*>(base), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return m;
}

CUtensorMap make_tmap_3d_bf16(const void* base, const int64_t dims[3], const int64_t strides[2],
                              const int box[3]) {
  CUtensorMap m;
  const cuuint64_t d[3] = {cuuint64_t(dims[0]), cuuint64_t(dims[1]), cuuint64_t(dims[2])};
  const cuuint64_t st[2] = {cuuint64_t(strides[0]), cuuint64_t(strides[1])};
  const cuuint32_t b[3] = {cuuint32_t(box[0]), cuuint32_t(box[1]), cuuint32_t(box[2])};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), d, st, b, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled (3-D) failed (" + std::to_string(int(r)) + ")");
  return m;
}

CUtensorMap make_tmap_out(const void* base, int64_t rows, int64_t cols) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                               strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled (output) failed (" + std::to_string(int(r)) + ")");
  return m;
}

CUtensorMap make_tmap_sf(const void* base, int64_t bytes) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {128, cuuint64_t(bytes / 128)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, 16};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled (scales) failed (" + std::to_string(int(r)) + ")");
  return m;
}

CUtensorMap make_tmap_bf16(const void* base, int64_t rows, int64_t cols, int box_rows) {
  return make_tmap_2d(base, rows, cols, box_rows, false);
}

CUtensorMap make_tmap_i8(const void* base, int64_t rows, int64_t cols, int box_rows) {
  return make_tmap_2d(base, rows, cols, box_rows, true);
}

void launch_grouped_gemm(int mode, const CUtensorMap& a, const CUtensorMap& a2,
                         const CUtensorMap& b0, const CUtensorMap& b1, const GemmArgs& args,
                         int max_tiles, cudaStream_t st, const CUtensorMap* sf) {
  static std::mutex mu;
  static uint64_t configured = 0;  // bit per device: smem attribute set
  static int sms[64] = {0};
  static int pair_clusters[64] = {0};  // co-resident CTA pairs (some TPCs cannot host one)
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!((configured >> dev) & 1)) {
      cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
      cudaFuncSetAttribute(grouped_gemm_kernel<kSwiGLU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           SMEM_BYTES);
      {  // maximal shared-memory carveout for every GEMM (see configure_max_shared_carveout_kernels)
        const int c = cudaSharedmemCarveoutMaxShared;
        const void* fs[] = {
            reinterpret_cast<const void*>(grouped_gemm_kernel<kSwiGLU>),
            reinterpret_cast<const void*>(grouped_gemm_kernel<kPlain>),
            reinterpret_cast<const void*>(grouped_gemm_kernel<kInt8>),
            reinterpret_cast<const void*>(grouped_gemm_kernel<kSwiGLU8>),
            reinterpret_cast<const void*>(grouped_gemm_kernel<kPlain8>),
            reinterpret_cast<const void*>(grouped_gemm_kernel<kSwiGLU4>),
            reinterpret_cast<const void*>(grouped_gemm_kernel<kPlain4>),
            reinterpret_cast<const void*>(grouped_gemm_pair_kernel<kSwiGLU>),
            reinterpret_cast<const void*>(grouped_gemm_pair_kernel<kPlain>),
            reinterpret_cast<const void*>(grouped_gemm_pair_kernel<kSwiGLU8>),
            reinterpret_cast<const void*>(grouped_gemm_pair_kernel<kPlain8>),
            reinterpret_cast<const void*>(grouped_gemm_pair_kernel<kInt8>),
            reinterpret_cast<const void*>(grouped_gemm_pair_fp4_kernel<kSwiGLU4>),
            reinterpret_cast<const void*>(grouped_gemm_pair_fp4_kernel<kPlain4>),
            reinterpret_cast<const void*>(router_gemm_kernel)};
        for (const void* f : fs) cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, c);
      }
      cudaFuncSetAttribute(grouped_gemm_kernel<kPlain>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           SMEM_BYTES);
      cudaFuncSetAttribute(grouped_gemm_kernel<kInt8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           SMEM_BYTES);
      cudaFuncSetAttribute(grouped_gemm_kernel<kSwiGLU8>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES8);
      cudaFuncSetAttribute(grouped_gemm_kernel<kPlain8>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES8);
      cudaFuncSetAttribute(grouped_gemm_kernel<kSwiGLU4>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES4);
      cudaFuncSetAttribute(grouped_gemm_kernel<kPlain4>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES4);
      cudaFuncSetAttribute(grouped_gemm_pair_fp4_kernel<kSwiGLU4>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, P4_SMEM_BYTES);
      cudaFuncSetAttribute(grouped_gemm_pair_fp4_kernel<kPlain4>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, P4_SMEM_BYTES);
      cudaFuncSetAttribute(grouped_gemm_pair_kernel<kSwiGLU>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM_BYTES);
      cudaFuncSetAttribute(grouped_gemm_pair_kernel<kPlain>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM_BYTES);
      cudaFuncSetAttribute(grouped_gemm_pair_kernel<kSwiGLU8>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM_BYTES);
      cudaFuncSetAttribute(grouped_gemm_pair_kernel<kPlain8>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM_BYTES);
      cudaFuncSetAttribute(grouped_gemm_pair_kernel<kInt8>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM_BYTES);
      {
        cudaLaunchConfig_t lc = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.gridDim = dim3(unsigned(sms[dev] & ~1));
        lc.blockDim = dim3(256);
        lc.dynamicSmemBytes = P_SMEM_BYTES;
        lc.attrs = at;
        lc.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, grouped_gemm_pair_kernel<kSwiGLU>, &lc) != cudaSuccess)
          n = 0;
        cudaGetLastError();
        pair_clusters[dev] = n > 0 ? n : sms[dev] / 2;
        if (std::getenv("DWDP_VERBOSE"))
          std::fprintf(stderr, "dwdp: device %d: %d SMs, %d co-resident CTA pairs\n", dev, sms[dev],
                       pair_clusters[dev]);
      }
      configured |= uint64_t(1) << dev;
    }
  }
  if (max_tiles <= 0) return;
  if ((mode == kSwiGLU4 || mode == kPlain4) && args.pair && sf != nullptr) {  // NVFP4 CTA pairs
    const int cap = 2 * pair_clusters[dev];
    int g = max_tiles < cap ? max_tiles : cap;
    g = g < 2 ? 2 : (g & ~1);
    if (mode == kSwiGLU4)
      grouped_gemm_pair_fp4_kernel<kSwiGLU4><<<g, 256, P4_SMEM_BYTES, st>>>(a, b0, b1, sf[0], sf[1], sf[2], sf[3],
                                                                            args);
    else
      grouped_gemm_pair_fp4_kernel<kPlain4><<<g, 256, P4_SMEM_BYTES, st>>>(a, b0, b1, sf[0], sf[1], sf[2], sf[3],
                                                                           args);
    return;
  }
  if (mode == kSwiGLU4 || mode == kPlain4) {  // NVFP4 1-SM kernel
    const int grid = max_tiles < sms[dev] ? max_tiles : sms[dev];
    if (mode == kSwiGLU4)
      grouped_gemm_kernel<kSwiGLU4><<<grid, 256, SMEM_BYTES4, st>>>(a, a2, b0, b1, a, args);
    else if (sf != nullptr)  // sf[3]: the bf16 output map (32 x 32 boxes, SWIZZLE_64B)
      grouped_gemm_kernel<kPlain4><<<grid, 256, SMEM_BYTES4, st>>>(a, a2, b0, b1, sf[3], args);
    else
      throw std::runtime_error("launch_grouped_gemm: the NVFP4 plain GEMM needs its output map");
    return;
  }
  if (args.pair) {
    const int cap = 2 * pair_clusters[dev];
    int g = max_tiles < cap ? max_tiles : cap;
    g = g < 2 ? 2 : (g & ~1);  // whole clusters of two, all co-resident (persistent)
    if (mode == kSwiGLU)
      grouped_gemm_pair_kernel<kSwiGLU><<<g, 256, P_SMEM_BYTES, st>>>(a, a2, b0, b1, args);
    else if (mode == kPlain)
      grouped_gemm_pair_kernel<kPlain><<<g, 256, P_SMEM_BYTES, st>>>(a, a2, b0, b1, args);
    else if (mode == kSwiGLU8)
      grouped_gemm_pair_kernel<kSwiGLU8><<<g, 256, P_SMEM_BYTES, st>>>(a, a2, b0, b1, args);
    else if (mode == kPlain8)
      grouped_gemm_pair_kernel<kPlain8><<<g, 256, P_SMEM_BYTES, st>>>(a, a2, b0, b1, args);
    else
      grouped_gemm_pair_kernel<kInt8><<<g, 256, P_SMEM_BYTES, st>>>(a, a2, b0, b1, args);
    return;
  }
  const int grid = max_tiles < sms[dev] ? max_tiles : sms[dev];
  if (mode == kSwiGLU)
    grouped_gemm_kernel<kSwiGLU><<<grid, 256, SMEM_BYTES, st>>>(a, a2, b0, b1, a, args);
  else if (mode == kPlain)
    grouped_gemm_kernel<kPlain><<<grid, 256, SMEM_BYTES, st>>>(a, a2, b0, b1, a, args);
  else if (mode == kInt8)
    grouped_gemm_kernel<kInt8><<<grid, 256, SMEM_BYTES, st>>>(a, a2, b0, b1, a, args);
  else if (mode == kSwiGLU8)
    grouped_gemm_kernel<kSwiGLU8><<<grid, 256, SMEM_BYTES8, st>>>(a, a2, b0, b1, a, args);
  else
    grouped_gemm_kernel<kPlain8><<<grid, 256, SMEM_BYTES8, st>>>(a, a2, b0, b1, a, args);
}

void launch_router_gemm_pair(const CUtensorMap& planes_x, const CUtensorMap& planes_w32, const int32_t* xe,
                             const int32_t* we, float* logits, int64_t T, int E, int64_t K, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(router_gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, RP_SMEM);
  });
  if (T <= 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (T + 2 * BM - 1) / (2 * BM) * (E / R_BN);
  const int g = int(std::min<int64_t>(tiles, sms / 2)) * 2;  // whole clusters of two, persistent
  router_gemm_pair_kernel<<<unsigned(g), 256, RP_SMEM, st>>>(planes_x, planes_w32, xe, we, logits, int(T), E,
                                                             int(K));
}

void launch_router_gemm(const CUtensorMap& planes_x, const CUtensorMap& planes_w, const int32_t* xe,
                        const int32_t* we, float* logits, int64_t T, int E, int64_t K, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(router_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, R_SMEM);
  });
  if (T <= 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (T + BM - 1) / BM * (E / R_BN);
  router_gemm_kernel<<<unsigned(std::min<int64_t>(tiles, sms)), 256, R_SMEM, st>>>(planes_x, planes_w, xe, we,
                                                                                    logits, int(T), E, int(K));
}

}  // namespace dwdp
