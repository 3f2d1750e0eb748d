// MLA prefill attention block on Blackwell (sm_100a): the attention step of
// the DWDP prefetch window, MoE(l) + Attention(l+1), whose
// cost the reference models as attention_entries (src/modelspec.cpp:38-55,
// phase AttnOps at src/simcore.cpp:666-674).
//
// DeepSeek-V3 MLA (no weight absorption, the prefill form):
//   q   = rms(x Wq_a^T) Wq_b^T                 [T][H][128 nope | 64 rope]
//   kva = x Wkv_a^T                            [T][512 ckv | 64 k_rope]
//   kv  = rms(ckv) Wkv_b^T                     [T][H][128 k_nope | 128 v]
//   q_rope, k_rope <- RoPE(position in sequence)
//   o   = softmax(q k^T / sqrt(192), causal per sequence) v   [T][H][128]
//   y   = o Wo^T
// The five projections run on the tcgen05 grouped-GEMM kernel (one dense
// group); RMSNorm, RoPE and the K / V^T assembly are small glue kernels; the
// attention core is mla_attn_kernel below.
//
// Two kernels: mla_attn_kernel (default, described here) and
// mla_attn2_kernel (DWDP_ATTN_PAIR=1, further below), two query tiles per
// CTA on one K/V stream.
// mla_attn_kernel: one CTA per (128-query tile of a sequence, head),
// 384 threads, warp-specialised:
//   warp 0      TMA producer: Q tile once (3 boxes of 128 x 64), then per
//               64-key tile K (3 boxes) and V^T (one [128 dv][64 keys] box)
//               into separate 4-stage rings
//   warp 1      MMA issuer (whole warp runs the schedule, one elected lane
//               issues): S_j = Q K_j^T (tcgen05 kind::f16, M128 N64 K192, A =
//               Q in TMEM) into S buffer j % 4, and O += P_j V_j (M128 N128
//               K64, A = P in TMEM) into ONE TMEM accumulator; S runs two
//               tiles ahead of PV
//   warp 2      TMEM allocator (512 columns: Q 96 | S/P x4 of 64 | O 128)
//   warps 4-11  softmax + epilogue, one query row per thread pair (TMEM lane),
//               each warp of a pair on 32 of the 64 S columns (warps 4-7
//               first copy the Q rows from smem into TMEM): tcgen05.ld S,
//               causal mask (diagonal tiles only), row max agreed through
//               smem + a named barrier, online softmax in exp2 form against a
//               LAZY reference max m_ref, P as bf16 pairs written over the S
//               columns it came from (tcgen05.st). O never leaves TMEM until
//               the epilogue: P = exp2(s - m_ref) is only rescaled when a
//               row's max grows by more than 2^8 over m_ref (then the warp
//               waits for the previous PV, multiplies its O rows in TMEM by
//               alpha = exp2(m_ref - m_new) with tcgen05.ld/st, and moves
//               m_ref) -- P <= 2^8 keeps the bf16 relative precision and the
//               fp32 accumulator has the range. Epilogue: O / l as bf16.
// A K stage is released when its S MMA completes, a V stage and the S/P
// buffer when the PV MMA of that tile completes.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <stdexcept>

#include "attn_sm100.hpp"

namespace dwdp {
namespace {

constexpr int AQ = 128, AK = 64, DQK = 192, DV = 128, KVS = 4;
constexpr int Q_BOX = AQ * 64 * 2;   // 16 KB: 128 rows x 64 columns
constexpr int K_BOX = AK * 64 * 2;   // 8 KB
constexpr int Q_BYTES = 3 * Q_BOX;   // 48 KB
constexpr int K_BYTES = 3 * K_BOX;   // 24 KB
constexpr int V_BYTES = DV * AK * 2; // 16 KB
constexpr int NG = 2;  // softmax column groups: NG warps per TMEM lane quarter, AK / NG S columns each
constexpr int XCH_BYTES = 2 * NG * AQ * 4;  // row-max exchange between the column groups, per tile parity
constexpr int ATT_THREADS = 128 + NG * 128;
constexpr int ATT_SMEM = 1024 + Q_BYTES + KVS * (K_BYTES + V_BYTES) + XCH_BYTES + 256;
// kind::f16 instruction descriptors, K-major A and B, bf16 in, fp32 out
constexpr uint32_t IDESC_S = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(AK >> 3) << 17) |
                             (uint32_t(AQ >> 4) << 24);
constexpr uint32_t IDESC_O = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(DV >> 3) << 17) |
                             (uint32_t(AQ >> 4) << 24);
// TMEM (512 columns): Q as the A operand of QK^T (192 bf16 per lane = 96
// columns), four S buffers that the softmax overwrites in place with P (the A
// operand of PV, 64 bf16 = 32 columns), one O accumulator.
constexpr int SB = 4;
constexpr uint32_t TM_Q = 0, TM_S = 128, TM_O = 384;
constexpr float RESCALE_LOG2 = 8.0f;      // lazy rescale threshold (log2 units)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// A operand in TMEM (lane = row, 2 bf16 per column), B from shared memory
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
// K-major SWIZZLE_128B operand descriptor (8-row atoms 1024 B apart, sm_100 version 1)
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
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
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
template <int N>
__device__ __forceinline__ void ldn(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 32) ld32(taddr, r); else ld16(taddr, r);
}
template <int N>
__device__ __forceinline__ void stn(uint32_t taddr, const uint32_t (&r)[N]) {
  if constexpr (N == 16) st16(taddr, r); else st8(taddr, r);
}
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void sts(float* p, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(su32(p)), "f"(v) : "memory");
}
__device__ __forceinline__ float lds(const float* p) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(su32(p)) : "memory");
  return v;
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\nselp.u32 %0, 1, 0, e;\n}" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t pack2(float a, float b) {  // one F2FP.BF16.F32.PACK_AB
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

__global__ void __launch_bounds__(ATT_THREADS, 1)
    mla_attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const AttnTile* __restrict__ tiles,
                    uint16_t* __restrict__ out, int H, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sQ = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sQ + Q_BYTES;
  uint8_t* sV = sK + KVS * K_BYTES;
  float* xch = reinterpret_cast<float*>(sV + KVS * V_BYTES);  // [tile parity][half][row]
  uint64_t* q_full = reinterpret_cast<uint64_t*>(sV + KVS * V_BYTES + XCH_BYTES);
  uint64_t* q_tmem = q_full + 1;  // Q copied into TMEM
  uint64_t* k_full = q_tmem + 1;  // K and V rings: a K stage is free once S_j is done, a V stage after PV_j
  uint64_t* k_empty = k_full + KVS;
  uint64_t* v_full = k_empty + KVS;
  uint64_t* v_empty = v_full + KVS;
  uint64_t* s_full = v_empty + KVS;  // S_j in buffer j % SB
  uint64_t* p_full = s_full + SB;    // P_j written over it
  uint64_t* s_free = p_full + SB;    // PV_j done: buffer reusable, and every earlier PV is done
  uint64_t* o_full = s_free + SB;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_full + 1);

  const AttnTile tile = tiles[blockIdx.x];
  const int head = blockIdx.y;
  const int q_hi = min(tile.q0 + AQ, tile.len);  // queries [q0, q_hi) attend keys [0, q_hi)
  const int nt = (q_hi + AK - 1) / AK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    bar_init(q_full, 1);
    bar_init(q_tmem, 4);
    for (int s = 0; s < KVS; ++s) {
      bar_init(&k_full[s], 1);
      bar_init(&k_empty[s], 1);
      bar_init(&v_full[s], 1);
      bar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < SB; ++b) {
      bar_init(&s_full[b], 1);
      bar_init(&p_full[b], 4 * NG);
      bar_init(&s_free[b], 1);
    }
    bar_init(o_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      bar_expect(q_full, Q_BYTES);
      for (int a = 0; a < 3; ++a) tma3(sQ + a * Q_BOX, &tmQ, q_full, a * 64, head, tile.start + tile.q0);
      for (int j = 0; j < nt; ++j) {
        const int s = j % KVS;
        bar_wait(&k_empty[s], ((j / KVS) & 1) ^ 1);
        bar_expect(&k_full[s], K_BYTES);
        for (int a = 0; a < 3; ++a)
          tma3(sK + s * K_BYTES + a * K_BOX, &tmK, &k_full[s], a * 64, head, tile.start + j * AK);
        bar_wait(&v_empty[s], ((j / KVS) & 1) ^ 1);
        bar_expect(&v_full[s], V_BYTES);
        tma3(sV + s * V_BYTES, &tmV, &v_full[s], tile.vstart + j * AK, 0, head);
      }
    }
  } else if (warp == 1) {  // ------------------------------------------ MMA issuer
    // The whole warp runs the schedule (waits, descriptor arithmetic) so the
    // operands are warp-uniform and live in uniform registers; one elected
    // lane issues. Both A operands come from TMEM (Q, and P written over S):
    // an SS-mode M128 N64 K16 MMA is bound by its shared-memory operand reads
    // (57 cycles measured vs 32 of math, scripts/micro/mma_rate.cu), a
    // TS-mode one reads only the 2 KB K slice.
    bar_wait(q_tmem, 0);
    fence_after();
    auto qk = [&](int j) {  // S_j = Q K_j^T into S buffer j % SB
      const int b = j % SB, s = j % KVS;
      bar_wait(&s_free[b], ((j / SB) & 1) ^ 1);  // PV_{j-SB} has consumed P_{j-SB}
      bar_wait(&k_full[s], (j / KVS) & 1);
      fence_after();
      const uint64_t kd = desc(su32(sK + s * K_BYTES));
      if (elect_one()) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_ts(tmem + TM_S + uint32_t(b) * AK, tmem + TM_Q + uint32_t(a * 32 + k * 8),
                   kd + uint64_t(a * (K_BOX >> 4)) + 2 * k, IDESC_S, (a | k) != 0);
        commit(&s_full[b]);
        commit(&k_empty[s]);
      }
      __syncwarp();
    };
    auto pv = [&](int i) {  // O += P_i V_i
      const int b = i % SB, s = i % KVS;
      bar_wait(&p_full[b], (i / SB) & 1);
      bar_wait(&v_full[s], (i / KVS) & 1);
      fence_after();
      const uint64_t vd = desc(su32(sV + s * V_BYTES));
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; ++k)  // 16 keys = 8 TMEM columns of P per MMA
          mma_ts(tmem + TM_O, tmem + TM_S + uint32_t(b) * AK + uint32_t(k * 8), vd + 2 * k, IDESC_O,
                 (i | k) != 0);
        commit(&v_empty[s]);
        commit(&s_free[b]);
      }
      __syncwarp();
    };
    // S runs two tiles ahead of PV: S_{j+2} is issued right after PV_{j-1},
    // so the tensor pipe has QK^T work while softmax(j) is still running
    qk(0);
    if (nt > 1) qk(1);
    for (int j = 0; j < nt; ++j) {
      if (j + 2 < nt) qk(j + 2);
      pv(j);
    }
    if (elect_one()) commit(o_full);
    __syncwarp();
  } else if (warp >= 4) {  // -------------------------------------------- softmax + epilogue
    // warps 4 + 4g + q (g < NG) take S columns [g AK/NG, (g+1) AK/NG) of
    // the TMEM lanes 32q ..: NG warps per SM sub-partition hide each other's
    // latency. The group agrees on the row max through xch + a named barrier
    // per lane quarter; each warp owns DV/NG columns of O.
    const int q = warp & 3, hf = (warp - 4) >> 2, row = q * 32 + lane;
    const int qi = tile.q0 + row;  // query position in its sequence
    const uint32_t lb = uint32_t(q * 32) << 16;
    constexpr int HC = AK / NG, HO = DV / NG;
    if (hf == 0) {  // Q row (SWIZZLE_128B smem, 16-byte chunk c of row r at c ^ (r % 8)) into TMEM
      bar_wait(q_full, 0);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        uint32_t v[32];
        const uint8_t* src = sQ + a * Q_BOX + (row >> 3) * 1024 + (row & 7) * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 u = *reinterpret_cast<const uint4*>(src + ((c ^ (row & 7)) << 4));
          v[4 * c] = u.x, v[4 * c + 1] = u.y, v[4 * c + 2] = u.z, v[4 * c + 3] = u.w;
        }
        st32(tmem + lb + TM_Q + uint32_t(a * 32), v);
      }
      st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(q_tmem);
    }
    float m_ref = -INFINITY, l = 0.0f;  // l = sum of exp2(s - m_ref) over this half's keys
    for (int j = 0; j < nt; ++j) {
      const int b = j & 1, sb = j % SB;
      const uint32_t sbuf = tmem + lb + TM_S + uint32_t(sb) * AK;
      bar_wait(&s_full[sb], (j / SB) & 1);
      fence_after();
      uint32_t r[HC];
      ldn<HC>(sbuf + uint32_t(hf * HC), r);
      ld_wait();
      float sv[HC];
      const int k0 = j * AK + hf * HC;
      float m0 = -INFINITY, m1 = -INFINITY;
      if (k0 + HC - 1 <= tile.q0) {  // all keys at or below every row's diagonal: no mask
#pragma unroll
        for (int c = 0; c < HC; c += 2) {
          sv[c] = __uint_as_float(r[c]);
          sv[c + 1] = __uint_as_float(r[c + 1]);
          m0 = fmaxf(m0, sv[c]);
          m1 = fmaxf(m1, sv[c + 1]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < HC; c += 2) {  // causal (keys past the sequence are > qi)
          sv[c] = (k0 + c <= qi) ? __uint_as_float(r[c]) : -INFINITY;
          sv[c + 1] = (k0 + c + 1 <= qi) ? __uint_as_float(r[c + 1]) : -INFINITY;
          m0 = fmaxf(m0, sv[c]);
          m1 = fmaxf(m1, sv[c + 1]);
        }
      }
      float mx = fmaxf(m0, m1);
      // the exchange barrier also orders every group's S loads before any
      // group writes P over columns [0, 32) of the buffer
      sts(xch + (b * NG + hf) * AQ + row, mx);
      asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(32 * NG) : "memory");
#pragma unroll
      for (int g = 1; g < NG; ++g) mx = fmaxf(mx, lds(xch + (b * NG + (hf + g) % NG) * AQ + row));
      mx *= scale_log2;
      const bool grow = mx > m_ref + RESCALE_LOG2;  // identical in every group
      if (j == 0) {
        m_ref = mx;  // key 0 is visible to every row: finite
      } else if (__any_sync(0xffffffffu, grow)) {
        // rescale this warp's half of its O rows in TMEM once PV_{j-1} (and
        // so every earlier PV) has completed; PV_j waits for p_full below
        const float alpha = grow ? ex2(m_ref - mx) : 1.0f;
        if (grow) {
          l *= alpha;
          m_ref = mx;
        }
        bar_wait(&s_free[(j - 1) % SB], ((j - 1) / SB) & 1);
        fence_after();
#pragma unroll
        for (int ch = 0; ch < HO / 32; ++ch) {
          uint32_t o[32];
          ld32(tmem + lb + TM_O + uint32_t(hf * HO + ch * 32), o);
          ld_wait();
#pragma unroll
          for (int x = 0; x < 32; ++x) o[x] = __float_as_uint(__uint_as_float(o[x]) * alpha);
          st32(tmem + lb + TM_O + uint32_t(hf * HO + ch * 32), o);
        }
      }
      const float nm = -m_ref;
      float s0 = 0.0f, s1 = 0.0f;
      uint32_t pk[HC / 2];
#pragma unroll
      for (int c = 0; c < HC; c += 2) {
        const float e0 = ex2(fmaf(sv[c], scale_log2, nm)), e1 = ex2(fmaf(sv[c + 1], scale_log2, nm));
        s0 += e0;
        s1 += e1;
        pk[c / 2] = pack2(e0, e1);
      }
      l += s0 + s1;
      // this group's keys of P (bf16 pairs) over TMEM columns [hf HC/2, (hf+1) HC/2) of the buffer
      stn<HC / 2>(sbuf + uint32_t(hf * (HC / 2)), pk);
      st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(&p_full[sb]);
    }
    // row sum over the groups (the exchange slot of parity nt & 1 is free:
    // every group passed the barrier of tile nt - 1, which used the other)
    sts(xch + ((nt & 1) * NG + hf) * AQ + row, l);
    asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(32 * NG) : "memory");
#pragma unroll
    for (int g = 1; g < NG; ++g) l += lds(xch + ((nt & 1) * NG + (hf + g) % NG) * AQ + row);
    bar_wait(o_full, 0);
    fence_after();
    const float inv = 1.0f / l;
    uint4* dst = reinterpret_cast<uint4*>(out + (int64_t(tile.start + qi) * H + head) * DV + hf * HO);
#pragma unroll
    for (int ch = 0; ch < HO / 32; ++ch) {
      uint32_t o[32];
      ld32(tmem + lb + TM_O + uint32_t(hf * HO + ch * 32), o);
      ld_wait();
      if (qi < tile.len) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float* f = reinterpret_cast<const float*>(&o[8 * c]);
          dst[ch * 4 + c] = make_uint4(pack2(f[0] * inv, f[1] * inv), pack2(f[2] * inv, f[3] * inv),
                                       pack2(f[4] * inv, f[5] * inv), pack2(f[6] * inv, f[7] * inv));
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------- two query tiles per CTA
// mla_attn2_kernel: one CTA per (256-query pair of tiles X = A, B of a
// sequence, head). The tensor pipe alternates between the tiles, so one
// tile's softmax overlaps the other tile's MMAs; K and V tiles are loaded
// once for both. QK^T runs in SS mode (both Q tiles stay in shared memory:
// the TMEM holds two S/P double buffers and two O accumulators), PV in TS
// mode with P written over S. One softmax warp per TMEM lane quarter and
// tile (64 columns per thread row), no cross-warp exchange.
constexpr int A2_KVS = 3;
constexpr int A2_THREADS = 384;
constexpr int A2_SMEM = 1024 + 2 * Q_BYTES + A2_KVS * (K_BYTES + V_BYTES) + 256;
// TMEM: tile X's S/P buffers at 256X (+ 64 b), its O accumulator at 256X + 128
__device__ __forceinline__ uint32_t a2_tm_s(int x) { return uint32_t(x) * 256u; }
__device__ __forceinline__ uint32_t a2_tm_o(int x) { return uint32_t(x) * 256u + 128u; }

__global__ void __launch_bounds__(A2_THREADS, 1)
    mla_attn2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const AttnTile* __restrict__ tiles,
                     uint16_t* __restrict__ out, int H, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sQ = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sQ + 2 * Q_BYTES;
  uint8_t* sV = sK + A2_KVS * K_BYTES;
  uint64_t* q_full = reinterpret_cast<uint64_t*>(sV + A2_KVS * V_BYTES);
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + A2_KVS;
  uint64_t* v_full = k_empty + A2_KVS;
  uint64_t* v_empty = v_full + A2_KVS;
  uint64_t* s_full = v_empty + A2_KVS;  // [tile][2]
  uint64_t* p_full = s_full + 4;        // [tile][2]
  uint64_t* s_free = p_full + 4;        // [tile][2]: PV done, buffer reusable
  uint64_t* o_full = s_free + 4;        // [tile]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_full + 2);

  const AttnTile tile = tiles[blockIdx.x];
  const int head = blockIdx.y;
  const int ntile = tile.q0 + AQ < tile.len ? 2 : 1;  // tile B exists
  int nt[2];
  for (int x = 0; x < 2; ++x) nt[x] = (min(tile.q0 + x * AQ + AQ, tile.len) + AK - 1) / AK;
  const int ntk = nt[ntile - 1];  // KV tiles to stream (B's range covers A's)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    bar_init(q_full, 1);
    for (int s = 0; s < A2_KVS; ++s) {
      bar_init(&k_full[s], 1);
      bar_init(&k_empty[s], 1);
      bar_init(&v_full[s], 1);
      bar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 4; ++b) {
      bar_init(&s_full[b], 1);
      bar_init(&p_full[b], 4);
      bar_init(&s_free[b], 1);
    }
    bar_init(&o_full[0], 1);
    bar_init(&o_full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      bar_expect(q_full, uint32_t(ntile * Q_BYTES));
      for (int x = 0; x < ntile; ++x)
        for (int a = 0; a < 3; ++a)
          tma3(sQ + x * Q_BYTES + a * Q_BOX, &tmQ, q_full, a * 64, head, tile.start + tile.q0 + x * AQ);
      for (int j = 0; j < ntk; ++j) {
        const int s = j % A2_KVS;
        bar_wait(&k_empty[s], ((j / A2_KVS) & 1) ^ 1);
        bar_expect(&k_full[s], K_BYTES);
        for (int a = 0; a < 3; ++a)
          tma3(sK + s * K_BYTES + a * K_BOX, &tmK, &k_full[s], a * 64, head, tile.start + j * AK);
        bar_wait(&v_empty[s], ((j / A2_KVS) & 1) ^ 1);
        bar_expect(&v_full[s], V_BYTES);
        tma3(sV + s * V_BYTES, &tmV, &v_full[s], tile.vstart + j * AK, 0, head);
      }
    }
  } else if (warp == 1) {  // ------------------------------------------ MMA issuer (warp-uniform)
    bar_wait(q_full, 0);
    fence_after();
    auto qk = [&](int x, int j) {  // S_X(j) = Q_X K_j^T into S_X buffer j % 2
      const int b = j & 1;
      bar_wait(&s_free[x * 2 + b], ((j >> 1) & 1) ^ 1);  // PV_X(j - 2) has consumed P_X(j - 2)
      fence_after();
      const uint64_t qd = desc(su32(sQ + x * Q_BYTES));
      const uint64_t kd = desc(su32(sK + (j % A2_KVS) * K_BYTES));
      if (elect_one()) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_ss(tmem + a2_tm_s(x) + uint32_t(b) * AK, qd + uint64_t(a * (Q_BOX >> 4)) + 2 * k,
                   kd + uint64_t(a * (K_BOX >> 4)) + 2 * k, IDESC_S, (a | k) != 0);
        commit(&s_full[x * 2 + b]);
      }
      __syncwarp();
    };
    auto pv = [&](int x, int i) {  // O_X += P_X(i) V_i
      const int b = i & 1;
      bar_wait(&p_full[x * 2 + b], (i >> 1) & 1);
      fence_after();
      const uint64_t vd = desc(su32(sV + (i % A2_KVS) * V_BYTES));
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; ++k)  // 16 keys = 8 TMEM columns of P per MMA
          mma_ts(tmem + a2_tm_o(x), tmem + a2_tm_s(x) + uint32_t(b) * AK + uint32_t(k * 8), vd + 2 * k, IDESC_O,
                 (i | k) != 0);
        commit(&s_free[x * 2 + b]);
      }
      __syncwarp();
    };
    auto pvs = [&](int i) {  // PV of KV tile i for every tile that uses it, then free its V stage
      const int s = i % A2_KVS;
      bar_wait(&v_full[s], (i / A2_KVS) & 1);
      for (int x = 0; x < ntile; ++x)
        if (i < nt[x]) pv(x, i);
      if (elect_one()) commit(&v_empty[s]);
      __syncwarp();
    };
    for (int j = 0; j < ntk; ++j) {
      const int s = j % A2_KVS;
      bar_wait(&k_full[s], (j / A2_KVS) & 1);
      for (int x = 0; x < ntile; ++x)
        if (j < nt[x]) qk(x, j);
      if (elect_one()) commit(&k_empty[s]);
      __syncwarp();
      if (j >= 1) pvs(j - 1);
    }
    pvs(ntk - 1);
    if (elect_one()) {
      commit(&o_full[0]);
      commit(&o_full[1]);
    }
    __syncwarp();
  } else if (warp >= 4) {  // ----------------------------------------- softmax + epilogue
    const int x = (warp - 4) >> 2, q = warp & 3, row = q * 32 + lane;
    const int q0 = tile.q0 + x * AQ;
    if (x < ntile) {  // no early return: every warp reaches the final barrier
      const int qi = q0 + row;  // query position in its sequence
      const uint32_t lb = uint32_t(q * 32) << 16;
      const uint32_t o_acc = tmem + lb + a2_tm_o(x);
      float m_ref = -INFINITY, l = 0.0f;
      for (int j = 0; j < nt[x]; ++j) {
        const int b = j & 1;
        const uint32_t sbuf = tmem + lb + a2_tm_s(x) + uint32_t(b) * AK;
        bar_wait(&s_full[x * 2 + b], (j >> 1) & 1);
        fence_after();
        uint32_t r0[32], r1[32];
        ld32(sbuf, r0);
        ld32(sbuf + 32, r1);
        ld_wait();
        float sv[AK];
        const int k0 = j * AK;
        float m0 = -INFINITY, m1 = -INFINITY;
        if (k0 + AK - 1 <= q0) {  // all keys at or below every row's diagonal: no mask
#pragma unroll
          for (int c = 0; c < AK; c += 2) {
            sv[c] = __uint_as_float(c < 32 ? r0[c] : r1[c - 32]);
            sv[c + 1] = __uint_as_float(c + 1 < 32 ? r0[c + 1] : r1[c - 31]);
            m0 = fmaxf(m0, sv[c]);
            m1 = fmaxf(m1, sv[c + 1]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < AK; c += 2) {  // causal (keys past the sequence are > qi)
            sv[c] = (k0 + c <= qi) ? __uint_as_float(c < 32 ? r0[c] : r1[c - 32]) : -INFINITY;
            sv[c + 1] = (k0 + c + 1 <= qi) ? __uint_as_float(c + 1 < 32 ? r0[c + 1] : r1[c - 31]) : -INFINITY;
            m0 = fmaxf(m0, sv[c]);
            m1 = fmaxf(m1, sv[c + 1]);
          }
        }
        const float mx = fmaxf(m0, m1) * scale_log2;
        const bool grow = mx > m_ref + RESCALE_LOG2;
        if (j == 0) {
          m_ref = mx;  // key 0 is visible to every row: finite
        } else if (__any_sync(0xffffffffu, grow)) {
          const float alpha = grow ? ex2(m_ref - mx) : 1.0f;
          if (grow) {
            l *= alpha;
            m_ref = mx;
          }
          bar_wait(&s_free[x * 2 + ((j - 1) & 1)], ((j - 1) >> 1) & 1);  // PV_X(j - 1) done
          fence_after();
#pragma unroll
          for (int ch = 0; ch < DV / 32; ++ch) {
            uint32_t o[32];
            ld32(o_acc + uint32_t(ch * 32), o);
            ld_wait();
#pragma unroll
            for (int y = 0; y < 32; ++y) o[y] = __float_as_uint(__uint_as_float(o[y]) * alpha);
            st32(o_acc + uint32_t(ch * 32), o);
          }
        }
        const float nm = -m_ref;
        float s0 = 0.0f, s1 = 0.0f;
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < AK; c += 2) {
          const float e0 = ex2(fmaf(sv[c], scale_log2, nm)), e1 = ex2(fmaf(sv[c + 1], scale_log2, nm));
          s0 += e0;
          s1 += e1;
          pk[c / 2] = pack2(e0, e1);
        }
        l += s0 + s1;
        st32(sbuf, pk);  // P (bf16 pairs) over the first 32 S columns
        st_wait();
        fence_before();
        __syncwarp();
        if (lane == 0) bar_arrive(&p_full[x * 2 + b]);
      }
      bar_wait(&o_full[x], 0);
      fence_after();
      const float inv = 1.0f / l;
      uint4* dst = reinterpret_cast<uint4*>(out + (int64_t(tile.start + qi) * H + head) * DV);
#pragma unroll
      for (int ch = 0; ch < DV / 32; ++ch) {
        uint32_t o[32];
        ld32(o_acc + uint32_t(ch * 32), o);
        ld_wait();
        if (qi < tile.len) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float* f = reinterpret_cast<const float*>(&o[8 * c]);
            dst[ch * 4 + c] = make_uint4(pack2(f[0] * inv, f[1] * inv), pack2(f[2] * inv, f[3] * inv),
                                         pack2(f[4] * inv, f[5] * inv), pack2(f[6] * inv, f[7] * inv));
          }
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------- glue
// RMSNorm without weight (x * rsqrt(mean(x^2) + eps)), one warp per row, fp32 math.
__global__ void rmsnorm_kernel(const uint16_t* __restrict__ in, int64_t ld_in, uint16_t* __restrict__ out,
                               int64_t ld_out, int64_t rows, int D, float eps) {
  const int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const uint16_t* x = in + r * ld_in;
  float ss = 0.0f;
  for (int i = lane; i < D; i += 32) {
    const float v = __uint_as_float(uint32_t(x[i]) << 16);
    ss += v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = rsqrtf(ss / float(D) + eps);
  uint16_t* y = out + r * ld_out;
  for (int i = lane; i < D; i += 32)
    y[i] = __bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(uint32_t(x[i]) << 16) * inv));
}

// RoPE on the 64 rope dims of every q head, in place (interleaved pairs
// (2i, 2i+1), angle pos * theta^(-2i/64)); one thread per (token, head, pair).
__global__ void q_rope_kernel(uint16_t* __restrict__ q, const int32_t* __restrict__ pos, int64_t T, int H,
                              float log2_theta) {
  const int64_t n = T * H * 32;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / (H * 32);
    const int p = int(i % 32);
    uint16_t* v = q + (i / 32) * DQK + 128 + 2 * p;
    const float ang = float(pos[t]) * exp2f(-log2_theta * float(2 * p) / 64.0f);
    float sn, cs;
    sincosf(ang, &sn, &cs);
    const float x1 = __uint_as_float(uint32_t(v[0]) << 16), x2 = __uint_as_float(uint32_t(v[1]) << 16);
    v[0] = __bfloat16_as_ushort(__float2bfloat16_rn(x1 * cs - x2 * sn));
    v[1] = __bfloat16_as_ushort(__float2bfloat16_rn(x1 * sn + x2 * cs));
  }
}

// K [T][H][192] = (k_nope of kv | RoPE(k_rope) shared by the heads) and
// V^T [H][128][ldv] (token t at column vcol[t]) from kv [T][H][256]
// (k_nope | v). One CTA per (64-token block, head); V goes through shared
// memory so the reads of kv and the writes of V^T are row-contiguous runs.
__global__ void __launch_bounds__(256) kv_assemble_kernel(const uint16_t* __restrict__ kv,
                                                          const uint16_t* __restrict__ kva, int64_t ld_kva,
                                                          int kv_lora, const int32_t* __restrict__ pos,
                                                          const int32_t* __restrict__ vcol, int64_t T, int H,
                                                          float log2_theta, uint16_t* __restrict__ K,
                                                          uint16_t* __restrict__ Vt, int64_t ldv) {
  __shared__ uint16_t tv[64][DV + 2];
  __shared__ int32_t col[64];
  const int64_t t0 = int64_t(blockIdx.x) * 64;
  const int h = blockIdx.y;
  if (threadIdx.x < 64) col[threadIdx.x] = t0 + threadIdx.x < T ? vcol[t0 + threadIdx.x] : -1;
  for (int i = threadIdx.x; i < 64 * (DQK / 2); i += blockDim.x) {  // K: pairs of elements
    const int tl = i / (DQK / 2), c = 2 * (i % (DQK / 2));
    const int64_t t = t0 + tl;
    if (t >= T) continue;
    uint16_t* dk = K + (t * H + h) * DQK + c;
    if (c < 128) {
      const uint16_t* s = kv + (t * H + h) * 256 + c;
      dk[0] = s[0];
      dk[1] = s[1];
    } else {
      const int p = (c - 128) / 2;
      const uint16_t* s = kva + t * ld_kva + kv_lora + 2 * p;
      const float ang = float(pos[t]) * exp2f(-log2_theta * float(2 * p) / 64.0f);
      float sn, cs;
      sincosf(ang, &sn, &cs);
      const float x1 = __uint_as_float(uint32_t(s[0]) << 16), x2 = __uint_as_float(uint32_t(s[1]) << 16);
      dk[0] = __bfloat16_as_ushort(__float2bfloat16_rn(x1 * cs - x2 * sn));
      dk[1] = __bfloat16_as_ushort(__float2bfloat16_rn(x1 * sn + x2 * cs));
    }
  }
  for (int i = threadIdx.x; i < 64 * DV; i += blockDim.x) {
    const int tl = i / DV, d = i % DV;
    const int64_t t = t0 + tl;
    tv[tl][d] = t < T ? kv[(t * H + h) * 256 + 128 + d] : uint16_t(0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < DV * 64; i += blockDim.x) {
    const int d = i / 64, tl = i % 64;
    if (col[tl] >= 0) Vt[(int64_t(h) * DV + d) * ldv + col[tl]] = tv[tl][d];
  }
}

}  // namespace

// 0 (default): one query tile per CTA (mla_attn_kernel, TS-mode QK^T);
// DWDP_ATTN_PAIR=1: two query tiles per CTA (mla_attn2_kernel)
static int attn_variant() {
  static const int v = [] {
    const char* e = std::getenv("DWDP_ATTN_PAIR");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

int mla_attention_query_step() {
  return attn_variant() ? 2 * AQ : AQ;
}

void launch_mla_attention(const uint16_t* q, const uint16_t* k, const uint16_t* vt, int64_t T, int64_t ldv,
                          int H, const AttnTile* tiles, int ntiles, float softmax_scale, uint16_t* out,
                          cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(mla_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ATT_SMEM);
    cudaFuncSetAttribute(mla_attn_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(mla_attn2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, A2_SMEM);

    cudaFuncSetAttribute(mla_attn2_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
  });
  if (ntiles <= 0 || T <= 0) return;
  const int64_t dq[3] = {DQK, H, T}, sq[2] = {DQK * 2, int64_t(H) * DQK * 2};
  const int bq[3] = {64, 1, AQ}, bk[3] = {64, 1, AK};
  const CUtensorMap tq = make_tmap_3d_bf16(q, dq, sq, bq);
  const CUtensorMap tk = make_tmap_3d_bf16(k, dq, sq, bk);
  const int64_t dv[3] = {ldv, DV, H}, sv[2] = {ldv * 2, int64_t(DV) * ldv * 2};
  const int bv[3] = {AK, DV, 1};
  const CUtensorMap tv = make_tmap_3d_bf16(vt, dv, sv, bv);
  if (attn_variant() == 1)
    mla_attn2_kernel<<<dim3(unsigned(ntiles), unsigned(H)), A2_THREADS, A2_SMEM, st>>>(
        tq, tk, tv, tiles, out, H, softmax_scale * 1.4426950408889634f);
  else
    mla_attn_kernel<<<dim3(unsigned(ntiles), unsigned(H)), ATT_THREADS, ATT_SMEM, st>>>(
        tq, tk, tv, tiles, out, H, softmax_scale * 1.4426950408889634f);
}

void launch_rmsnorm(const uint16_t* in, int64_t ld_in, uint16_t* out, int64_t ld_out, int64_t rows, int D,
                    float eps, cudaStream_t st) {
  if (rows > 0) rmsnorm_kernel<<<unsigned((rows + 7) / 8), 256, 0, st>>>(in, ld_in, out, ld_out, rows, D, eps);
}

void launch_q_rope(uint16_t* q, const int32_t* pos, int64_t T, int H, float theta, cudaStream_t st) {
  const int64_t n = T * H * 32;
  if (n > 0)
    q_rope_kernel<<<unsigned(std::min<int64_t>((n + 255) / 256, 148 * 16)), 256, 0, st>>>(q, pos, T, H,
                                                                                         std::log2(theta));
}

void launch_kv_assemble(const uint16_t* kv, const uint16_t* kva, int64_t ld_kva, int kv_lora, const int32_t* pos,
                        const int32_t* vcol, int64_t T, int H, float theta, uint16_t* K, uint16_t* Vt,
                        int64_t ldv, cudaStream_t st) {
  if (T > 0)
    kv_assemble_kernel<<<dim3(unsigned((T + 63) / 64), unsigned(H)), 256, 0, st>>>(
        kv, kva, ld_kva, kv_lora, pos, vcol, T, H, std::log2(theta), K, Vt, ldv);
}

}  // namespace dwdp
