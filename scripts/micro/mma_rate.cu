// Microbenchmark: tcgen05.mma kind::f16 (SS mode, bf16 -> fp32) issue rate vs N
// on one CTA per SM. Prints cycles per MMA instruction for N = 64, 128, 256,
// with and without a concurrent TMEM-reading warp group.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_rate scripts/micro/mma_rate.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\nselp.u32 %0, 1, 0, e;\n}" : "=r"(p));
  return p != 0;
}

__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
  } while (!ok);
}

template <int N, int TLD>
__global__ void __launch_bounds__(256, 1) mma_rate(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[2];
  __shared__ uint32_t holder;
  __shared__ int done;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    done = 0;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = holder;
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
  if (warp == 1) {
    const uint64_t a = desc(su32(base)), b = desc(su32(base + 16384));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                       "l"(a + 2 * (k & 3)), "l"(b + 2 * (k & 3)), "r"(IDESC), "r"(k));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bars[it & 1]))
                     : "memory");
      }
      __syncwarp();
      if (it >= 1) wait_bar(&bars[(it - 1) & 1], uint32_t(((it - 1) >> 1) & 1));
    }
    wait_bar(&bars[(iters - 1) & 1], uint32_t(((iters - 1) >> 1) & 1));
    long long t1 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) *cyc = (unsigned long long)(t1 - t0);
    if (threadIdx.x == 32) atomicExch(&done, 1);
  } else if (warp >= 4 && TLD) {  // TMEM readers on columns 256.. (not the accumulator)
    const uint32_t lb = uint32_t((warp & 3) * 32) << 16;
    float acc = 0;
    while (!*(volatile int*)&done) {
      uint32_t r[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
            "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
            "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(tmem + lb + 256u));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
    }
    if (acc == 12345.f) *cyc = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int TLD>
void run(unsigned long long* d) {
  const int iters = 2000;
  cudaFuncSetAttribute(mma_rate<N, TLD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  mma_rate<N, TLD><<<148, 256, 64 * 1024>>>(iters, d);
  mma_rate<N, TLD><<<148, 256, 64 * 1024>>>(iters, d);
  unsigned long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double per = double(c) / (iters * 16.0);
  printf("{\"N\": %d, \"tmem_readers\": %d, \"cycles_per_mma\": %.2f, \"ideal\": %.1f, \"err\": \"%s\"}\n", N, TLD, per,
         128.0 * N / 256.0, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  run<64, 0>(d); run<128, 0>(d); run<256, 0>(d);
  run<64, 1>(d); run<128, 1>(d); run<256, 1>(d);
  return 0;
}
