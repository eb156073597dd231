// Microbenchmark (not part of the library): latency of one dependent
// "layer" of tcgen05 MMAs -- issue K/16 MMAs (A in TMEM, B in shared memory),
// commit to an mbarrier, all threads wait -- repeated back to back, as in the
// decoder's per-front network.  Variants: M in {64,128}, N in {128,256},
// with or without a __syncthreads + TMEM round trip (a minimal epilogue).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_mma scripts/mb_mma.cu && ./mb_mma
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}

#define R4(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3])
template <int OFF>
__device__ __forceinline__ void ld16h(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16], %17;"
      : R4(0), R4(4), R4(8), R4(12)
      : "r"(taddr), "n"(OFF));
}
template <int OFF>
__device__ __forceinline__ void st8h(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.16x32bx2.x8.b32 [%0], %1, {%2,%3,%4,%5,%6,%7,%8,%9};" ::"r"(taddr), "n"(OFF),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

template <int M, int N, int EPI>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < N * 128 * 2 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3C003C00u ^ i;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  uint32_t phase = 0;
  unsigned long long t0 = 0, issue_cyc = 0;
  for (int it = 0; it < iters + 8; ++it) {
    if (it == 8) t0 = clock64();
    if (EPI) {
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
    }
    if (threadIdx.x == 256) {
      const unsigned long long ti0 = clock64();
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t id = umma_idesc(M, N);
      const uint32_t kstep = 2u * (N / 8) * 128u;
      uint32_t at = tmem + 256;
      if (EPI == 7) {  // B in the 128-byte-swizzled K-major layout: atoms of 8 rows x 64 K
        const uint64_t sw = (uint64_t)2 << 61;  // SWIZZLE_128B
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t addr = smem_u32(sm) + (uint32_t)(kk / 4) * N * 128u + (uint32_t)(kk % 4) * 32u;
          const uint64_t bd = umma_desc(addr, 16u, 1024u) | sw;
          umma_ts(tmem, at, bd, id, kk > 0);
          at += 8;
        }
      } else {
        uint64_t bd = umma_desc(smem_u32(sm), N * 16u, 128u);
        for (int kk = 0; kk < 8; ++kk) {
          umma_ts(tmem, at, bd, id, kk > 0);
          bd += kstep >> 4;
          at += 8;
        }
      }
      if (EPI == 6) {  // a second batch of 8 (as the split last layer)
        uint64_t bd2 = umma_desc(smem_u32(sm), N * 16u, 128u);
        uint32_t at2 = tmem + 256;
        for (int kk = 0; kk < 8; ++kk) {
          umma_ts(tmem + 128, at2, bd2, id, kk > 0);
          bd2 += kstep >> 4;
          at2 += 8;
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      if (it >= 8) issue_cyc += clock64() - ti0;
    }
    float2 bpre[8];
    if (EPI == 3) {  // bias loaded before the MMA wait
      const int j = threadIdx.x >> 7, h = (threadIdx.x >> 4) & 1;
      const float2* b2 = reinterpret_cast<const float2*>(sm) + 16 * j + 8 * h;
#pragma unroll
      for (int q = 0; q < 8; ++q) bpre[q] = b2[q];
    }
    mbar_wait(smem_u32(&bar), phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (EPI >= 3) {  // 3: preloaded bias, 4: no bias, 5: load + store only
      const uint32_t lo = ((threadIdx.x >> 5) & 3u) << 21;
      const int j = threadIdx.x >> 7;
      uint32_t v[16];
      ld16h<16>(tmem + lo + 32u * j, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      uint32_t pk[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (EPI == 5) {
          pk[q] = v[2 * q] ^ v[2 * q + 1];
        } else {
          float x0 = __uint_as_float(v[2 * q]), x1 = __uint_as_float(v[2 * q + 1]);
          if (EPI == 3) {
            x0 += bpre[q].x;
            x1 += bpre[q].y;
          }
          uint32_t r;
          asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x1), "f"(x0));
          pk[q] = r;
        }
      }
      st8h<8>(tmem + lo + 256 + 16u * j, pk);
      asm volatile("tcgen05.wait::st.sync.aligned;");
    } else if (EPI == 2) {  // the decoder's hidden-layer epilogue: 16 columns per thread
      const uint32_t lo = ((threadIdx.x >> 5) & 3u) << 21;
      const int j = threadIdx.x >> 7, h = (threadIdx.x >> 4) & 1;
      uint32_t v[16];
      ld16h<16>(tmem + lo + 32u * j, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      const float2* b2 = reinterpret_cast<const float2*>(sm) + 16 * j + 8 * h;
      uint32_t pk[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float2 b = b2[q];
        const float x0 = __uint_as_float(v[2 * q]) + b.x, x1 = __uint_as_float(v[2 * q + 1]) + b.y;
        uint32_t r;
        asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x1), "f"(x0));
        pk[q] = r;
      }
      st8h<8>(tmem + lo + 256 + 16u * j, pk);
      asm volatile("tcgen05.wait::st.sync.aligned;");
    } else if (EPI) {  // minimal epilogue: one TMEM load + store round trip per thread
      uint32_t v;
      const uint32_t lo = ((threadIdx.x >> 5) & 3u) << 21;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + lo));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      v += 1;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lo + 256 + (threadIdx.x >> 7)), "r"(v));
      asm volatile("tcgen05.wait::st.sync.aligned;");
    }
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (threadIdx.x == 256) out[1] = issue_cyc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int M, int N, int EPI>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int sm = N * 128 * 2;
  cudaFuncSetAttribute(k<M, N, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  const int iters = 2000;
  k<M, N, EPI><<<1, 512, sm>>>(iters, d);
  unsigned long long h[2] = {0, 0};
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-34s %s  %7.1f cycles per layer (8 x K=16; floor %d); issuing thread busy %.1f\n", name,
         cudaGetErrorString(e), (double)h[0] / iters, 8 * (M > 128 ? M : 128) * N / 256, (double)h[1] / iters);
  cudaFree(d);
}

int main() {
  run<64, 128, 0>("M=64  N=128 chain");
  run<128, 128, 0>("M=128 N=128 chain");
  run<64, 256, 0>("M=64  N=256 chain");
  run<64, 128, 1>("M=64  N=128 + sync + TMEM rt");
  run<64, 256, 1>("M=64  N=256 + sync + TMEM rt");
  run<64, 128, 2>("M=64  N=128 + sync + real epilogue");
  run<64, 128, 3>("  .. bias preloaded before wait");
  run<64, 128, 4>("  .. no bias");
  run<64, 128, 5>("  .. ld16 + st8 only");
  run<64, 128, 6>("M=64 2 x 8 x N=128 chain");
  run<64, 128, 7>("M=64  N=128 chain, B SWIZZLE_128B");
  run<64, 256, 7>("M=64  N=256 chain, B SWIZZLE_128B");
  return 0;
}
