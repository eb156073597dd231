// Ping-pong latency between the two CTAs of a cluster (B200 microbenchmark):
// mode 0: st.async (4 B, complete_tx) + remote arrive.expect_tx, receiver try_wait
// mode 1: same, receiver test_wait spin
// mode 2: remote plain arrive (no data), receiver try_wait
// mode 3: barrier.cluster arrive/wait (both CTAs), per round trip 2 barriers
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_pingpong mb_pingpong.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ bool tw(uint32_t b, uint32_t ph, int spin) {
  uint32_t ok;
  if (spin) asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(b), "r"(ph) : "memory");
  else asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(b), "r"(ph) : "memory");
  return ok;
}
__global__ void __cluster_dims__(2, 1, 1) k(int mode, int iters, unsigned long long* out) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t buf[4];
  uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const uint32_t rbar = mapa(smem_u32(&bar), rank ^ 1), rbuf = mapa(smem_u32(buf), rank ^ 1);
  long long t0 = clock64();
  uint32_t ph = 0, v = 0;
  for (int i = 0; i < iters; ++i) {
    if (mode == 3) {
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      continue;
    }
    if (threadIdx.x == 0) {
      auto send = [&]() {
        if (mode == 2) asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
        else {
          asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], 4;" ::"r"(rbar) : "memory");
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(rbuf), "r"(v + 1), "r"(rbar) : "memory");
        }
      };
      auto recv = [&]() { while (!tw(smem_u32(&bar), ph, mode == 1)) {} ph ^= 1; v = buf[0]; };
      if (rank == 0) { send(); recv(); } else { recv(); send(); }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) out[0] = (unsigned long long)(t1 - t0);
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  const char* nm[4] = {"st.async+arrive.expect_tx, try_wait", "st.async+arrive.expect_tx, test_wait spin",
                       "remote arrive only, try_wait", "2x barrier.cluster (sync) per iteration"};
  for (int mode = 0; mode < 4; ++mode) {
    const int iters = 10000;
    k<<<2, 128>>>(mode, iters, d);
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-45s round trip %.0f cycles (%s)\n", nm[mode], (double)h / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
