// dlic_device.cuh — device building blocks of the B200 DLIC hot path.
//
// * PTX wrappers for tcgen05 (MMA with A in TMEM, TMEM ld/st/alloc), mbarrier
//   and thread-block-cluster (DSMEM) operations, sm_100a only.
// * The two density-estimator engines (P:96 dense network, reading R4):
//     TcEngine   bf16 operands on 5th-gen tensor cores; weights resident in
//                shared memory in the UMMA no-swizzle K-major core-matrix
//                layout; activations and accumulators live in TMEM; one
//                thread owns one TMEM lane = one pixel row of the M=128 tile.
//     Fp32Engine fp32 FFMA on CUDA cores, one thread per pixel, k ascending.
// * The deterministic softmax -> Q1 table -> CDF step (reading R5),
//   written with explicit _rn/_rd intrinsics so encoder and decoder derive
//   bit-identical tables ("the same matrices ... rounding errors ... are
//   the same").
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace dlic {

// ---------------------------------------------------------------- constants
constexpr int KIN = 78;        // causal 9x9 window (R1)
constexpr int KPAD = 80;       // layer-1 K padded to a multiple of 16 for kind::f16
constexpr int HID = 128;       // P100K hidden width (R4)
constexpr int NOUT = 256;      // 8-bit alphabet
constexpr int NLAYER = 6;      // "six dense layers"
constexpr int ROWS = 128;      // rows per CTA = TMEM lanes = threads
constexpr uint32_t RANS_L = 1u << 16;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float Q1_SCALE = 65280.0f;  // 2^16 - 256 (R5)

// bf16 weight image (bytes) per layer, core-matrix layout (see host packer)
__host__ __device__ constexpr int layer_k(int l) { return l == 0 ? KPAD : HID; }
__host__ __device__ constexpr int layer_n(int l) { return l == NLAYER - 1 ? NOUT : HID; }
__host__ __device__ constexpr uint32_t wimg_off(int l) {
  return l == 0 ? 0u : (l <= 5 ? 20480u + 32768u * (uint32_t)(l - 1) : 217088u);
}
constexpr uint32_t WIMG_BYTES = 217088;  // 20480 + 4*32768 + 65536
constexpr int BIAS_OFF_LAST = 5 * HID;   // biases: 5 x 128 hidden, then 256
constexpr int BIAS_TOTAL = 5 * HID + NOUT;

// fp32 weight blob: per layer W[K][N] then b[N]; K of layer 0 is KIN (78)
__host__ __device__ constexpr int f32_k(int l) { return l == 0 ? KIN : HID; }
__host__ __device__ constexpr uint32_t f32_off(int l) {
  uint32_t o = 0;
  for (int i = 0; i < l; ++i) o += (uint32_t)(f32_k(i) * layer_n(i) + layer_n(i));
  return o;
}

// TMEM column map (one 512-column allocation per CTA)
constexpr uint32_t TM_D = 0;     // accumulator, up to 256 columns
constexpr uint32_t TM_A = 256;   // A operand, K/2 columns (bf16 pairs), up to 64
constexpr uint32_t TM_COLS = 512;

// ------------------------------------------------------------- small PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}

// ---- tcgen05
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// whole warp; writes the allocated base column address to *slot (shared)
__device__ __forceinline__ void tmem_alloc(uint32_t slot_saddr, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot_saddr),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// UMMA shared-memory descriptor: SWIZZLE_NONE, K-major canonical layout
// ((8,n),2):((1,SBO),LBO) in 16-byte units; version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, dense.
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// D[tmem] (+)= A[tmem] * B[smem]; issued by one thread.
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

#define DLIC_R8(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), "=r"(v[i + 5]), "=r"(v[i + 6]), "=r"(v[i + 7])
#define DLIC_W8(i) "r"(v[i]), "r"(v[i + 1]), "r"(v[i + 2]), "r"(v[i + 3]), "r"(v[i + 4]), "r"(v[i + 5]), "r"(v[i + 6]), "r"(v[i + 7])

// 32 lanes (one per thread of the warp) x 32 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : DLIC_R8(0), DLIC_R8(8), DLIC_R8(16), DLIC_R8(24)
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      DLIC_W8(0), DLIC_W8(8)
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               DLIC_W8(0)
               : "memory");
}

// ---- clusters / DSMEM
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_cluster(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_u8(uint32_t caddr, uint32_t v) {
  asm volatile("st.shared::cluster.u8 [%0], %1;" ::"r"(caddr), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);  // .x = lo (bits 0-15), .y = hi
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---------------------------------------------------------------- engines
// Both engines expose:  run(...) then logits32(j, v) giving logits
// [32j, 32j+32) of this thread's row, bias included, as fp32.

struct TcEngine {
  uint32_t tmem;       // TMEM base (lane 0, column base)
  uint32_t wsmem;      // shared address of the bf16 weight image
  const float* bias;   // global [BIAS_TOTAL]
  uint32_t bar;        // shared address of the MMA-completion mbarrier
  uint32_t phase;

  __device__ __forceinline__ uint32_t lane_off() const { return ((threadIdx.x >> 5) & 3u) << 21; }

  // a[40]: this row's 80 bf16 inputs packed in pairs (element 2i in bits 0-15)
  __device__ void run(const uint32_t (&a)[40]) {
    const uint32_t lo = lane_off();
    tmem_st16(tmem + lo + TM_A, *reinterpret_cast<const uint32_t(*)[16]>(&a[0]));
    tmem_st16(tmem + lo + TM_A + 16, *reinterpret_cast<const uint32_t(*)[16]>(&a[16]));
    tmem_st8(tmem + lo + TM_A + 32, &a[32]);
    tc_wait_st();
#pragma unroll 1
    for (int l = 0; l < NLAYER; ++l) {
      tc_fence_before();
      __syncthreads();
      if (threadIdx.x == 0) {
        tc_fence_after();
        const int K = layer_k(l), N = layer_n(l);
        const uint32_t id = umma_idesc(128, N);
        const uint32_t lbo = (uint32_t)N * 16u;        // next 8-wide K core matrix
        const uint32_t kstep = 2u * (uint32_t)(N / 8) * 128u;  // one K=16 slice
        for (int kk = 0; kk < K / 16; ++kk) {
          const uint64_t bd = umma_desc(wsmem + wimg_off(l) + (uint32_t)kk * kstep, lbo, 128u);
          umma_ts(tmem + TM_D, tmem + TM_A + (uint32_t)kk * 8u, bd, id, kk > 0 ? 1u : 0u);
        }
        umma_commit(bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1u;
      tc_fence_after();
      if (l < NLAYER - 1) {
        const float* b = bias + l * HID;
#pragma unroll 1
        for (int j = 0; j < HID / 32; ++j) {
          uint32_t v[32];
          tmem_ld32(tmem + lo + TM_D + (uint32_t)j * 32u, v);
          tc_wait_ld();
          uint32_t p[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float x0 = fmaxf(__fadd_rn(__uint_as_float(v[2 * i]), __ldg(b + 32 * j + 2 * i)), 0.0f);
            const float x1 = fmaxf(__fadd_rn(__uint_as_float(v[2 * i + 1]), __ldg(b + 32 * j + 2 * i + 1)), 0.0f);
            p[i] = pack_bf16(x0, x1);
          }
          tmem_st16(tmem + lo + TM_A + (uint32_t)j * 16u, p);
        }
        tc_wait_st();
      }
    }
  }

  __device__ __forceinline__ void logits32(int j, float (&o)[32]) const {
    uint32_t v[32];
    tmem_ld32(tmem + lane_off() + TM_D + (uint32_t)j * 32u, v);
    tc_wait_ld();
    const float* b = bias + BIAS_OFF_LAST + 32 * j;
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = __fadd_rn(__uint_as_float(v[i]), __ldg(b + i));
  }
};

// CUDA-core fp32 engine.  buf0: [256][ROWS] floats, buf1: [128][ROWS] floats
// (shared, column = thread).  The input features must be written by the
// caller to buf0[k*ROWS + tid], k < 78.  Each thread reads/writes only its own
// column, so no barriers are needed.
struct Fp32Engine {
  float* buf0;
  float* buf1;
  const float* w;  // global fp32 blob (f32_off layout)

  __device__ void run() {
    const int t = threadIdx.x;
#pragma unroll 1
    for (int l = 0; l < NLAYER; ++l) {
      const float* in = (l & 1) ? buf1 : buf0;
      float* out = (l & 1) ? buf0 : buf1;
      const int K = f32_k(l), N = layer_n(l);
      const float* W = w + f32_off(l);
      const float* B = W + K * N;
#pragma unroll 1
      for (int n0 = 0; n0 < N; n0 += 32) {
        float acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.0f;
#pragma unroll 2
        for (int k = 0; k < K; ++k) {
          const float a = in[k * ROWS + t];
          const float4* wr = reinterpret_cast<const float4*>(W + k * N + n0);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 w4 = __ldg(wr + q);
            acc[4 * q + 0] = __fmaf_rn(a, w4.x, acc[4 * q + 0]);
            acc[4 * q + 1] = __fmaf_rn(a, w4.y, acc[4 * q + 1]);
            acc[4 * q + 2] = __fmaf_rn(a, w4.z, acc[4 * q + 2]);
            acc[4 * q + 3] = __fmaf_rn(a, w4.w, acc[4 * q + 3]);
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float z = __fadd_rn(acc[j], __ldg(B + n0 + j));
          if (l < NLAYER - 1) z = fmaxf(z, 0.0f);
          out[(n0 + j) * ROWS + t] = z;
        }
      }
    }
  }
  __device__ __forceinline__ void logits32(int j, float (&o)[32]) const {
    const int t = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = buf0[(32 * j + i) * ROWS + t];
  }
};

// ------------------------------------------------- softmax -> Q1 -> CDF
// Reading R5: p_i = fl(e_i * fl(1/Z)), e_i = 2^(l_i*log2e - m*log2e) (MUFU ex2,
// identical instruction in encoder and decoder), Z summed i = 0..255 in order;
// f_i = 1 + floor(fl(p_i * 65280)); R = 65536 - sum f; f_a += R at the first
// argmax a; c = exclusive prefix sum.

struct SoftmaxStats {
  float nm;   // -m * log2e
  float inv;  // 1 / Z
};

template <class Eng>
__device__ __forceinline__ SoftmaxStats softmax_stats(const Eng& e) {
  float m = -INFINITY;
#pragma unroll 1
  for (int j = 0; j < NOUT / 32; ++j) {
    float v[32];
    e.logits32(j, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) m = fmaxf(m, v[i]);
  }
  SoftmaxStats s;
  s.nm = __fmul_rn(-m, LOG2E);
  float z = 0.0f;
#pragma unroll 1
  for (int j = 0; j < NOUT / 32; ++j) {
    float v[32];
    e.logits32(j, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) z = __fadd_rn(z, ex2_approx(__fmaf_rn(v[i], LOG2E, s.nm)));
  }
  s.inv = __frcp_rn(z);
  return s;
}

__device__ __forceinline__ float q1_prob(float l, const SoftmaxStats& s) {
  return __fmul_rn(ex2_approx(__fmaf_rn(l, LOG2E, s.nm)), s.inv);
}
// 1 + floor(p * 65280) for p in [0, 1]: x + 2^23 rounded toward -inf has ulp 1.
__device__ __forceinline__ uint32_t q1_freq(float p) {
  const float x = __fmul_rn(p, Q1_SCALE);
  return __float_as_uint(__fadd_rd(x, 8388608.0f)) - 0x4B000000u + 1u;
}

// Pass over the unadjusted table: total F, first argmax a (and f_a), and for
// `sym` its f and exclusive cum.
template <class Eng>
__device__ __forceinline__ void q1_scan(const Eng& e, const SoftmaxStats& s, int sym, uint32_t& F, int& a,
                                        uint32_t& fsym, uint32_t& csym) {
  F = 0;
  a = 0;
  uint32_t best = 0;
  fsym = 0;
  csym = 0;
#pragma unroll 1
  for (int j = 0; j < NOUT / 32; ++j) {
    float v[32];
    e.logits32(j, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const uint32_t f = q1_freq(q1_prob(v[i], s));
      const int idx = 32 * j + i;
      if (idx == sym) {
        fsym = f;
        csym = F;
      }
      if (f > best) {
        best = f;
        a = idx;
      }
      F += f;
    }
  }
}

// Encoder: (f_s, c_s) of the true symbol after the residual adjustment.
template <class Eng>
__device__ __forceinline__ uint32_t q1_encode(const Eng& e, int sym) {
  const SoftmaxStats s = softmax_stats(e);
  uint32_t F, fs, cs;
  int a;
  q1_scan(e, s, sym, F, a, fs, cs);
  const uint32_t R = 65536u - F;  // may wrap if F > 65536 (guarded: unsigned add is exact mod 2^32)
  if (a == sym) fs += R;
  if (a < sym) cs += R;
  return fs | (cs << 16);
}

// Decoder: symbol s with c_s <= slot < c_s + f_s.  Returns s; fs/cs adjusted.
template <class Eng>
__device__ __forceinline__ int q1_decode(const Eng& e, uint32_t slot, uint32_t& fs_out, uint32_t& cs_out) {
  const SoftmaxStats s = softmax_stats(e);
  uint32_t F, fs, cs;
  int a;
  q1_scan(e, s, -1, F, a, fs, cs);
  const uint32_t R = 65536u - F;
  uint32_t cum = 0;
  int sym = 0;
  uint32_t f_sel = 0, c_sel = 0;
#pragma unroll 1
  for (int j = 0; j < NOUT / 32; ++j) {
    float v[32];
    e.logits32(j, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int idx = 32 * j + i;
      uint32_t f = q1_freq(q1_prob(v[i], s));
      if (idx == a) f += R;
      if (slot - cum < f) {  // cum <= slot < cum + f (unsigned: slot >= cum)
        sym = idx;
        f_sel = f;
        c_sel = cum;
      }
      cum += f;
    }
  }
  fs_out = f_sel;
  cs_out = c_sel;
  return sym;
}

// Debug export of p (fp32) and the final integer table.
template <class Eng>
__device__ void q1_export(const Eng& e, float* probs, uint16_t* freqs) {
  const SoftmaxStats s = softmax_stats(e);
  uint32_t F, fs, cs;
  int a;
  q1_scan(e, s, -1, F, a, fs, cs);
  const uint32_t R = 65536u - F;
#pragma unroll 1
  for (int j = 0; j < NOUT / 32; ++j) {
    float v[32];
    e.logits32(j, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int idx = 32 * j + i;
      const float p = q1_prob(v[i], s);
      uint32_t f = q1_freq(p);
      if (idx == a) f += R;
      if (probs) probs[idx] = p;
      if (freqs) freqs[idx] = (uint16_t)f;
    }
  }
}

}  // namespace dlic
