// dlic_x3.cuh — the fp32 path on the tensor cores (engine 4): P100K with
// every product in three bf16 limbs ("bf16x3").
//
// encoder and decoder agree "as long as the precision of the floating
// point arithmetic is the same"; north_star holds the fp32 path to 1e-4
// relative logits against the fp64 oracle.  A plain bf16 MMA is ~4e-3 off;
// splitting each fp32 operand x into hi = bf16_rn(x) and lo = bf16_rn(x - hi)
// (16 significant bits together) and summing three bf16 MMAs per K-slice,
//     a w ~= a_hi w_hi + a_hi w_lo + a_lo w_hi      (a_lo w_lo, ~2^-16, dropped)
// with fp32 accumulation in TMEM, is within ~2e-5.  Layer-1 inputs v/256 are
// exact in bf16 (a_lo = 0: two MMAs per slice); hidden activations are split
// in the epilogue into two packed TMEM operands A_hi, A_lo.
//
// Weights: the hi and lo images (434 KB) exceed one SM's shared memory, so
// layer 1 (5 slices x 2 limbs, 40 KB) stays resident and layers 2-6 stream
// through the same ring/producer machinery as the P350K engine
// (dlic_stream.cuh): 12 chunks of 32 KB per network -- a hidden layer (N=128,
// 4 KB per slice and limb) is 2 chunks of 4 K-slices x {hi, lo}, the logits
// layer (N=256, 8 KB per slice and limb) 4 chunks of 2 K-slices x {hi, lo}.
// TMEM: D [0,256) (hidden layers use [0,128)), A_hi [256,320), A_lo [320,384),
// A0 [384,424), exchange [448,512).  Per row the thread split is TcEngine's
// (8 threads: hidden columns [32j + 16h, +16), logits [64j + 32h, +32)), the
// softmax/Q1'/search code is shared with the bf16 path, the fresh taps and
// biases are fp32 (exact weights), and the encoder runs the same routine
// (R8).  (The FFMA engine Fp32Engine remains for 3D volumes.)
#pragma once
#include "dlic_stream.cuh"

namespace dlic {

constexpr uint32_t X3_SL = 4096;                    // K=16 slice, N=128, one limb
constexpr uint32_t X3_SL_LAST = 8192;               // K=16 slice, N=256, one limb
constexpr int X3_CPN = 4 * 2 + 4;                   // 12 stream chunks per network
constexpr uint32_t X3_L1_BYTES = SL_L0 * 2 * X3_SL;  // 40 KB resident
constexpr uint32_t X3_WIMG_BYTES = X3_L1_BYTES + X3_CPN * CH_BYTES;
// biases: [5][128] layers 1-5, [256] logits, fresh table (fp32 float4 per
// hidden pair {wa[n], wa[n+1], wb[n], wb[n+1]})
constexpr int X3_B_LAST = 5 * HID;       // 640
constexpr int X3_B_FRESH = X3_B_LAST + NOUT;  // 896
constexpr uint32_t X3_BIAS_BYTES = (X3_B_FRESH + 2 * HID) * 4;  // 4,608
constexpr uint32_t X3_AHI = 256, X3_ALO = 320;

struct TcX3 {
  static constexpr int S = 5;
  static constexpr int CPN = X3_CPN;
  static constexpr uint32_t L1_BYTES = X3_L1_BYTES, L1_O = 0, RING_O = X3_L1_BYTES;
  static constexpr uint32_t BIAS_O = RING_O + S * CH_BYTES, BIAS_BYTES = X3_BIAS_BYTES;
  static constexpr uint32_t BARS_O = BIAS_O + BIAS_BYTES, SMEM = BARS_O + 2 * S * 8;
  static constexpr bool HEAD = false;
  static constexpr int LAST_BIAS = X3_B_LAST;

  uint32_t tmem;
  const float* bias;       // shared
  const float* b0;         // layer-1 biases (shared, or the image's metadata-folded bias)
  uint32_t bar, bar2;
  uint32_t phase;
  uint32_t ring, full0, empty0, l1s;
  uint32_t aready;
  uint32_t dfull0, dfree0;  // (unused: no streamed head)
  const uint8_t* wstream;
  uint32_t ccnt = 0, pcnt = 0;
  bool prof = false;
  uint32_t mode = 0;
  unsigned long long pw[3] = {0, 0, 0};

  __device__ __forceinline__ uint32_t lane_off() const { return ((threadIdx.x >> 5) & 3u) << 21; }
  // hidden accumulators alternate between D columns [128,256) (layers 1, 3,
  // 5) and [0,128) (2, 4): layer l+1's first K-chunk is issued once column
  // groups 0-1 signalled, while groups 2-3 still read layer l's accumulator
  static __device__ __forceinline__ uint32_t dcol(int l) { return (l & 1) ? 0u : 128u; }

  // ---- row warps
  __device__ __forceinline__ void put_input(const uint32_t (&a)[5]) const {
    const uint32_t base = tmem + lane_off() + TS_A0 + 10u * (uint32_t)col_grp();
    tmem_st4h<5>(base, a);
    tmem_st1h<5>(base + 4, a[4]);
  }
  __device__ __forceinline__ void wait_mma() {
    mbar_wait(bar, phase);
    phase ^= 1u;
    tc_fence_after();
  }
  // this thread's 16 biases of hidden layer l: columns [32j + 16h, +16)
  __device__ __forceinline__ void load_bias(int l, float2 (&bq)[8]) const {
    const float4* b4 =
        reinterpret_cast<const float4*>((l == 0 ? b0 : bias + l * HID) + 32 * col_grp() + 16 * half_id());
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 b = b4[q];
      bq[2 * q] = make_float2(b.x, b.y);
      bq[2 * q + 1] = make_float2(b.z, b.w);
    }
  }
  // bias (+ the fresh taps in fp32 for layer 1) + ReLU, split into bf16 hi and
  // lo limbs -> A_hi, A_lo packed columns [16j + 8h, +8)
  template <bool L0>
  __device__ __forceinline__ void epilogue(const float2 (&b2)[8], float xa, float xb, uint32_t dc) const {
    const uint32_t lo = lane_off();
    const int j = col_grp(), h = half_id();
    uint32_t v[16];
    tmem_ld16h<16>(tmem + lo + TS_D + dc + 32u * (uint32_t)j, v);
    tc_wait_ld();
    const float4* fw = reinterpret_cast<const float4*>(bias + X3_B_FRESH) + 16 * j + 8 * h;
    uint32_t phi[8], plo[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float x0 = __uint_as_float(v[2 * q]), x1 = __uint_as_float(v[2 * q + 1]);
      if constexpr (L0) {
        const float4 w = fw[q];
        x0 = __fmaf_rn(xb, w.z, __fmaf_rn(xa, w.x, x0));
        x1 = __fmaf_rn(xb, w.w, __fmaf_rn(xa, w.y, x1));
      }
      x0 = fmaxf(__fadd_rn(x0, b2[q].x), 0.0f);
      x1 = fmaxf(__fadd_rn(x1, b2[q].y), 0.0f);
      const __nv_bfloat162 hb = __floats2bfloat162_rn(x0, x1);
      const float h0 = __low2float(hb), h1 = __high2float(hb);
      phi[q] = *reinterpret_cast<const uint32_t*>(&hb);
      plo[q] = pack_bf16(__fsub_rn(x0, h0), __fsub_rn(x1, h1));  // x - hi is exact in fp32
    }
    tmem_st8h<8>(tmem + lo + X3_AHI + 16u * (uint32_t)j, phi);
    tmem_st8h<8>(tmem + lo + X3_ALO + 16u * (uint32_t)j, plo);
    tc_wait_st();
  }
  template <class Hook, class Pre0>
  __device__ __forceinline__ void run_rest_ws(float xa, float xb, Hook&& hook, Pre0&&) {
    float2 bq[8];
    const uint32_t gbar = 8u + (uint32_t)col_grp();
    auto signal = [&]() {
      tc_fence_before();
      asm volatile("bar.arrive %0, 160;" ::"r"(gbar) : "memory");
    };
    load_bias(0, bq);
    wait_mma();
    epilogue<true>(bq, xa, xb, dcol(0));
    signal();
#pragma unroll 1
    for (int l = 1; l < NLAYER; ++l) {
      hook(l);
      if (l < NLAYER - 1) load_bias(l, bq);
      if (l == NLAYER - 1 && col_grp() >= 2) {  // logits [128,256): the second half (bar2; == bar in the encoder)
        mbar_wait(bar2, phase);
        phase ^= 1u;
        tc_fence_after();
      } else {
        wait_mma();
      }
      if (l < NLAYER - 1) {
        epilogue<false>(bq, 0.0f, 0.0f, dcol(l));
        signal();
      }
    }
  }
  __device__ __forceinline__ void start_l0() const {
    tc_wait_st();
    tc_fence_before();
    __syncwarp();
    if (lane_id() == 0) mbar_arrive(aready);
  }
  template <class Hook>
  __device__ __forceinline__ void run_rest(float xa, float xb, Hook&& hook, Prof* = nullptr) {
    run_rest_ws(xa, xb, hook, [](auto&) {});
  }
  // softmax interface (as TcEngine)
  __device__ __forceinline__ void ld32(uint32_t (&v)[32]) const {
    tmem_ld32h<32>(tmem + lane_off() + TS_D + 64u * (uint32_t)col_grp(), v);
    tc_wait_ld();
  }
  __device__ __forceinline__ float2 bias_pair(int i) const {
    return reinterpret_cast<const float2*>(bias + X3_B_LAST + 64 * col_grp() + 32 * half_id())[i];
  }
  __device__ __forceinline__ void xput(int slot, uint32_t v) const {
    tmem_st1h<TM_XUP>(tmem + lane_off() + TS_X + 4u * (uint32_t)slot + (uint32_t)col_grp(), v);
  }
  __device__ __forceinline__ void xsync() const {
    tc_wait_st();
    tc_fence_before();
    quad_sync();
    tc_fence_after();
  }
  __device__ __forceinline__ void xget8(int slot, uint32_t (&v)[8]) const {
    tmem_ld8h<TM_XUP>(tmem + lane_off() + TS_X + 4u * (uint32_t)slot, v);
    tc_wait_ld();
  }
  __device__ __forceinline__ void xget4(int slot, uint32_t (&v)[4]) const {
    tmem_ld4h<TM_XUP>(tmem + lane_off() + TS_X + 4u * (uint32_t)slot, v);
    tc_wait_ld();
  }

  // ---- producer warp
  __device__ __forceinline__ void produce_one(int c) {
    const uint32_t s = pcnt % (uint32_t)S;
    if (pcnt >= (uint32_t)S) {
      const long long t0 = prof ? clock64() : 0;
      mbar_wait(empty0 + 8u * s, ((pcnt / (uint32_t)S) - 1u) & 1u);
      if (prof) pw[1] += clock64() - t0;
    }
    if (lane_id() == 0) {
      if (mode & 2u) {
        mbar_arrive(full0 + 8u * s);
      } else {
        mbar_expect_tx(full0 + 8u * s, CH_BYTES);
        bulk_g2s(ring + s * CH_BYTES, wstream + X3_L1_BYTES + (uint64_t)c * CH_BYTES, CH_BYTES, full0 + 8u * s);
      }
    }
    __syncwarp();
    ++pcnt;
  }
  template <class Next>
  __device__ __forceinline__ void produce_all(Next&& next) {
    int c;
    while (next(c)) produce_one(c);
  }

  // ---- MMA issuer warp
  // three MMAs of one K-slice: hi.hi (accumulate unless the layer's first), hi.lo, lo.hi
  // (ni: instruction N, columns [n0, n0 + ni) of a layer of width n, into D
  // columns [dc, dc + ni))
  __device__ __forceinline__ void x3_slice(uint32_t whi, uint32_t wlo, uint32_t n, int kk, bool first, uint32_t ni,
                                           uint32_t n0, uint32_t dc) const {
    const uint32_t id = umma_idesc(64, (int)(ni ? ni : n));
    const uint32_t bo = (n0 / 8u) * 128u;
    const uint64_t bh = umma_desc(whi + bo, n * 16u, 128u), bl = umma_desc(wlo + bo, n * 16u, 128u);
    const uint32_t ah = tmem + X3_AHI + 8u * (uint32_t)kk, al = tmem + X3_ALO + 8u * (uint32_t)kk;
    umma_ts_warp(tmem + TS_D + dc, ah, bh, id, first ? 0u : 1u);
    umma_ts_warp(tmem + TS_D + dc, ah, bl, id, 1u);
    umma_ts_warp(tmem + TS_D + dc, al, bh, id, 1u);
  }
  // one stream chunk of layer l (1..5): hidden layers 4 K-slices, the
  // logits layer 2, each {hi, lo}
  __device__ __forceinline__ void consume(int l, int cl) {
    const uint32_t s = ccnt % (uint32_t)S;
    const long long t0 = prof ? clock64() : 0;
    mbar_wait(full0 + 8u * s, (ccnt / (uint32_t)S) & 1u);
    if (prof) pw[0] += clock64() - t0;
    tc_fence_after();
    const uint32_t base = ring + s * CH_BYTES;
    if (mode & 4u) {
      if (lane_id() == 0) mbar_arrive(empty0 + 8u * s);
      __syncwarp();
    } else if (l < NLAYER - 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        x3_slice(base + (2u * i) * X3_SL, base + (2u * i + 1u) * X3_SL, (uint32_t)HID, 4 * cl + i, cl == 0 && i == 0, 0u,
                 0u, dcol(l));
      umma_commit_warp(empty0 + 8u * s);
    } else {
#pragma unroll
      for (int i = 0; i < 2; ++i)
        x3_slice(base + (2u * i) * X3_SL_LAST, base + (2u * i + 1u) * X3_SL_LAST, (uint32_t)NOUT, 2 * cl + i,
                 cl == 0 && i == 0, 0u, 0u, 0u);
      umma_commit_warp(empty0 + 8u * s);
    }
    ++ccnt;
  }
  // layer 1 from the resident image: two MMAs per slice (exact inputs)
  __device__ __forceinline__ void issue_l0() const {
    tc_fence_after();
    const uint32_t id = umma_idesc(64, HID);
#pragma unroll
    for (int kk = 0; kk < SL_L0; ++kk) {
      const uint32_t a = tmem + TS_A0 + 8u * (uint32_t)kk;
      const uint64_t bh = umma_desc(l1s + (2u * kk) * X3_SL, (uint32_t)HID * 16u, 128u);
      const uint64_t bl = umma_desc(l1s + (2u * kk + 1u) * X3_SL, (uint32_t)HID * 16u, 128u);
      umma_ts_warp(tmem + TS_D + dcol(0), a, bh, id, kk > 0 ? 1u : 0u);
      umma_ts_warp(tmem + TS_D + dcol(0), a, bl, id, 1u);
    }
    umma_commit_warp(bar);
    if (bar2 != bar) umma_commit_warp(bar2);
  }
  // Decoder (bar2 != bar): every layer completes both barriers, except the
  // logits layer, issued as two N=128 halves -- [0,128) for all four chunks
  // (their stages held), committed to bar (column groups 0-1 start their
  // softmax), then [128,256) from the same stages, committed to bar2.  Per
  // element the K order is the encoder's single N=256 layer's.
  __device__ __forceinline__ void issue_network() {
#pragma unroll 1
    for (int l = 1; l < NLAYER; ++l) {
      const long long t0 = prof ? clock64() : 0;
      if (l < NLAYER - 1) {
        // hidden layer: K-chunk 0 (column groups 0-1's activations) once they
        // signalled, chunk 1 once groups 2-3 did (double-buffered D: the
        // previous layer's accumulator is still read meanwhile)
#pragma unroll 1
        for (int cl = 0; cl < 2; ++cl) {
          asm volatile("bar.sync %0, 160;" ::"r"(8 + 2 * cl) : "memory");
          asm volatile("bar.sync %0, 160;" ::"r"(9 + 2 * cl) : "memory");
          if (prof) pw[2] += clock64() - t0;
          tc_fence_after();
          consume(l, cl);
        }
        umma_commit_warp(bar);
        if (bar2 != bar) umma_commit_warp(bar2);
        continue;
      }
      if (bar2 != bar && !(mode & 4u)) {
        // decoder logits as two N=128 halves: [0,128) (the accumulator the
        // last hidden layer did not use) K-chunk cl once column group cl
        // signalled, the chunks' stages held, committed to bar (groups 0-1
        // start their softmax); then [128,256) from the same stages after
        // every group, committed to bar2.  Per element the encoder's K order.
#pragma unroll 1
        for (int cl = 0; cl < 4; ++cl) {
          asm volatile("bar.sync %0, 160;" ::"r"(8 + cl) : "memory");
          tc_fence_after();
          const uint32_t c = ccnt + (uint32_t)cl, s = c % (uint32_t)S;
          mbar_wait(full0 + 8u * s, (c / (uint32_t)S) & 1u);
          tc_fence_after();
          const uint32_t base = ring + s * CH_BYTES;
#pragma unroll
          for (int i = 0; i < 2; ++i)
            x3_slice(base + (2u * i) * X3_SL_LAST, base + (2u * i + 1u) * X3_SL_LAST, (uint32_t)NOUT, 2 * cl + i,
                     cl == 0 && i == 0, 128u, 0u, 0u);
        }
        if (prof) pw[2] += clock64() - t0;
        umma_commit_warp(bar);
#pragma unroll 1
        for (int cl = 0; cl < 4; ++cl) {
          const uint32_t s = (ccnt + (uint32_t)cl) % (uint32_t)S;
          const uint32_t base = ring + s * CH_BYTES;
#pragma unroll
          for (int i = 0; i < 2; ++i)
            x3_slice(base + (2u * i) * X3_SL_LAST, base + (2u * i + 1u) * X3_SL_LAST, (uint32_t)NOUT, 2 * cl + i,
                     cl == 0 && i == 0, 128u, 128u, 128u);
          umma_commit_warp(empty0 + 8u * s);
        }
        ccnt += 4;
        umma_commit_warp(bar2);
        continue;
      }
      // (encoder) the logits over [0,256) once every group's last epilogue is done
#pragma unroll
      for (int j = 0; j < NGRP; ++j) asm volatile("bar.sync %0, 160;" ::"r"(8 + j) : "memory");
      if (prof) pw[2] += clock64() - t0;
      tc_fence_after();
#pragma unroll 1
      for (int cl = 0; cl < 4; ++cl) consume(l, cl);
      umma_commit_warp(bar);
      if (bar2 != bar) umma_commit_warp(bar2);
    }
  }
  __device__ __forceinline__ void issue_tiles(uint64_t n) {
    const long long t00 = clock64();
    uint32_t aph = 0;
#pragma unroll 1
    for (uint64_t k = 0; k < n; ++k) {
      mbar_wait(aready, aph);
      aph ^= 1u;
      issue_l0();
      issue_network();
    }
    if (prof && lane_id() == 0) {
      atomicAdd(&g_sprof[0], pw[0]);
      atomicAdd(&g_sprof[2], pw[2]);
      atomicAdd(&g_sprof[3], (unsigned long long)(clock64() - t00));
      atomicAdd(&g_sprof[4], (unsigned long long)ccnt);
    }
  }
};

}  // namespace dlic
