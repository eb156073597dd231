// dlic_stream.cuh — the P350K engine (§8(f) f1): the paper's larger network
// ("The number of neurons in the hidden layers varies between 128
// neurons to 4096 neurons"; Table I ~350K row; reading R4: 78 ->
// 256 x5 -> 256, 349,184 parameters).
//
// Its bf16 weights (696,320 B padded) do not fit one SM's shared memory
// (227 KB).  Layer 1 (5 K=16 slices, 40 KB) stays resident; layers 2-6 (80
// slices, 640 KB) are STREAMED from L2 for every network evaluation in
// chunks of 4 slices (32 KB, K=64): every slice is an 8 KB block already in
// the UMMA no-swizzle K-major core-matrix layout (element (n, k) of slice kk
// at (k/8 - 2kk)*(N/8)*128 + (n/8)*128 + (n%8)*16 + (k%8)*2), a chunk is 4
// consecutive slices, so one `cp.async.bulk` (TMA bulk copy, mbarrier
// complete_tx) moves it into a ring of S_STAGES shared-memory stages.  Two
// warps: the PRODUCER walks the chunks in consumption order and refills a
// stage as soon as its empty barrier says the MMAs that read it completed;
// the MMA ISSUER only waits for a chunk's `full` barrier, issues its MMAs and
// commits them to the stage's `empty` barrier.  (The tensor core's issue
// queue is shallow -- an issuing thread is blocked for most of an MMA's
// execution, profiles/r1_mb_mma.txt -- so any other work in the issuer idles
// the tensor core; per-slice stages cost ~800 issuer cycles per 8 KB slice, an
// mbarrier try_wait alone ~90 cycles, B300_MICROARCH.)
//
// Per row the arithmetic mirrors TcEngine (the same softmax/Q1'/search code
// consumes the same 256 logits, 8 threads x 32 columns per row): layer 1 =
// MMA over the 76 early taps + the two fresh taps' fp32 FMAs in its epilogue,
// hidden epilogues bias + ReLU + RN-to-bf16, M=64 tiles, K ascending.  The
// encoder and the decoder run this same code, so tables stay bit-identical
// (R8).  Hidden layers are N=256 and the accumulator is not double-buffered
// (TMEM: D [0,256), A [256,384), A0 [384,424), exchange [448,512)), so a layer
// is issued once every column group's epilogue of the previous layer is done.
#pragma once
#include "dlic_device.cuh"

namespace dlic {

constexpr int SH = 256;                     // P350K hidden width
constexpr uint32_t SL_BYTES = 8192;         // one K=16 slice of an N=256 layer
constexpr int SL_L0 = KPAD / 16;            // layer 1: 5 slices (76 taps + pads)
constexpr int SL_H = SH / 16;               // layers 2-6: 16 slices each
constexpr int SL_NET = 5 * SL_H;            // 80
constexpr int SL_ALL = SL_L0 + SL_NET;      // 85
constexpr uint32_t SWIMG_BYTES = SL_ALL * SL_BYTES;  // 696,320
__host__ __device__ constexpr uint32_t s_slice(int l, int kk) {
  return (l == 0 ? 0u : (uint32_t)(SL_L0 + (l - 1) * SL_H)) + (uint32_t)kk;
}
// biases in shared memory: [5][256] hidden, [256] logits, then the fresh-tap
// table: float4 per output pair n, n+1 = {wa[n], wa[n+1], wb[n], wb[n+1]}
constexpr int SB_LAST = 5 * SH;
constexpr int SB_TOTAL = 5 * SH + NOUT;     // 1536
constexpr int SB_FRESH = SB_TOTAL;
constexpr int SB_FRESH_FLOATS = 2 * SH;     // 512
constexpr uint32_t SBIAS_BYTES = (SB_TOTAL + SB_FRESH_FLOATS) * 4;  // 8,192
constexpr int CH_SL = 4;                    // slices per streamed chunk
constexpr uint32_t CH_BYTES = CH_SL * SL_BYTES;  // 32 KB
constexpr int CH_LAYER = SL_H / CH_SL;      // 4 chunks per hidden layer
constexpr int CH_NET = SL_NET / CH_SL;      // 20 chunks per network
constexpr uint32_t SL1_BYTES = SL_L0 * SL_BYTES;  // resident layer 1: 40 KB
// 12-bit alphabet (§8(f) f3, engine 3; readings R15-R17): P12 = P350K's
// layers 1-5 and a 4096-neuron output layer.  The head is computed in N=128
// column chunks (32 per pass) into a double-buffered accumulator (TMEM
// [0,128) / [128,256)), twice per network: pass 1 takes the row max and sum
// of exponentials (online), pass 2 recomputes the same logits (the same MMAs
// on the same operands: bit-identical) for p_i, the integer table and the
// search.  Each head chunk is K=256 x N=128 (16 slices of 4 KB) = two 32 KB
// stream chunks.
constexpr int H12_N = 4096;
constexpr int H12_CN = 128;                     // head columns per accumulator chunk
constexpr int H12_NCH = H12_N / H12_CN;         // 32
constexpr uint32_t H12_SL_BYTES = 4096;         // one K=16 slice of an N=128 chunk
constexpr int H12_CH_SL = 8;                    // slices per 32 KB stream chunk
constexpr int H12_STREAM = 2 * H12_NCH;         // 64 stream chunks per pass
constexpr int CH_HID12 = 4 * CH_LAYER;          // layers 2-5: 16 stream chunks
constexpr int CH_NET12 = CH_HID12 + 2 * H12_STREAM;  // 144 per network (head twice)
constexpr uint32_t SWIMG12_BYTES = SL1_BYTES + (uint32_t)(CH_HID12 + H12_STREAM) * CH_BYTES;
// biases (12-bit): [5][256] layers 1-5, the fresh table at SB_FRESH, head at SB12_HEAD
constexpr int SB12_HEAD = 2048;
constexpr uint32_t SBIAS12_BYTES = (SB12_HEAD + H12_N) * 4;  // 24 KB
constexpr float Q12_SCALE = 61376.0f;           // 2^16 - 4096 - 64 (R17)

template <bool H12>
struct StreamCfg {
  static constexpr int S = H12 ? 4 : 5;         // ring stages (160 KB / 128 KB)
  static constexpr uint32_t RING = S * CH_BYTES;
  static constexpr uint32_t BIAS = H12 ? SBIAS12_BYTES : SBIAS_BYTES;
  static constexpr uint32_t L1 = 0, RINGO = SL1_BYTES, BIASO = SL1_BYTES + RING;
  static constexpr uint32_t BARS = BIASO + BIAS;
  // full[S] empty[S] (+ 12-bit: dfull[2] dfree[2])
  static constexpr uint32_t BYTES = BARS + 2 * S * 8 + (H12 ? 32 : 0);
};
constexpr int S_STAGES = StreamCfg<false>::S;
constexpr uint32_t SRING_BYTES = StreamCfg<false>::RING;
constexpr uint32_t SENG_L1 = 0, SENG_RING = SL1_BYTES, SENG_BIAS = StreamCfg<false>::BIASO;
constexpr uint32_t SENG_BARS = StreamCfg<false>::BARS;
constexpr uint32_t SENG_BYTES = StreamCfg<false>::BYTES;
constexpr uint32_t SENG12_BYTES = StreamCfg<true>::BYTES;
constexpr uint32_t TS_D = 0, TS_A = 256, TS_A0 = 384, TS_X = 448;

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// issuer-side cycle counters (DLIC_PROF_STREAM=1, encoder): [0] waiting
// for slice data, [1] waiting for a stage's MMA before refilling it, [2]
// waiting for the previous layer's epilogues, [3] total issuer cycles, [4]
// slices consumed
__device__ unsigned long long g_sprof[8];

template <bool H12>
struct TcStreamT {
  using Cfg = StreamCfg<H12>;
  static constexpr int S = Cfg::S;
  // engine layout (shared by the streamed engines, see engine_setup)
  static constexpr int CPN = H12 ? CH_NET12 : CH_NET;  // stream chunks per network
  static constexpr uint32_t L1_BYTES = SL1_BYTES, L1_O = Cfg::L1, RING_O = Cfg::RINGO;
  static constexpr uint32_t BIAS_O = Cfg::BIASO, BIAS_BYTES = Cfg::BIAS, BARS_O = Cfg::BARS, SMEM = Cfg::BYTES;
  static constexpr bool HEAD = H12;     // dfull/dfree barriers of the 12-bit head
  static constexpr int LAST_BIAS = SB_LAST;
  uint32_t tmem;
  const float* bias;       // shared
  const float* b0;         // layer-1 biases (shared)
  uint32_t bar, bar2;      // MMA completion (bar2: interface only)
  uint32_t phase;
  uint32_t ring, full0, empty0;  // shared addresses
  uint32_t l1s;                  // resident layer-1 image (shared)
  uint32_t aready;         // layer-1 input ready: one arrival per row warp
  uint32_t dfull0, dfree0; // 12-bit head: accumulator buffer b full / released (+8b)
  uint32_t hph = 0;        // 12-bit head: dfull parities of buffers 0, 1 (bits 0, 1)
  uint32_t huse = 0;       // 12-bit head: accumulator-chunk uses so far (buffer = huse & 1; both sides)
  uint32_t* nq2s = nullptr;  // 12-bit encoder: per-tile pass-2 chunk counts ([2], tile-tagged), shared
  const uint8_t* wstream;  // the streamed weight image (global)
  uint32_t ccnt = 0, pcnt = 0;   // chunks consumed / produced (issuer warp)
  bool prof = false;
  uint32_t mode = 0;  // diagnostics: bit 1 no copies, bit 2 no MMAs (results invalid)
  unsigned long long pw[3] = {0, 0, 0};

  __device__ __forceinline__ uint32_t lane_off() const { return ((threadIdx.x >> 5) & 3u) << 21; }

  // ---- row warps
  // layer-1 input: 5 packed bf16 pairs of this thread (kpos_tap order) at A0
  __device__ __forceinline__ void put_input(const uint32_t (&a)[5]) const {
    const uint32_t base = tmem + lane_off() + TS_A0 + 10u * (uint32_t)col_grp();
    tmem_st4h<5>(base, a);
    tmem_st1h<5>(base + 4, a[4]);
  }
  // this thread's 32 biases of layer l: columns [64j + 32h, +32)
  __device__ __forceinline__ void load_bias(int l, float2 (&bq)[16]) const {
    const float4* b4 =
        reinterpret_cast<const float4*>((l == 0 ? b0 : bias + l * SH) + 64 * col_grp() + 32 * half_id());
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 b = b4[q];
      bq[2 * q] = make_float2(b.x, b.y);
      bq[2 * q + 1] = make_float2(b.z, b.w);
    }
  }
  __device__ __forceinline__ void wait_mma() {
    mbar_wait(bar, phase);
    phase ^= 1u;
    tc_fence_after();
  }
  // bias (+ fresh taps for layer 1) + ReLU + RN to bf16 -> A; columns
  // [64j + 32h, +32) -> packed A columns [32j + 16h, +16)
  template <bool L0>
  __device__ __forceinline__ void epilogue(const float2 (&b2)[16], float xa, float xb) const {
    const uint32_t lo = lane_off();
    const int j = col_grp(), h = half_id();
    uint32_t v[32];
    tmem_ld32h<32>(tmem + lo + TS_D + 64u * (uint32_t)j, v);
    tc_wait_ld();
    const float4* fw = reinterpret_cast<const float4*>(bias + SB_FRESH) + 32 * j + 16 * h;
    const f2 xa2 = f2_make(xa, xa), xb2 = f2_make(xb, xb);
    uint32_t pk[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      f2 acc = f2_bits(v[2 * q], v[2 * q + 1]);
      if constexpr (L0) {
        const float4 w = fw[q];
        acc = f2_fma(xa2, f2_make(w.x, w.y), acc);
        acc = f2_fma(xb2, f2_make(w.z, w.w), acc);
      }
      float x0, x1;
      f2_split(f2_add(acc, f2_make(b2[q].x, b2[q].y)), x0, x1);
      pk[q] = pack_bf16_relu(x0, x1);
    }
    tmem_st8h<16>(tmem + lo + TS_A + 32u * (uint32_t)j, pk);
    tmem_st8h<16>(tmem + lo + TS_A + 32u * (uint32_t)j + 8u, pk + 8);
    tc_wait_st();
  }
  // Layers 1-6 (12-bit: 1-5; the head follows in q12_row) after layer 1's
  // MMA was issued; hook(l) runs in layer l+1's MMA wait (as
  // TcEngine::run_rest_ws); pre0 is the interface's layer-1 bias hook
  // (unused: volumes run on the P100K engine).  Column group j signals on
  // named barrier 8 + j (4 warps + the issuer: 160 threads).
  template <class Hook, class Pre0>
  __device__ __forceinline__ void run_rest_ws(float xa, float xb, Hook&& hook, Pre0&&) {
    float2 bq[16];
    const uint32_t gbar = 8u + (uint32_t)col_grp();
    auto signal = [&]() {
      tc_fence_before();
      asm volatile("bar.arrive %0, 160;" ::"r"(gbar) : "memory");
    };
    load_bias(0, bq);
    wait_mma();
    epilogue<true>(bq, xa, xb);
    signal();
    constexpr int LAST = H12 ? NLAYER - 2 : NLAYER - 1;  // 12-bit: stop after layer 5's epilogue
#pragma unroll 1
    for (int l = 1; l <= LAST; ++l) {
      hook(l);
      if (l < NLAYER - 1) load_bias(l, bq);
      wait_mma();
      if (l < NLAYER - 1) {
        epilogue<false>(bq, 0.0f, 0.0f);
        signal();
      }
    }
  }
  // (encoder) the layer-1 input of this warp is in TMEM and its previous
  // logits are loaded: the issuer may run layer 1
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
    return reinterpret_cast<const float2*>(bias + SB_LAST + 64 * col_grp() + 32 * half_id())[i];
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
  // 12-bit head, row side: this thread's 16 logits of head chunk u (pass-major
  // counter; buffer u & 1, columns [32j + 16h, +16) of the chunk), the buffer
  // released once loaded
  __device__ __forceinline__ void head_ld(uint32_t (&v)[16]) {
    const uint32_t b = huse++ & 1u;
    mbar_wait(dfull0 + 8u * b, (hph >> b) & 1u);
    hph ^= 1u << b;
    tc_fence_after();
    tmem_ld16h<16>(tmem + lane_off() + TS_D + H12_CN * b + 32u * (uint32_t)col_grp(), v);
    tc_wait_ld();
    tc_fence_before();
    __syncwarp();
    if (lane_id() == 0) mbar_arrive(dfree0 + 8u * b);
  }

  // ---- issuer warp (whole converged warp)
  // global address of stream chunk c of a network (8-bit: 0..19 = layers 2-6;
  // 12-bit: 0..15 layers 2-5, then the head's 64 chunks twice)
  __device__ __forceinline__ const uint8_t* chunk_src(int c) const {
    if constexpr (H12) {
      if (c >= CH_HID12) c = CH_HID12 + (c - CH_HID12) % H12_STREAM;
    }
    return wstream + SL1_BYTES + (uint64_t)c * CH_BYTES;
  }
  // ---- producer warp (whole converged warp): chunk c of a network into the
  // next ring stage once the stage's previous chunk was consumed (its empty
  // barrier: the MMAs that read it completed)
  __device__ __forceinline__ void produce_one(int c) {
    {
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
          bulk_g2s(ring + s * CH_BYTES, chunk_src(c), CH_BYTES, full0 + 8u * s);
        }
      }
      __syncwarp();
      ++pcnt;
    }
  }
  // produce until next(c) ends the schedule
  template <class Next>
  __device__ __forceinline__ void produce_all(Next&& next) {
    int c;
    while (next(c)) produce_one(c);
  }
  // one stream chunk: wait for its data, its MMAs into D (N=256: 4 K-slices of
  // a hidden layer, K-chunk cl; 12-bit head: 8 K-slices of N=128 into buffer
  // dcol, K-half cl), release its stage when they complete
  __device__ __forceinline__ void consume(int cl, bool head = false, uint32_t dcol = 0) {
    const uint32_t s = ccnt % (uint32_t)S;
    const long long t0 = prof ? clock64() : 0;
    mbar_wait(full0 + 8u * s, (ccnt / (uint32_t)S) & 1u);
    if (prof) pw[0] += clock64() - t0;
    tc_fence_after();
    if (mode & 4u) {
      if (lane_id() == 0) mbar_arrive(empty0 + 8u * s);
      __syncwarp();
    } else if (head) {
      const uint32_t id = umma_idesc(64, H12_CN);
#pragma unroll
      for (int i = 0; i < H12_CH_SL; ++i) {
        const int kk = H12_CH_SL * cl + i;
        const uint64_t bd =
            umma_desc(ring + s * CH_BYTES + (uint32_t)i * H12_SL_BYTES, (uint32_t)H12_CN * 16u, 128u);
        umma_ts_warp(tmem + TS_D + dcol, tmem + TS_A + 8u * (uint32_t)kk, bd, id, kk > 0 ? 1u : 0u);
      }
      umma_commit_warp(empty0 + 8u * s);
    } else {
      const uint32_t id = umma_idesc(64, SH);
#pragma unroll
      for (int i = 0; i < CH_SL; ++i) {
        const int kk = CH_SL * cl + i;
        const uint64_t bd = umma_desc(ring + s * CH_BYTES + (uint32_t)i * SL_BYTES, (uint32_t)SH * 16u, 128u);
        umma_ts_warp(tmem + TS_D, tmem + TS_A + 8u * (uint32_t)kk, bd, id, kk > 0 ? 1u : 0u);
      }
      umma_commit_warp(empty0 + 8u * s);
    }
    ++ccnt;
  }
  // layer 1 from the resident image, committed to `bar`
  __device__ __forceinline__ void issue_l0() const {
    tc_fence_after();
    const uint32_t id = umma_idesc(64, SH);
#pragma unroll
    for (int kk = 0; kk < SL_L0; ++kk) {
      const uint64_t bd = umma_desc(l1s + (uint32_t)kk * SL_BYTES, (uint32_t)SH * 16u, 128u);
      umma_ts_warp(tmem + TS_D, tmem + TS_A0 + 8u * (uint32_t)kk, bd, id, kk > 0 ? 1u : 0u);
    }
    umma_commit_warp(bar);
  }
  // (encoder) n networks back to back, each once the row warps signal start_l0
  // (12-bit: with the tile's pass-2 chunk count, written before that signal)
  __device__ __forceinline__ void issue_tiles(uint64_t n) {
    const long long t00 = clock64();
    uint32_t aph = 0;
#pragma unroll 1
    for (uint64_t k = 0; k < n; ++k) {
      mbar_wait(aready, aph);
      aph ^= 1u;
      issue_l0();
      if constexpr (H12) issue_network(nq2s ? (nq2s[k & 1u] & 0xFFu) : (uint32_t)H12_NCH);
      else issue_network();
    }
    if (prof && lane_id() == 0) {
      atomicAdd(&g_sprof[0], pw[0]);
      atomicAdd(&g_sprof[1], pw[1]);
      atomicAdd(&g_sprof[2], pw[2]);
      atomicAdd(&g_sprof[3], (unsigned long long)(clock64() - t00));
      atomicAdd(&g_sprof[4], (unsigned long long)ccnt);
    }
  }
  // the layers after layer 1, each once every column group signalled its
  // previous epilogue; 12-bit: layers 2-5, then the head's two passes, each
  // accumulator chunk once the row warps released its buffer (two chunks ago)
  // 12-bit: nq2 = head chunks of the second pass (the encoder stops after the
  // chunk holding its tile's largest true symbol; the decoder runs all 32)
  __device__ __forceinline__ void issue_network(uint32_t nq2 = (uint32_t)H12_NCH) {
    constexpr int NHID = H12 ? NLAYER - 2 : NLAYER - 1;
#pragma unroll 1
    for (int l = 1; l <= NHID; ++l) {
      const long long t0 = prof ? clock64() : 0;
#pragma unroll
      for (int j = 0; j < NGRP; ++j) asm volatile("bar.sync %0, 160;" ::"r"(8 + j) : "memory");
      if (prof) pw[2] += clock64() - t0;
      tc_fence_after();
#pragma unroll 1
      for (int cl = 0; cl < CH_LAYER; ++cl) consume(cl);
      umma_commit_warp(bar);
    }
    if constexpr (H12) {
      // the last hidden layer's epilogues (A of the head, and D free)
#pragma unroll
      for (int j = 0; j < NGRP; ++j) asm volatile("bar.sync %0, 160;" ::"r"(8 + j) : "memory");
      tc_fence_after();
#pragma unroll 1
      for (uint32_t i = 0; i < (uint32_t)H12_NCH + nq2; ++i) {
        const uint32_t u = huse++, b = u & 1u;
        if (u >= 2) {  // buffer b held use u-2: wait until every row warp loaded it
          const long long t0 = prof ? clock64() : 0;
          mbar_wait(dfree0 + 8u * b, ((u >> 1) - 1u) & 1u);
          if (prof) pw[2] += clock64() - t0;
          tc_fence_after();
        }
        consume(0, true, H12_CN * b);
        consume(1, true, H12_CN * b);
        umma_commit_warp(dfull0 + 8u * b);
      }
    }
  }
};
using TcStream = TcStreamT<false>;
using TcStream12 = TcStreamT<true>;

// ---------------------------------------------------------------- 12-bit head, row side
// One pixel row = 8 threads (group j, half h); thread t = 2j + h owns the
// columns [32j + 16h, +16) of every 128-column chunk q, i.e. symbols
// 128q + 32j + 16h + i.  Reading R17 on the GPU (the same routine in the
// encoder and the decoder, R8), in packed fp32 pairs (f32x2, each lane IEEE
// RN like the scalar instruction):
//   e(x; M) = ex2.approx(fma(x, log2e, -M log2e))
//   pass 1 (online): per chunk l_i = acc_i + b_i, c = max of the 16 (exact in
//     any order), m' = max(m, c), z = z e(m; m') + s with s the pair tree
//     ((e_0 + e_1) + (e_2 + e_3)) + ((e_4 + e_5) + (e_6 + e_7)) over the 8
//     column pairs (lanes summed last: s = s.x + s.y); then halves (h = 0
//     term first) and groups (((z0 w0 + z1 w1) + z2 w2) + z3 w3, w_g = e(m_g; M))
//     combine to M, Z; r = rcp_rn(Z);
//   pass 2: p_i = e(l_i; M) r, f_i = 1 + floor(p_i 61376) (RN product, the
//     floor by a round-toward-minus-infinity add of 2^23), the row's running
//     cumulative through one exchange of the groups' chunk sums per chunk;
//     symbol 4095 takes f = 2^16 - c_4095 (the residual, R17).  Only the
//     thread whose range [c, c + sum of its 16 f) holds the key scans its
//     columns (decode: the slot; encode: the true symbol's column).
// mid() runs once the last chunk is loaded (the accumulator is free).
struct Q12Dbg {
  float* logits;   // [4096] of this row or null
  float* probs;
  uint16_t* freqs;
};
__device__ __forceinline__ float q12_e(float x, float nml) { return ex2_approx(__fmaf_rn(x, LOG2E, nml)); }
// pairs i >= 8 - DLIC_Q12_POLY of each thread's 8 column pairs take the
// FMA-pipe polynomial (f2_exp2_poly) instead of MUFU ex2 (fixed per column)
__device__ __forceinline__ f2 q12_e2(f2 l, f2 l2e, f2 nml, int i) {
  const f2 t = f2_fma(l, l2e, nml);
  if (i >= 8 - DLIC_Q12_POLY) return f2_exp2_poly(t);
  float t0, t1;
  f2_split(t, t0, t1);
  return f2_make(ex2_approx(t0), ex2_approx(t1));
}
template <bool ENC, class Mid>
__device__ __forceinline__ int q12_row(TcStream12& e, uint32_t key, bool& mine_out, uint32_t& fs_out,
                                       uint32_t& cs_out, Mid&& mid, const Q12Dbg* dbg = nullptr,
                                       uint32_t nq2 = (uint32_t)H12_NCH) {
  const int j = col_grp(), h = half_id();
  const int cb = 32 * j + 16 * h;
  const float2* hb2 = reinterpret_cast<const float2*>(e.bias + SB12_HEAD + cb);
  const f2 l2e = f2_splat(LOG2E);
  // ---- pass 1
  float m = -INFINITY, z = 0.0f;
#pragma unroll 1
  for (uint32_t q = 0; q < (uint32_t)H12_NCH; ++q) {
    uint32_t v[16];
    e.head_ld(v);
    f2 l[8];
    float a[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float2 b = hb2[(H12_CN / 2) * q + i];
      l[i] = f2_add(f2_bits(v[2 * i], v[2 * i + 1]), f2_make(b.x, b.y));
      f2_split(l[i], a[2 * i], a[2 * i + 1]);
    }
    if (dbg && dbg->logits) {
#pragma unroll
      for (int i = 0; i < 16; ++i) dbg->logits[H12_CN * q + cb + i] = a[i];
    }
    const float c = fmax3(fmax3(fmax3(a[0], a[1], a[2]), fmax3(a[3], a[4], a[5]), fmax3(a[6], a[7], a[8])),
                          fmax3(a[9], a[10], a[11]), fmax3(fmax3(a[12], a[13], a[14]), a[15], -INFINITY));
    const float mn = fmaxf(m, c);
    const float nml = __fmul_rn(-mn, LOG2E);
    const f2 nml2 = f2_splat(nml);
    f2 ex[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) ex[i] = q12_e2(l[i], l2e, nml2, i);
    const f2 s2 = f2_add(f2_add(f2_add(ex[0], ex[1]), f2_add(ex[2], ex[3])),
                         f2_add(f2_add(ex[4], ex[5]), f2_add(ex[6], ex[7])));
    float sx, sy;
    f2_split(s2, sx, sy);
    const float s = __fadd_rn(sx, sy);
    z = __fadd_rn(q > 0 ? __fmul_rn(z, q12_e(m, nml)) : 0.0f, s);
    m = mn;
  }
  // halves: the h = 0 term first on both lanes
  const float mo = __shfl_xor_sync(0xFFFFFFFFu, m, 16), zo = __shfl_xor_sync(0xFFFFFFFFu, z, 16);
  const float m_lo = h ? mo : m, m_hi = h ? m : mo, z_lo = h ? zo : z, z_hi = h ? z : zo;
  const float m2 = fmaxf(m_lo, m_hi);
  const float nm2 = __fmul_rn(-m2, LOG2E);
  const float z2 = __fadd_rn(__fmul_rn(z_lo, q12_e(m_lo, nm2)), __fmul_rn(z_hi, q12_e(m_hi, nm2)));
  e.xput(0, __float_as_uint(m2));
  e.xput(1, __float_as_uint(z2));
  e.xsync();
  uint32_t mm[4], zz[4];
  e.xget4(0, mm);
  e.xget4(1, zz);
  const float M = fmaxf(fmaxf(__uint_as_float(mm[0]), __uint_as_float(mm[1])),
                        fmaxf(__uint_as_float(mm[2]), __uint_as_float(mm[3])));
  const float nM = __fmul_rn(-M, LOG2E);
  float Z = __fmul_rn(__uint_as_float(zz[0]), q12_e(__uint_as_float(mm[0]), nM));
#pragma unroll
  for (int g = 1; g < NGRP; ++g) Z = __fadd_rn(Z, __fmul_rn(__uint_as_float(zz[g]), q12_e(__uint_as_float(mm[g]), nM)));
  const float rz = __frcp_rn(Z);
  // ---- pass 2
  const f2 nM2 = f2_splat(nM), rz2 = f2_splat(rz), sc2 = f2_splat(Q12_SCALE);
  const f2 two23 = f2_splat(8388608.0f), fbias = f2_splat(-8388607.0f);  // y - 2^23 + 1 = 1 + floor(x), exact
  float base = 0.0f;  // cumulative frequency before the current chunk (exact integers)
  bool mine = false;
  uint32_t fs = 0, cs = 0;
  int sym = 0;
  const float keyf = (float)key;
#pragma unroll 1
  for (uint32_t q = 0; q < nq2; ++q) {
    uint32_t v[16];
    e.head_ld(v);
    if (q == nq2 - 1) mid();
    f2 f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float2 b = hb2[(H12_CN / 2) * q + i];
      const f2 l = f2_add(f2_bits(v[2 * i], v[2 * i + 1]), f2_make(b.x, b.y));
      const f2 p = f2_mul(q12_e2(l, l2e, nM2, i), rz2);
      f[i] = f2_add(f2_add_rm(f2_mul(p, sc2), two23), fbias);
      if (dbg && dbg->probs) {
        float p0, p1;
        f2_split(p, p0, p1);
        dbg->probs[H12_CN * q + cb + 2 * i] = p0;
        dbg->probs[H12_CN * q + cb + 2 * i + 1] = p1;
      }
    }
    const f2 S2 = f2_add(f2_add(f2_add(f[0], f[1]), f2_add(f[2], f[3])), f2_add(f2_add(f[4], f[5]), f2_add(f[6], f[7])));
    float Sx, Sy;
    f2_split(S2, Sx, Sy);
    const float S = Sx + Sy;  // integers < 2^24: exact in any order
    const float So = __shfl_xor_sync(0xFFFFFFFFu, S, 16);
    e.xput(2 + (int)(q & 1u), __float_as_uint(S + So));  // this group's part of the chunk
    e.xsync();
    uint32_t g4[4];
    e.xget4(2 + (int)(q & 1u), g4);
    float pre = 0.0f, tot = 0.0f;
#pragma unroll
    for (int g = 0; g < NGRP; ++g) {
      const float G = __uint_as_float(g4[g]);
      pre += g < j ? G : 0.0f;
      tot += G;
    }
    const float c0 = base + pre + (h ? So : 0.0f);  // cumulative before my first column
    const bool last = q == H12_NCH - 1 && j == NGRP - 1 && h == 1;  // my column 15 is symbol 4095
    const int s0 = (int)(H12_CN * q) + cb;
    const bool scan = (dbg && dbg->freqs) ||
                      (ENC ? ((int)key >= s0 && (int)key < s0 + 16) : (keyf >= c0 && (last || keyf < c0 + S)));
    if (scan) {
      float fv[16];
#pragma unroll
      for (int i = 0; i < 8; ++i) f2_split(f[i], fv[2 * i], fv[2 * i + 1]);
      float c = c0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float fi = (last && i == 15) ? 65536.0f - c : fv[i];
        if (dbg && dbg->freqs) dbg->freqs[s0 + i] = (uint16_t)fi;
        const bool hit = ENC ? (s0 + i == (int)key) : (!mine && keyf >= c && keyf < c + fi);
        if (hit) {
          mine = true;
          sym = s0 + i;
          fs = (uint32_t)fi;
          cs = (uint32_t)c;
        }
        c += fi;
      }
    }
    base += tot;
  }
  mine_out = mine;
  fs_out = fs;
  cs_out = cs;
  return sym;
}

}  // namespace dlic
