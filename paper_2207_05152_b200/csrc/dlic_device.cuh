// dlic_device.cuh — device building blocks of the B200 DLIC hot path.
//
// * PTX wrappers for tcgen05 (MMA with A in TMEM, TMEM ld/st/alloc), mbarrier
//   and thread-block-cluster (DSMEM) operations, sm_100a only.
// * Thread organisation shared by the encoder and the decoder: 512 threads =
//   16 warps per CTA and 64 pixel rows = an M=64 tcgen05 tile, whose rows sit
//   in the half-subpartition TMEM layout (row m -> lane (m%16) + 32*(m/16)).
//   Warp w serves lane quadrant q = w&3 (rows 16q..16q+15) and column group
//   j = w>>2; its two half-warps h (lanes 0-15 / 16-31) address the same 16
//   rows at two column offsets (tcgen05 .16x32bx2 shape).  Each row is thus
//   served by 8 threads (4 groups x 2 halves), each owning a contiguous column
//   range; per-row partials combine with one shuffle (xor 16) and an exchange
//   through spare TMEM columns (TcEngine) or shared memory (Fp32Engine).
// * The two density-estimator engines (P:96 dense network, reading R4):
//     TcEngine   bf16 operands on 5th-gen tensor cores; weights resident in
//                shared memory in the UMMA no-swizzle K-major core-matrix
//                layout; activations and accumulators live in TMEM.
//     Fp32Engine fp32 FFMA on CUDA cores, k ascending for every output.
// * The deterministic softmax -> Q1' table -> CDF step (reading R5),
//   written with explicit _rn/_rd intrinsics and a fixed reduction tree so
//   encoder and decoder derive bit-identical tables ("the same matrices
//   ... rounding errors ... are the same during encoding and decoding").
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace dlic {

// ---------------------------------------------------------------- constants
constexpr int KIN = 78;        // causal 9x9 window (R1)
constexpr int KIN3 = 87;       // + the 3x3 box of the slice below (3D window R13)
constexpr int KPAD = 80;       // layer-1 K padded to a multiple of 16 for kind::f16
constexpr int HID = 128;       // P100K hidden width (R4)
constexpr int NOUT = 256;      // 8-bit alphabet
constexpr int NLAYER = 6;      // "six dense layers"
constexpr int ROWS = 64;       // pixel rows per CTA = M of the tcgen05 tile
constexpr int NGRP = 4;        // column groups per row (4 warps each)
constexpr int NTHREADS = 512;
constexpr uint32_t RANS_L = 1u << 16;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float Q1_SCALE = 65279.0f;  // 2^16 - 257 (R5, Q1')
// exp pairs q with q % 8 >= DLIC_POLY_FROM use the FMA-pipe polynomial (4 of
// 16 pairs), the rest MUFU ex2 (measured best split on C2 decode)
#ifndef DLIC_POLY_FROM
#define DLIC_POLY_FROM 6
#endif
// the same for column groups 2-3 (logits [128, 256), the decoder's later half)
#ifndef DLIC_POLY_FROM_HI
#define DLIC_POLY_FROM_HI DLIC_POLY_FROM
#endif
// group max in s1a as a 3-input tree (1) or the sequential chain (0); exact
// either way
#ifndef DLIC_MAX_TREE
#define DLIC_MAX_TREE 0
#endif
// 12-bit head (q12_row): column pairs on the FMA-pipe polynomial, of 8
#ifndef DLIC_Q12_POLY
#define DLIC_Q12_POLY 0
#endif
// thread whose clock profile the DLIC_PROF decoder records (a row thread)
#ifndef DLIC_PROF_TID
#define DLIC_PROF_TID 32
#endif
// Arithmetic revision of the density estimator + softmax/Q1' (container
// header field "numerics"): the integer tables are a function of the exact
// instruction sequence (engine K order, layer-1 split, epilogue rounding, the
// MUFU/polynomial exp split), so a container decodes only with a build of the
// same revision.  Bump NUMERICS_BASE on any change that can alter a table bit;
// the exp split is folded in so that a -DDLIC_POLY_FROM variant build can never
// decode another build's containers.  Value 0 is reserved for the oracle's own
// arithmetic (fp64 / bf16-emulated network, fp64 softmax).
constexpr uint32_t NUMERICS_BASE = 3;  // 2: fp32 path on the tensor cores (bf16x3); 3: packed 12-bit head (fma exp arguments)
constexpr uint32_t NUMERICS_REV = (NUMERICS_BASE << 8) | (uint32_t)DLIC_POLY_FROM | ((uint32_t)DLIC_Q12_POLY << 4) |
                                   (DLIC_POLY_FROM_HI != DLIC_POLY_FROM ? (uint32_t)DLIC_POLY_FROM_HI << 12 : 0u);

// Layer-1 K order of the bf16 engine.  K position p = 10u + i belongs to
// thread u = 2j + h (column group j, half h), which feeds A packed columns
// [5u, 5u + 5).  Thread u owns window row dr = u - 8 (i < 9: dc = i - 6) and
// one tap of the target row (i = 9, u < 6: dc = u - 6); positions 69 and 79
// are zero pads.  With this order every tap of a thread is a fixed offset from
// one per-thread ring address (decoder gather).  Returns the R1 row-major
// tap index of position p, or -1 for a pad; the host packer permutes
// W1's rows the same way, so the product is unchanged.
__host__ __device__ constexpr int kpos_tap(int p) {
  return p % 10 < 9 ? 9 * (p / 10) + p % 10 : (p / 10 < 6 ? 72 + p / 10 : -1);
}

// bf16 weight image (bytes) per layer, core-matrix layout (see host packer)
__host__ __device__ constexpr int layer_k(int l) { return l == 0 ? KPAD : HID; }
__host__ __device__ constexpr int layer_n(int l) { return l == NLAYER - 1 ? NOUT : HID; }
__host__ __device__ constexpr uint32_t wimg_off(int l) {
  return l == 0 ? 0u : (l <= 5 ? 20480u + 32768u * (uint32_t)(l - 1) : 217088u);
}
constexpr uint32_t WIMG_BYTES = 217088;  // 20480 + 4*32768 + 65536
constexpr int BIAS_OFF_LAST = 5 * HID;   // biases: 5 x 128 hidden, then 256
constexpr int BIAS_TOTAL = 5 * HID + NOUT;
// The two "fresh" taps of the wavefront: the only window cells of pixel
// (r, c) decoded on the immediately preceding front (c-1+3r and c+2+3(r-1)
// both equal step(r,c) - 1, reading R3).  Their layer-1 weights are taken out
// of the bf16 MMA image and applied on the CUDA cores in the layer-1
// epilogue (exact products v/256 * bf16 weight, fp32 FMA), so that the MMA
// over the other 76 taps can be issued one front early.
constexpr int TAP_FA = 77;  // (dr, dc) = (0, -1)
constexpr int TAP_FB = 71;  // (dr, dc) = (-1, +2)
// fresh-tap weight table after the biases: float4 per output pair n, n+1 =
// {wa[n], wa[n+1], wb[n], wb[n+1]} (bf16-rounded, as fp32)
constexpr int FRESH_OFF = BIAS_TOTAL;
constexpr int FRESH_FLOATS = 2 * HID;
constexpr uint32_t BIAS_BYTES = (BIAS_TOTAL + FRESH_FLOATS) * 4;
// 3D models: the 9 lower-layer taps' layer-1 weights after the fresh table,
// bf16 pairs [9][HID/2] (2,304 B; only loaded for 3D plans).  Their
// contribution is added to the layer-1 bias term on the CUDA cores (the taps
// were decoded long before, so it never waits), keeping the MMA at K = 80.
constexpr int W3D_OFF = BIAS_TOTAL + FRESH_FLOATS;
constexpr int W3D_WORDS = 9 * HID / 2;
constexpr uint32_t W3D_BYTES = W3D_WORDS * 4;

// fp32 weight blob: per layer W[K][N] then b[N]; K of layer 0 is KIN (78)
__host__ __device__ constexpr int f32_k(int l) { return l == 0 ? KIN : HID; }
__host__ __device__ constexpr uint32_t f32_off(int l) {
  uint32_t o = 0;
  for (int i = 0; i < l; ++i) o += (uint32_t)(f32_k(i) * layer_n(i) + layer_n(i));
  return o;
}

// TMEM column map (one 512-column allocation per CTA)
constexpr uint32_t TM_D = 0;     // accumulator / logits / e / f, 256 columns
constexpr uint32_t TM_A = 256;   // A operand of layers 2-6, K/2 columns (bf16 pairs), 64
constexpr uint32_t TM_A0 = 384;  // A operand of layer 1 (80 inputs -> 40 columns)
// decoder: second A buffer.  With split layers the epilogue of layer l starts
// (column groups 0-1) while the second half of layer l still reads its input,
// so consecutive layers' inputs alternate between TM_A and TM_A2.
constexpr uint32_t TM_A2 = 448;
constexpr uint32_t TM_X = 320;   // exchange slot s: columns TM_X+4s+j (lower half-warp)
constexpr uint32_t TM_XUP = 32;  //   and TM_X+32+4s+j (upper half-warp copy)
constexpr uint32_t TM_COLS = 512;
constexpr int NXSLOT = 7;  // 0 max, 1 Z, 2 F, 3 fc, 4/5 search result, 6 slot
#ifndef DLIC_SPLIT_LOGITS
#define DLIC_SPLIT_LOGITS 1
#endif

// decoder: last layer as two N=128 halves, the first issued per column group
constexpr bool DEC_SPLIT_LOGITS = DLIC_SPLIT_LOGITS != 0;
// decoder hidden accumulator of odd layers (layer l at dcol_of(l)); with the
// split logits, layer 5 (l = 4) must sit in [128,256)
constexpr uint32_t DEC_D_ODD = DEC_SPLIT_LOGITS ? 0u : 128u;
#ifndef DLIC_NSPLIT
#define DLIC_NSPLIT 1
#endif
#ifndef DLIC_EPI2H
#define DLIC_EPI2H 0  // (1: two 8-column TMEM loads in flight; 0.45% slower since the slot mbarrier)
#endif
#ifndef DLIC_LOGIT_EARLY
#define DLIC_LOGIT_EARLY 1
#endif
#ifndef DLIC_NSPLIT_ORDER
#define DLIC_NSPLIT_ORDER 1
#endif
// decoder: hidden layers as two N=64 halves committed separately
constexpr bool DEC_NSPLIT = DLIC_NSPLIT != 0;
constexpr int NXS_SMEM = 4;  // shared-memory exchange slots of the encoder engines (0 max, 1 Z, 2 F, 3 fc)

// ------------------------------------------------------------- small PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int quad() { return (threadIdx.x >> 5) & 3; }
// (& 3: in the decoder the row warps are warps 1-16 after the rANS warp 0;
// warp 16 then takes (quadrant 0, group 0), every pair still exactly once)
__device__ __forceinline__ int col_grp() { return (threadIdx.x >> 7) & 3; }
__device__ __forceinline__ int half_id() { return (threadIdx.x >> 4) & 1; }
__device__ __forceinline__ int tile_row() { return 16 * quad() + (threadIdx.x & 15); }

// named barrier over the 16 row warps (the decoder's rANS warp is not part)
__device__ __forceinline__ void row_sync() { asm volatile("bar.sync 6, 512;" ::: "memory"); }

// named barrier over the 4 warps that share one TMEM lane quadrant
__device__ __forceinline__ void quad_sync() {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + ((threadIdx.x >> 5) & 3)), "r"(128) : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
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

// pure spin on the phase (mbarrier.test_wait never suspends the thread)
__device__ __forceinline__ void mbar_spin(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
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
// Warp-wide variants: all 32 lanes execute them (converged, identical
// operands) and one elected lane issues, so the operands can live in uniform
// registers instead of a per-MMA elect/broadcast loop.
__device__ __forceinline__ void umma_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_warp(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

#define DLIC_R4(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3])
#define DLIC_R8(i) DLIC_R4(i), DLIC_R4(i + 4)
#define DLIC_W2(i) "r"(v[i]), "r"(v[i + 1])
#define DLIC_W8(i) "r"(v[i]), "r"(v[i + 1]), "r"(v[i + 2]), "r"(v[i + 3]), "r"(v[i + 4]), "r"(v[i + 5]), "r"(v[i + 6]), "r"(v[i + 7])


// .16x32bx2: lanes 0-15 of the warp address TMEM lanes base..base+15 at
// column taddr, lanes 16-31 the same TMEM lanes at column taddr + OFF;
// .xN = N consecutive columns per thread.
template <int OFF>
__device__ __forceinline__ void tmem_ld32h(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], %33;"
      : DLIC_R8(0), DLIC_R8(8), DLIC_R8(16), DLIC_R8(24)
      : "r"(taddr), "n"(OFF));
}
template <int OFF>
__device__ __forceinline__ void tmem_ld16h(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16], %17;"
      : DLIC_R8(0), DLIC_R8(8)
      : "r"(taddr), "n"(OFF));
}
template <int OFF>
__device__ __forceinline__ void tmem_ld8h(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : DLIC_R8(0)
               : "r"(taddr), "n"(OFF));
}
template <int OFF>
__device__ __forceinline__ void tmem_ld4h(uint32_t taddr, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], %5;" : DLIC_R4(0) : "r"(taddr), "n"(OFF));
}
template <int OFF>
__device__ __forceinline__ void tmem_st8h(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.16x32bx2.x8.b32 [%0], %1, {%2,%3,%4,%5,%6,%7,%8,%9};" ::"r"(taddr), "n"(OFF),
               DLIC_W8(0)
               : "memory");
}
template <int OFF>
__device__ __forceinline__ void tmem_st4h(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.16x32bx2.x4.b32 [%0], %1, {%2,%3,%4,%5};" ::"r"(taddr), "n"(OFF),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
               : "memory");
}
template <int OFF>
__device__ __forceinline__ void tmem_st1h(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.16x32bx2.x1.b32 [%0], %1, {%2};" ::"r"(taddr), "n"(OFF), "r"(v) : "memory");
}

// ---- clusters / DSMEM
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
// (no release: for a warp that publishes no memory to other CTAs -- a
// release arrive waits for every outstanding memory operation of the thread,
// including its TMA bulk copies in flight)
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
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
__device__ __forceinline__ void st_cluster_u16(uint32_t caddr, uint32_t v) {
  asm volatile("st.shared::cluster.u16 [%0], %1;" ::"r"(caddr), "h"((unsigned short)v) : "memory");
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
// relu then RN to bf16, lo in bits 0-15 (F2FP.RELU.BF16.PACK_AB)
__device__ __forceinline__ uint32_t pack_bf16_relu(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// packed fp32 pairs (FADD2 / FMUL2 / FFMA2 on sm_100); each lane is IEEE RN
// (or RM for add_rm), bit-identical to the scalar instruction.
struct f2 {
  uint64_t v;
};
__device__ __forceinline__ f2 f2_make(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ f2 f2_bits(uint32_t a, uint32_t b) { return f2_make(__uint_as_float(a), __uint_as_float(b)); }
__device__ __forceinline__ void f2_split(f2 x, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x.v));
}
__device__ __forceinline__ f2 f2_add(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 f2_add_rm(f2 a, f2 b) {
  f2 r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 f2_mul(f2 a, f2 b) {
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 f2_fma(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}

// Optional phase profiler (debug: thread 0, clock64 deltas).
struct Prof {
  unsigned long long t = 0, acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long t2 = 0, acc2[4] = {0, 0, 0, 0};
  bool on = false;
  __device__ __forceinline__ void mark(int k) {
    if (on) {
      const unsigned long long n = clock64();
      acc[k] += n - t;
      t = n;
      t2 = n;
    }
  }
  __device__ __forceinline__ void mark2(int k) {  // sub-phases of the network
    if (on) {
      const unsigned long long n = clock64();
      acc2[k] += n - t2;
      t2 = n;
    }
  }
};

// ---------------------------------------------------------------- engines
// Common engine interface (per thread = one row, group j, half h):
//   put_input(...)      this thread's share of the layer-1 input
//   start_l0 / issue_l0 layer 1 (the MMA over the 76 early taps for TcEngine)
//   run_rest(xa, xb, hook)  the rest of the network, fresh taps (xa, xb)
//                       applied in layer 1's epilogue; hook(l) in MMA waits
//   ld32(v)             this thread's 32 logits [64j+32h, +32)
//   bias_pair(i)        final-layer bias of its columns 2i, 2i+1 (added once)
//   xput(slot, v); xsync(); xget4(slot, v4)   exchange one word per group
//                        (v must already be equal in both half-warps)

// Template parameters: the TMEM columns of the hidden-layer accumulator (DH),
// of the A operand of layers 2-6 (AO) and of layer 1 (A0O); the logits always
// land in columns [TM_D, TM_D + 256).  XS: exchange words through shared
// memory (xs) instead of TMEM columns.  The decoder uses the default map
// (TcEngine); the encoder runs two tiles in flight with two maps (k_enc_pp).
// The per-row arithmetic is the same instruction sequence for every map.
template <uint32_t DH, uint32_t AO, uint32_t A0O, bool XS>
struct TcEngineT {
  uint32_t tmem;       // TMEM base (lane 0, column base)
  uint32_t wsmem;      // shared address of the bf16 weight image
  const float* bias;   // shared [BIAS_TOTAL]
  uint32_t bar;        // shared address of the MMA-completion mbarrier
  uint32_t phase;
  uint32_t* xs;        // XS: shared exchange words [NXS_SMEM][NGRP][ROWS]
  uint32_t bar2;       // decoder (DEC_NSPLIT): completion of the hidden layers' columns [64,128)
  const float* b0;     // layer-1 biases (HID): `bias`, or the tile's image's metadata-folded bias (global)

  __device__ __forceinline__ uint32_t lane_off() const { return ((threadIdx.x >> 5) & 3u) << 21; }

  // Layer-1 input: this thread's 5 packed bf16 pairs = inputs [20j+10h, +10)
  // (A packed columns [10j+5h, +5)).
  __device__ __forceinline__ void put_input(const uint32_t (&a)[5]) const {
    const uint32_t base = tmem + lane_off() + A0O + 10u * (uint32_t)col_grp();
    tmem_st4h<5>(base, a);
    tmem_st1h<5>(base + 4, a[4]);
  }

  // Issuers of run_rest (the single-tile-chain path k_enc_mlp<1>, used for the
  // bf16 debug exports of logits/probabilities/tables): the MMAs of a layer are issued by
  // warp 13 (layer 3's by warp 14) after a CTA barrier.  The production
  // encoder (k_enc_pp) and the decoder (run_rest_ws) use a dedicated issuer
  // warp instead.
  static constexpr unsigned MMA_ISSUER = 416;   // warp 13
  static constexpr unsigned MMA_ISSUER2 = 448;  // warp 14
  __device__ __forceinline__ static unsigned issuer(int l) { return l == 2 ? MMA_ISSUER2 : MMA_ISSUER; }

  // Issuer only: layer l's MMAs (K/16 slices, M=64) and their commit.
  __device__ __forceinline__ void issue(int l) const {
    tc_fence_after();
    const int K = layer_k(l), N = layer_n(l);
    const uint32_t id = umma_idesc(64, N);
    const uint32_t lbo = (uint32_t)N * 16u;                // next 8-wide K core matrix
    const uint32_t kstep = 2u * (uint32_t)(N / 8) * 128u;  // one K=16 slice
    // start-address field (bits 0-13, 16-byte units) advances by kstep/16
    uint64_t bd = umma_desc(wsmem + wimg_off(l), lbo, 128u);
    uint32_t at = tmem + (l == 0 ? A0O : AO);
    const uint32_t dt = tmem + (l == NLAYER - 1 ? TM_D : DH);
    umma_ts(dt, at, bd, id, 0u);
    for (int kk = 1; kk < K / 16; ++kk) {
      bd += kstep >> 4;
      at += 8u;
      umma_ts(dt, at, bd, id, 1u);
    }
    umma_commit(bar);
  }
  // The same, executed by a whole (converged) warp; one elected lane issues.
  __device__ __forceinline__ void issue_warp(int l) const {
    tc_fence_after();
    const int K = layer_k(l), N = layer_n(l);
    const uint32_t id = umma_idesc(64, N);
    const uint32_t lbo = (uint32_t)N * 16u;
    const uint32_t kstep = 2u * (uint32_t)(N / 8) * 128u;
    uint64_t bd = umma_desc(wsmem + wimg_off(l), lbo, 128u);
    uint32_t at = tmem + (l == 0 ? A0O : AO);
    const uint32_t dt = tmem + (l == NLAYER - 1 ? TM_D : DH);
    umma_ts_warp(dt, at, bd, id, 0u);
    for (int kk = 1; kk < K / 16; ++kk) {
      bd += kstep >> 4;
      at += 8u;
      umma_ts_warp(dt, at, bd, id, 1u);
    }
    umma_commit_warp(bar);
  }
  // K-slices [s0, s1) of layer l into the accumulator at column dcol (whole
  // converged warp, one elected lane issues; no commit).
  // NI/N0: instruction N and first output column (a column range of the
  // layer's weight image; NI = 0 -> the whole layer)
  __device__ __forceinline__ void issue_slices(int l, int s0, int s1, uint32_t dcol, int NI = 0, int N0 = 0,
                                               uint32_t acol = 0xFFFFFFFFu) const {
    tc_fence_after();
    const int N = layer_n(l);
    const uint32_t id = umma_idesc(64, NI ? NI : N);
    const uint32_t lbo = (uint32_t)N * 16u;
    const uint32_t kstep = 2u * (uint32_t)(N / 8) * 128u;
    const uint64_t bd = umma_desc(wsmem + wimg_off(l) + (uint32_t)(N0 / 8) * 128u, lbo, 128u);
    const uint32_t at = tmem + (acol != 0xFFFFFFFFu ? acol : (l == 0 ? A0O : AO));
    for (int kk = s0; kk < s1; ++kk)
      umma_ts_warp(tmem + dcol, at + 8u * (uint32_t)kk, bd + (uint64_t)((kstep >> 4) * (uint32_t)kk), id,
                   kk > 0 ? 1u : 0u);
  }
  __device__ __forceinline__ void commit_warp() const { umma_commit_warp(bar); }
  // Layer 0 over the 76 early taps (fresh weights are zero in the image),
  // after put_input (all threads; the caller supplies the barrier).
  __device__ __forceinline__ void issue_l0() const {
    if (threadIdx.x == MMA_ISSUER) issue(0);
  }
  // Encoder: input stored -> barrier -> layer 0 issued.
  __device__ __forceinline__ void start_l0() const {
    tc_wait_st();
    tc_fence_before();
    row_sync();
    issue_l0();
  }
  __device__ __forceinline__ void wait_mma() {
    mbar_wait(bar, phase);
    phase ^= 1u;
    tc_fence_after();
  }
  // decoder: column groups 0-1 wait on `bar`, groups 2-3 on `bar2` (the two
  // N=64 halves of a hidden layer complete separately)
  __device__ __forceinline__ void wait_mma_g() {
    if (DEC_NSPLIT) mbar_wait(col_grp() < 2 ? bar : bar2, phase);
    else mbar_wait(bar, phase);
    phase ^= 1u;
    tc_fence_after();
  }
  __device__ __forceinline__ void commit_both() const {
    umma_commit_warp(bar);
    if (DEC_NSPLIT) umma_commit_warp(bar2);
  }
  // bias + ReLU + bf16 -> next A; this thread's columns [32j+16h, +16)
  // (packed column 16j+8h+q holds activations 32j+16h+2q, +1: identity K order).
  // Layer 0 also adds the fresh taps: fma(xb, wb, fma(xa, wa, acc)) + bias.
  // this thread's 16 biases of layer l (loaded before the MMA wait, so the
  // adds after the TMEM load are register-only)
  __device__ __forceinline__ void load_bias(int l, float2 (&bq)[8]) const {
    const float4* b4 = reinterpret_cast<const float4*>((l == 0 ? b0 : bias + l * HID) + 32 * col_grp() + 16 * half_id());
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 b = b4[q];
      bq[2 * q] = make_float2(b.x, b.y);
      bq[2 * q + 1] = make_float2(b.z, b.w);
    }
  }
  template <bool L0>
  __device__ __forceinline__ void epilogue(const float2 (&b2)[8], float xa, float xb) const {
    epilogue_at<L0>(DH, b2, xa, xb, AO);
  }
  // hidden-layer epilogue in two 8-column halves (the second TMEM load is in
  // flight while the first half is converted)
  __device__ __forceinline__ void epilogue_2h(uint32_t dcol, uint32_t acol, const float2 (&b2)[8]) const {
    const uint32_t lo = lane_off();
    const int j = col_grp();
    uint32_t va[8], vb[8];
    tmem_ld8h<16>(tmem + lo + dcol + 32u * (uint32_t)j, va);
    tmem_ld8h<16>(tmem + lo + dcol + 32u * (uint32_t)j + 8u, vb);
    tc_wait_ld();
    uint32_t p[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float x0, x1;
      f2_split(f2_add(f2_bits(va[2 * q], va[2 * q + 1]), f2_make(b2[q].x, b2[q].y)), x0, x1);
      p[q] = pack_bf16_relu(x0, x1);
      f2_split(f2_add(f2_bits(vb[2 * q], vb[2 * q + 1]), f2_make(b2[4 + q].x, b2[4 + q].y)), x0, x1);
      p[4 + q] = pack_bf16_relu(x0, x1);
    }
    tmem_st8h<8>(tmem + lo + acol + 16u * (uint32_t)j, p);
    tc_wait_st();
  }
  // the same with the accumulator at TMEM column dcol (the decoder's
  // double-buffered hidden accumulator)
  template <bool L0>
  __device__ __forceinline__ void epilogue_at(uint32_t dcol, const float2 (&b2)[8], float xa, float xb,
                                              uint32_t acol) const {
    const uint32_t lo = lane_off();
    const int j = col_grp(), h = half_id();
    const float4* fw = reinterpret_cast<const float4*>(bias + FRESH_OFF) + 16 * j + 8 * h;
    uint32_t v[16];
    tmem_ld16h<16>(tmem + lo + dcol + 32u * (uint32_t)j, v);
    tc_wait_ld();
    const f2 xa2 = f2_make(xa, xa), xb2 = f2_make(xb, xb);
    uint32_t p[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float2 b = b2[q];
      f2 acc = f2_bits(v[2 * q], v[2 * q + 1]);
      if constexpr (L0) {
        const float4 w = fw[q];
        acc = f2_fma(xa2, f2_make(w.x, w.y), acc);
        acc = f2_fma(xb2, f2_make(w.z, w.w), acc);
      }
      float x0, x1;
      f2_split(f2_add(acc, f2_make(b.x, b.y)), x0, x1);
      p[q] = pack_bf16_relu(x0, x1);  // relu(x) rounded to bf16 (RN)
    }
    tmem_st8h<8>(tmem + lo + acol + 16u * (uint32_t)j, p);
    tc_wait_st();
  }
  // Layers 1..6 after layer 0's MMAs were issued (start_l0 / issue_l0):
  // wait, layer-0 epilogue with the fresh taps (xa, xb), then per layer:
  // barrier, issue, hook(l) (all threads; overlaps the tensor core), wait,
  // epilogue.  The logits are left in TMEM columns [0, 256).
  template <class Hook>
  __device__ __forceinline__ void run_rest(float xa, float xb, Hook&& hook, Prof* pf = nullptr) {
    if (pf) pf->t2 = clock64();
    float2 bq[8];
    load_bias(0, bq);
    wait_mma();
    if (pf) pf->mark2(2);
    epilogue<true>(bq, xa, xb);
    if (pf) pf->mark2(3);
#pragma unroll
    for (int l = 1; l < NLAYER; ++l) {
      tc_fence_before();
      row_sync();
      if (pf) pf->mark2(0);
      if ((threadIdx.x >> 5) == (issuer(l) >> 5)) issue_warp(l);  // the whole (converged) issuer warp
      hook(l);
      if (pf) pf->mark2(1);
      if (l < NLAYER - 1) load_bias(l, bq);
      wait_mma();
      if (pf) pf->mark2(2);
      if (l < NLAYER - 1) epilogue<false>(bq, 0.0f, 0.0f);
      if (pf) pf->mark2(3);
    }
  }

  // Decoder network with a dedicated issuer warp (k_decode): the 16 row warps
  // never meet at a CTA barrier inside the network.  Each warp arrives on
  // grp[j] (j = its column group, 4 warps) once its epilogue of layer l is in
  // TMEM; the issuer issues layer l+1's K-slices 2j, 2j+1 (the activations of
  // group j) as soon as group j has arrived, so the MMA starts while the other
  // groups still finish.  Hidden accumulators alternate between columns
  // [0,128) and [128,256) (layer l at 128*(l&1)); the logits take [0,256)
  // after every group's last hidden epilogue (dec_issue_network).
  // input columns of layer l >= 1 (its A operand), alternating
  static __device__ __forceinline__ uint32_t ao_of(int l) { return (l & 1) ? TM_A : TM_A2; }
  static __device__ __forceinline__ uint32_t dcol_of(int l) { return (l & 1) ? DEC_D_ODD : 128u - DEC_D_ODD; }
  // group j signals on named barrier 8 + j (its 4 warps arrive, the issuer
  // warp syncs: 160 threads)
  template <class Hook, class Pre0>
  __device__ __forceinline__ void run_rest_ws(float xa, float xb, Hook&& hook, Pre0&& pre0) {
    float2 bq[8];
    const uint32_t gbar = 8u + (uint32_t)col_grp();
    auto signal = [&]() {
      tc_fence_before();
      asm volatile("bar.arrive %0, 160;" ::"r"(gbar) : "memory");
    };
    load_bias(0, bq);
    pre0(bq);  // 3D window: the lower layer's term joins the layer-1 bias (add_w3d)
    wait_mma_g();
    epilogue_at<true>(dcol_of(0), bq, xa, xb, ao_of(1));
    signal();
#pragma unroll
    for (int l = 1; l < NLAYER; ++l) {
      hook(l);
      if (l < NLAYER - 1) load_bias(l, bq);
      wait_mma_g();
      if (l < NLAYER - 1) {
#if DLIC_EPI2H
        epilogue_2h(dcol_of(l), ao_of(l + 1), bq);
#else
        epilogue_at<false>(dcol_of(l), bq, 0.0f, 0.0f, ao_of(l + 1));
#endif
        signal();
      }
    }
  }
  // issuer side of run_rest_ws for layers 2..6 (whole warp)
  __device__ __forceinline__ void dec_issue_network() const {
#pragma unroll
    for (int l = 1; l < NLAYER; ++l) {
      if (l < NLAYER - 1 && DEC_NSPLIT) {
        // two N=64 halves: columns [0,64) (groups 0-1's next epilogue) are
        // committed to bar first, [64,128) to bar2
        const uint32_t d = dcol_of(l);
        asm volatile("bar.sync 8, 160;" ::: "memory");
        issue_slices(l, 0, 2, d, 64, 0, ao_of(l));
        asm volatile("bar.sync 9, 160;" ::: "memory");
        issue_slices(l, 2, 4, d, 64, 0, ao_of(l));
#if DLIC_NSPLIT_ORDER == 0
        issue_slices(l, 0, 4, d + 64u, 64, 64, ao_of(l));
#endif
        asm volatile("bar.sync 10, 160;" ::: "memory");
        issue_slices(l, 4, 6, d, 64, 0, ao_of(l));
        asm volatile("bar.sync 11, 160;" ::: "memory");
        issue_slices(l, 6, 8, d, 64, 0, ao_of(l));
        umma_commit_warp(bar);
#if DLIC_NSPLIT_ORDER == 0
        issue_slices(l, 4, 8, d + 64u, 64, 64, ao_of(l));
#else
        issue_slices(l, 0, 8, d + 64u, 64, 64, ao_of(l));
#endif
        umma_commit_warp(bar2);
        continue;
      }
      if (l < NLAYER - 1) {
#pragma unroll
        for (int j = 0; j < NGRP; ++j) {
          asm volatile("bar.sync %0, 160;" ::"r"(8 + j) : "memory");
          issue_slices(l, 2 * j, 2 * j + 2, dcol_of(l), 0, 0, ao_of(l));
        }
      } else if (DEC_SPLIT_LOGITS) {
        // logits columns [0,128) into [0,128) (layer 4's accumulator, long
        // read) group by group; [128,256) over layer 5's accumulator after
        // every group's epilogue
#pragma unroll
        for (int j = 0; j < NGRP; ++j) {
          asm volatile("bar.sync %0, 160;" ::"r"(8 + j) : "memory");
          issue_slices(l, 2 * j, 2 * j + 2, TM_D, 128, 0, ao_of(l));
        }
#if DLIC_LOGIT_EARLY
        if (DEC_NSPLIT) {  // groups 0-1's logits are columns [0,128): their softmax may start
          umma_commit_warp(bar);
          issue_slices(l, 0, 8, TM_D + 128u, 128, 128, ao_of(l));
          umma_commit_warp(bar2);
          continue;
        }
#endif
        issue_slices(l, 0, 8, TM_D + 128u, 128, 128, ao_of(l));
      } else {  // logits over [0,256): after every group's last hidden epilogue
#pragma unroll
        for (int j = 0; j < NGRP; ++j) asm volatile("bar.sync %0, 160;" ::"r"(8 + j) : "memory");
        issue_slices(l, 0, 8, TM_D, 0, 0, ao_of(l));
      }
      commit_both();
    }
  }

  __device__ __forceinline__ void ld32(uint32_t (&v)[32]) const {
    tmem_ld32h<32>(tmem + lane_off() + TM_D + 64u * (uint32_t)col_grp(), v);
    tc_wait_ld();
  }
  __device__ __forceinline__ float2 bias_pair(int i) const {
    return reinterpret_cast<const float2*>(bias + BIAS_OFF_LAST + 64 * col_grp() + 32 * half_id())[i];
  }
  __device__ __forceinline__ void xput(int slot, uint32_t v) const {
    if constexpr (XS) {
      if (half_id() == 0) xs[(slot * NGRP + col_grp()) * ROWS + tile_row()] = v;
    } else {
      tmem_st1h<TM_XUP>(tmem + lane_off() + TM_X + 4u * (uint32_t)slot + (uint32_t)col_grp(), v);
    }
  }
  __device__ __forceinline__ void xsync() const {
    if constexpr (XS) {
      quad_sync();
    } else {
      tc_wait_st();
      tc_fence_before();
      quad_sync();
      tc_fence_after();
    }
  }
  // slots s and s+1 (adjacent TMEM columns) with one load
  __device__ __forceinline__ void xget8(int slot, uint32_t (&v)[8]) const {
    if constexpr (XS) {
#pragma unroll
      for (int g = 0; g < 2 * NGRP; ++g) v[g] = xs[(slot * NGRP + g) * ROWS + tile_row()];
    } else {
      tmem_ld8h<TM_XUP>(tmem + lane_off() + TM_X + 4u * (uint32_t)slot, v);
      tc_wait_ld();
    }
  }
  __device__ __forceinline__ void xget4(int slot, uint32_t (&v)[4]) const {
    if constexpr (XS) {
#pragma unroll
      for (int g = 0; g < NGRP; ++g) v[g] = xs[(slot * NGRP + g) * ROWS + tile_row()];
    } else {
      tmem_ld4h<TM_XUP>(tmem + lane_off() + TM_X + 4u * (uint32_t)slot, v);
      tc_wait_ld();
    }
  }
};
using TcEngine = TcEngineT<TM_D, TM_A, TM_A0, false>;

// CUDA-core fp32 engine.  Shared buffers, column index = tile row (64):
//   buf0: [256][ROWS] floats (input features / hidden / logits), buf1: [128][ROWS],
//   xbuf: [NXSLOT][NGRP][ROWS] words.  Thread (row, j, h) computes outputs
//   [N/4*j + N/8*h, +N/8) of every layer for its row, k ascending.
struct Fp32Engine {
  float* buf0;
  float* buf1;
  uint32_t* xbuf;
  const float* w;   // global fp32 blob (f32_off layout, layer 0 with k0 rows)
  const float* b0;  // per-image layer-1 biases (metadata folded in), or null: the blob's
  int k0 = KIN;     // layer-1 inputs: 78, or 87 for the 3D window (R13)

  __device__ __forceinline__ void put_input(int k, float x) const { buf0[k * ROWS + tile_row()] = x; }

  __device__ __forceinline__ void issue_l0() const {}
  __device__ __forceinline__ void start_l0() const {}
  // Same interface as TcEngine: the whole network on the CUDA cores, after
  // the fresh taps are stored with the others (the fp32 engine has no early
  // layer 0).
  template <class Hook>
  __device__ __forceinline__ void run_rest(float xa, float xb, Hook&& hook, Prof* = nullptr) {
    put_input(TAP_FA, xa);
    put_input(TAP_FB, xb);
#pragma unroll 1
    for (int l = 1; l < NLAYER; ++l) {
      if (l > 1) row_sync();  // the hooks rely on the layer barriers between them
      hook(l);
    }
    run();
  }
  __device__ void run() {
    const int t = tile_row(), j = col_grp(), h = half_id();
#pragma unroll 1
    for (int l = 0; l < NLAYER; ++l) {
      quad_sync();  // this layer's inputs (written by the row's 8 threads) are complete
      const float* in = (l & 1) ? buf1 : buf0;
      float* out = (l & 1) ? buf0 : buf1;
      const int K = l == 0 ? k0 : f32_k(l), N = layer_n(l);
      const float* W = w + f32_off(l) + (l > 0 ? (uint32_t)(k0 - KIN) * HID : 0u);
      const float* B = (l == 0 && b0) ? b0 : W + K * N;
      const int n8 = N / 8;
#pragma unroll 1
      for (int n0 = j * 2 * n8 + h * n8; n0 < j * 2 * n8 + (h + 1) * n8; n0 += 16) {
        float acc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = 0.0f;
#pragma unroll 4
        for (int k = 0; k < K; ++k) {
          const float a = in[k * ROWS + t];
          const float4* wr = reinterpret_cast<const float4*>(W + k * N + n0);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 w4 = __ldg(wr + q);
            acc[4 * q + 0] = __fmaf_rn(a, w4.x, acc[4 * q + 0]);
            acc[4 * q + 1] = __fmaf_rn(a, w4.y, acc[4 * q + 1]);
            acc[4 * q + 2] = __fmaf_rn(a, w4.z, acc[4 * q + 2]);
            acc[4 * q + 3] = __fmaf_rn(a, w4.w, acc[4 * q + 3]);
          }
        }
        // ping-pong buffers: `out` was last read by the previous layer, which
        // every thread of the row finished before this layer's top sync.
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float z = __fadd_rn(acc[i], __ldg(B + n0 + i));
          if (l < NLAYER - 1) z = fmaxf(z, 0.0f);
          out[(n0 + i) * ROWS + t] = z;
        }
      }
    }
    quad_sync();  // logits complete
  }
  __device__ __forceinline__ void ld32(uint32_t (&v)[32]) const {
    const int t = tile_row(), c0 = 64 * col_grp() + 32 * half_id();
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(buf0[(c0 + i) * ROWS + t]);
  }
  __device__ __forceinline__ float2 bias_pair(int) const { return make_float2(0.f, 0.f); }
  __device__ __forceinline__ void xput(int slot, uint32_t v) const {
    if (half_id() == 0) xbuf[(slot * NGRP + col_grp()) * ROWS + tile_row()] = v;
  }
  __device__ __forceinline__ void xsync() const { quad_sync(); }
  __device__ __forceinline__ void xget8(int slot, uint32_t (&v)[8]) const {  // slots s, s+1
#pragma unroll
    for (int g = 0; g < 2 * NGRP; ++g) v[g] = xbuf[(slot * NGRP + g) * ROWS + tile_row()];
  }
  __device__ __forceinline__ void xget4(int slot, uint32_t (&v)[4]) const {
#pragma unroll
    for (int g = 0; g < NGRP; ++g) v[g] = xbuf[(slot * NGRP + g) * ROWS + tile_row()];
  }
};

// ------------------------------------------------- 3D window: the lower layer
// The 9 taps of the slice below (R13) enter layer 1 through the bias term:
// for this thread's 16 columns [32j+16h, +16), pre_n = sum_k x_k w_kn (x_k =
// v_k / 256, w bf16; fp32 FMA, k ascending, from 0: the first product is
// exact) and b'_n = b_n + pre_n (fp32 RN).  The encoder and the decoder call
// this same routine, so their layer-1 inputs stay bit-identical (R8).
// taps: bytes 0-3 / 4-7 / 8 of the 9 taps (row-major 3x3 box) in t[0..2].
__device__ __forceinline__ void add_w3d(const float* bias, const uint32_t (&t)[3], float2 (&bq)[8]) {
  const uint4* w3 = reinterpret_cast<const uint4*>(bias + W3D_OFF) + 4 * col_grp() + 2 * half_id();
  f2 acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = f2_make(0.0f, 0.0f);
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const uint32_t v = (t[k >> 2] >> (8 * (k & 3))) & 0xFFu;
    const float x = __fadd_rn(__uint_as_float(0x3F800000u | (v << 15)), -1.0f);  // v / 256, exact
    const f2 xx = f2_make(x, x);
    const uint4 wa = w3[k * (HID / 8)], wb = w3[k * (HID / 8) + 1];  // 8 bf16 pairs = 16 columns
    const uint32_t wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
    for (int q = 0; q < 8; ++q)
      acc[q] = f2_fma(xx, f2_bits(wv[q] << 16, wv[q] & 0xFFFF0000u), acc[q]);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float a0, a1;
    f2_split(f2_add(f2_make(bq[q].x, bq[q].y), acc[q]), a0, a1);
    bq[q] = make_float2(a0, a1);
  }
}

// ------------------------------------------------- softmax -> Q1' -> CDF
// Reading R5 (Q1'), per row; thread (j, h) owns logits [64j+32h, +32):
//   m_j = max over group j;  e_i = 2^(l_i*log2e - m_j*log2e) (MUFU ex2 or the
//   FMA-pipe polynomial, fixed per column);  z_jh = (sum of even-position
//   terms) + (sum of odd-position terms), each ascending;  z_j = z_j0 + z_j1;
//   M = max_j m_j;  w_j = 2^(m_j*log2e - M*log2e);
//   Z = ((z_0 w_0 + z_1 w_1) + z_2 w_2) + z_3 w_3;  p_i = e_i * (w_j * (1/Z));
//   f_i = 1 + floor(p_i * 65279);  R = 2^16 - sum f_i >= 0 ; f_255 += R ;
//   c_i = exclusive prefix sum.
// Integers are carried as exact integer-valued floats (< 2^24).  The logit
// space is overwritten in place: biased logits, then e, then f.

struct Q1Row {
  float F[NGRP];  // per-group sums of the unadjusted f (exact integers)
  float R;        // residual on symbol 255
  float Fmine;    // this thread's half-group sum
  float hbase;    // sum of the lower half of this group if h == 1, else 0
  float P[3];     // this thread's prefix sums after 8, 16, 24 of its 32 entries
};

__device__ __forceinline__ f2 f2_splat(float a) { return f2_make(a, a); }
// max of three (FMNMX3)
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// 2^t for a pair, t <= ~0, on the FMA pipe (offloads MUFU, FA4-style):
// n = floor(t) via a round-toward-minus-infinity add of 1.5*2^23, f = t - n in
// [0,1), degree-5 fit of 2^f (max rel. error 1.8e-7, ~1.5 ulp, comparable to
// ex2.approx), exponent inserted with an integer add.  Clamped at -126 so the
// result stays normal (smaller values are < 2^-126 relative to the row max).
__device__ __forceinline__ f2 f2_exp2_poly(f2 t) {
  float t0, t1;
  f2_split(t, t0, t1);
  t = f2_make(fmaxf(t0, -126.0f), fmaxf(t1, -126.0f));
  const f2 j = f2_add_rm(t, f2_splat(12582912.0f));  // 1.5 * 2^23 + floor(t)
  const f2 n = f2_add(j, f2_splat(-12582912.0f));
  float n0, n1;
  f2_split(n, n0, n1);
  const f2 f = f2_add(t, f2_make(-n0, -n1));
  f2 p = f2_splat(0.0018951073288917542f);
  p = f2_fma(p, f, f2_splat(0.00894621480256319f));
  p = f2_fma(p, f, f2_splat(0.055863283574581146f));
  p = f2_fma(p, f, f2_splat(0.24014076590538025f));
  p = f2_fma(p, f, f2_splat(0.6931546330451965f));
  p = f2_fma(p, f, f2_splat(0.9999998807907104f));
  float j0, j1, p0, p1;
  f2_split(j, j0, j1);
  f2_split(p, p0, p1);
  const uint32_t r0 = __float_as_uint(p0) + ((__float_as_uint(j0) - 0x4B400000u) << 23);
  const uint32_t r1 = __float_as_uint(p1) + ((__float_as_uint(j1) - 0x4B400000u) << 23);
  return f2_bits(r0, r1);
}

// Passes 1 and A over this thread's 32 values, held in registers throughout:
// v = raw logits on entry (ld32), the integer table f (as floats) on return.
// ENC: also returns f and the half-local exclusive cum of `sym` when it lies in
// this thread's columns.  probs (nullable): p_i of the
// row (debug export, 256 entries).
// The softmax -> Q1' -> CDF computation of one row in stages, so that the
// encoder can interleave them with the next tile's network (each stage is a
// fixed instruction sequence; q1_table runs them back to back and gives the
// decoder the identical arithmetic):
//   s1a  biased logits (in place) and the group max m_j
//   s1b  e_i = 2^(l_i*log2e - m_j*log2e) for pairs [q0, q1) (in place),
//        accumulated into the even/odd pair sums zz in pair order
//   s1c  z_j (halves combined)
//   x1   one exchange of (m_j, z_j): M = max_j m_j, Z = sum_j z_j 2^(m_j - M)
//        in a fixed order, this group's scale w_j / Z
//   sA   pass A: f_i = 1 + floor(p_i * 65279) (x + 2^23 rounded toward -inf
//        has ulp 1) in place, block sums; posts the group sum
//   x2   the F exchange: per-group sums, residual R
template <bool ENC>
struct Q1Work {
  float m = 0.0f, z = 0.0f;
  f2 zz;
  f2 inv;
  float fs = 0.0f, cs_local = 0.0f;
  Q1Row r;

  template <class Eng>
  __device__ __forceinline__ void s1a(const Eng& e, uint32_t (&v)[32]) {
    float mm = -INFINITY;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const float2 b = e.bias_pair(q);
      float l0, l1;
      f2_split(f2_add(f2_bits(v[2 * q], v[2 * q + 1]), f2_make(b.x, b.y)), l0, l1);
      v[2 * q] = __float_as_uint(l0);
      v[2 * q + 1] = __float_as_uint(l1);
      if (!DLIC_MAX_TREE) mm = fmax3(mm, l0, l1);
    }
    if (DLIC_MAX_TREE) {
      float t1[11];
#pragma unroll
      for (int i = 0; i < 10; ++i)
        t1[i] = fmax3(__uint_as_float(v[3 * i]), __uint_as_float(v[3 * i + 1]), __uint_as_float(v[3 * i + 2]));
      t1[10] = fmaxf(__uint_as_float(v[30]), __uint_as_float(v[31]));
      mm = fmax3(fmax3(fmax3(t1[0], t1[1], t1[2]), fmax3(t1[3], t1[4], t1[5]), fmax3(t1[6], t1[7], t1[8])), t1[9],
                 t1[10]);
    }
    m = fmaxf(mm, __shfl_xor_sync(0xFFFFFFFFu, mm, 16));  // m_j, equal in both halves
    zz = f2_splat(0.0f);
  }
  template <int Q0, int Q1>
  __device__ __forceinline__ void s1b(uint32_t (&v)[32]) {
    const f2 nm = f2_splat(__fmul_rn(-m, LOG2E));
    const f2 l2e = f2_splat(LOG2E);
    const int pfrom = col_grp() < 2 ? DLIC_POLY_FROM : DLIC_POLY_FROM_HI;  // (warp-uniform)
#pragma unroll
    for (int q = Q0; q < Q1; ++q) {
      const f2 t = f2_fma(f2_bits(v[2 * q], v[2 * q + 1]), l2e, nm);
      float e0, e1;
      if (q % 8 >= pfrom) {  // 4 of 16 pairs on the FMA pipe, the rest on MUFU (DLIC_POLY_FROM)
        f2_split(f2_exp2_poly(t), e0, e1);
      } else {
        float t0, t1;
        f2_split(t, t0, t1);
        e0 = ex2_approx(t0);
        e1 = ex2_approx(t1);
      }
      zz = f2_add(zz, f2_make(e0, e1));
      v[2 * q] = __float_as_uint(e0);
      v[2 * q + 1] = __float_as_uint(e1);
    }
  }
  __device__ __forceinline__ void s1c() {
    float za, zb;
    f2_split(zz, za, zb);
    const float zl = __fadd_rn(za, zb);
    z = __fadd_rn(zl, __shfl_xor_sync(0xFFFFFFFFu, zl, 16));  // commutative: identical in both halves
  }
  template <class Eng>
  __device__ __forceinline__ void x1(const Eng& e) {
    const int j = col_grp();
    e.xput(0, __float_as_uint(m));
    e.xput(1, __float_as_uint(z));
    e.xsync();
    uint32_t x8[8];
    e.xget8(0, x8);  // m_j (slot 0) and z_j (slot 1) in one load
    const uint32_t* x4 = x8;
    const uint32_t* z4 = x8 + 4;
    // M = max_j m_j;  Z = sum_j z_j 2^(m_j - M) in a fixed order;  group scale
    // s_j = 2^(m_j - M) / Z, so p_i = e_i * s_j = exp(l_i - M) / Z.
    const float M = fmaxf(fmaxf(__uint_as_float(x4[0]), __uint_as_float(x4[1])),
                          fmaxf(__uint_as_float(x4[2]), __uint_as_float(x4[3])));
    const float nM = __fmul_rn(-M, LOG2E);
    float wg[4];
#pragma unroll
    for (int g = 0; g < NGRP; ++g) wg[g] = ex2_approx(__fmaf_rn(__uint_as_float(x4[g]), LOG2E, nM));
    const float Z = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(__uint_as_float(z4[0]), wg[0]),
                                                  __fmul_rn(__uint_as_float(z4[1]), wg[1])),
                                        __fmul_rn(__uint_as_float(z4[2]), wg[2])),
                              __fmul_rn(__uint_as_float(z4[3]), wg[3]));
    float wmine = wg[0];
#pragma unroll
    for (int g = 1; g < NGRP; ++g)
      if (g == j) wmine = wg[g];
    inv = f2_splat(__fmul_rn(wmine, __frcp_rn(Z)));
  }
  template <class Eng>
  __device__ __forceinline__ void sA(const Eng& e, uint32_t (&v)[32], int sym, float* probs) {
    const int h = half_id();
    const int c0 = 64 * col_grp() + 32 * h;
    const f2 scale = f2_splat(Q1_SCALE);
    const f2 two23 = f2_splat(8388608.0f);
    const f2 fbias = f2_splat(-8388607.0f);  // y - 2^23 + 1 = 1 + floor(x), exact
    f2 FB[4] = {f2_splat(0.0f), f2_splat(0.0f), f2_splat(0.0f), f2_splat(0.0f)};  // 8-entry blocks
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const f2 p = f2_mul(f2_bits(v[2 * q], v[2 * q + 1]), inv);
      const f2 f = f2_add(f2_add_rm(f2_mul(p, scale), two23), fbias);
      FB[q >> 2] = f2_add(FB[q >> 2], f);
      float f0, f1;
      f2_split(f, f0, f1);
      if (probs) {
        float p0, p1;
        f2_split(p, p0, p1);
        probs[c0 + 2 * q] = p0;
        probs[c0 + 2 * q + 1] = p1;
      }
      v[2 * q] = __float_as_uint(f0);
      v[2 * q + 1] = __float_as_uint(f1);
    }
    float B[4];  // exact integer block sums
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      float Fa, Fb;
      f2_split(FB[b], Fa, Fb);
      B[b] = __fadd_rn(Fa, Fb);
    }
    r.P[0] = B[0];
    r.P[1] = B[0] + B[1];
    r.P[2] = r.P[1] + B[2];
    r.Fmine = r.P[2] + B[3];
    if (ENC) {
      // f_s and the exclusive cum of s within this thread's 32 columns (when
      // s lies there): the 8-entry block of s from the block sums, then the
      // block's entries.  All values are integers < 2^16 and all partial
      // sums < 2^24, so every fp32 sum here is exact in any order.
      const int d = sym - c0;
      const int kb = (d >> 3) & 3, ib = d & 7;
      float within = 0.0f, fsel = 0.0f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t lo01 = (kb & 1) ? v[8 + i] : v[i];
        const uint32_t hi01 = (kb & 1) ? v[24 + i] : v[16 + i];
        const float f = __uint_as_float((kb & 2) ? hi01 : lo01);
        within += i < ib ? f : 0.0f;
        fsel = i == ib ? f : fsel;
      }
      fs = fsel;
      cs_local = (kb == 0 ? 0.0f : (kb == 1 ? r.P[0] : (kb == 2 ? r.P[1] : r.P[2]))) + within;
    }
    const float Fo = __shfl_xor_sync(0xFFFFFFFFu, r.Fmine, 16);
    r.hbase = h ? Fo : 0.0f;
    e.xput(2, __float_as_uint(__fadd_rn(r.Fmine, Fo)));  // exact integer sum
  }
  template <class Eng>
  __device__ __forceinline__ void x2(const Eng& e) {
    e.xsync();
    uint32_t x4[4];
    e.xget4(2, x4);
#pragma unroll
    for (int g = 0; g < NGRP; ++g) r.F[g] = __uint_as_float(x4[g]);
    r.R = 65536.0f - (((r.F[0] + r.F[1]) + r.F[2]) + r.F[3]);
  }
};

// Passes 1 and A over this thread's 32 values, held in registers throughout:
// v = raw logits on entry (ld32), the integer table f (as floats) on return.
// ENC: also returns f and the half-local exclusive cum of `sym` when it lies
// in this thread's columns.  probs (nullable): p_i of the row (debug export).
template <bool ENC, class Eng>
__device__ __forceinline__ Q1Row q1_table(const Eng& e, uint32_t (&v)[32], int sym, float& fs, float& cs_local,
                                          float* probs, Prof* pf = nullptr) {
  Q1Work<ENC> w;
  w.s1a(e, v);
  if (pf) pf->mark2(2);
  w.template s1b<0, 16>(v);
  w.s1c();
  if (pf) pf->mark2(3);
  if (pf) pf->mark(4);
  w.x1(e);
  if (pf) pf->mark(5);
  w.sA(e, v, sym, probs);
  if (pf) pf->mark(7);
  w.x2(e);
  fs = w.fs;
  cs_local = w.cs_local;
  return w.r;
}

__device__ __forceinline__ float q1_base(const Q1Row& r) {
  const int j = col_grp();
  float base = r.hbase;
#pragma unroll
  for (int g = 0; g < NGRP; ++g)
    if (g < j) base += r.F[g];
  return base;
}

// Final integer table of this thread's 32 columns (debug export).
__device__ __forceinline__ void q1_store_freqs(const uint32_t (&v)[32], const Q1Row& r, uint16_t* freqs) {
  const int c0 = 64 * col_grp() + 32 * half_id();
  if (freqs) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float f = __uint_as_float(v[i]);
      if (c0 + i == NOUT - 1) f += r.R;
      freqs[c0 + i] = (uint16_t)f;
    }
  }
}

// Encoder: (f_s | c_s << 16) of the true symbol (all threads of the row).
// probs/freqs (nullable, per row, 256 entries): debug export.
template <class Eng>
__device__ __forceinline__ uint32_t q1_encode(const Eng& e, int sym, float* probs = nullptr,
                                              uint16_t* freqs = nullptr, bool export_freqs = false) {
  float fs, csl;
  uint32_t v[32];
  e.ld32(v);
  const Q1Row r = q1_table<true>(e, v, sym, fs, csl, probs);
  if (export_freqs) q1_store_freqs(v, r, freqs);
  const int c0 = 64 * col_grp() + 32 * half_id();
  uint32_t packed = 0;
  if (sym >= c0 && sym < c0 + 32) {
    if (sym == NOUT - 1) fs += r.R;
    packed = (uint32_t)fs | ((uint32_t)(q1_base(r) + csl) << 16);
  }
  packed |= __shfl_xor_sync(0xFFFFFFFFu, packed, 16);
  e.xput(3, packed);
  e.xsync();
  uint32_t x4[4];
  e.xget4(3, x4);
  return x4[0] | x4[1] | x4[2] | x4[3];
}

// Decoder: symbol s with c_s <= slot < c_s + f_s (all threads of the row call
// it with the row's slot).  Exactly one of the row's 8 threads holds the slot
// in its column range (the ranges partition [0, 2^16)): it returns mine = true
// with the symbol and its (f_s, c_s); the others return mine = false.
// Search: 8-entry block sums from pass A pick the block, a reverse scan of its
// 8 entries with the monotone test slot < c_{i+1} finds s.  mid() runs (all
// threads) once the logits are loaded: the network's TMEM output is free.
template <class Eng, class Slot, class Mid>
__device__ __forceinline__ int q1_decode(const Eng& e, Slot&& slot_fn, bool& mine_out, uint32_t& fs_out,
                                         uint32_t& cs_out, Mid&& mid, Prof* pf = nullptr) {
  float fs, csl;
  uint32_t v[32];
  e.ld32(v);
  if (pf) pf->mark2(0);
  mid();
  if (pf) pf->mark2(1);
  const Q1Row r = q1_table<false>(e, v, -1, fs, csl, nullptr, pf);
  const float slot = (float)slot_fn();  // the row's rANS slot (may wait for the rANS warp)
  const int c0 = 64 * col_grp() + 32 * half_id();
  const float base = q1_base(r);
  const bool last = c0 == NOUT - 32;  // symbol 255 carries the residual R
  const float cum = base + r.Fmine + (last ? r.R : 0.0f);  // c at the end of my columns
  const bool mine = slot >= base && slot < cum;
  if (last) v[31] = __float_as_uint(__uint_as_float(v[31]) + r.R);
  // level 1: the 8-entry block holding the slot (block prefix sums from pass A)
  const float sl = slot - base;  // exact
  const int kb = (sl >= r.P[0]) + (sl >= r.P[1]) + (sl >= r.P[2]);
  float cend = kb == 0 ? r.P[0] : (kb == 1 ? r.P[1] : (kb == 2 ? r.P[2] : cum - base));
  // level 2: reverse scan of the block's 8 entries, test sl < c_{i+1}
  int sym = 0;
  float fsel = 0.0f, csel = 0.0f;
#pragma unroll
  for (int i = 7; i >= 0; --i) {
    const uint32_t lo01 = (kb & 1) ? v[8 + i] : v[i];
    const uint32_t hi01 = (kb & 1) ? v[24 + i] : v[16 + i];
    const float f = __uint_as_float((kb & 2) ? hi01 : lo01);
    const float lo = cend - f;  // exact
    if (sl < cend) {
      sym = i;
      fsel = f;
      csel = lo;
    }
    cend = lo;
  }
  if (pf) pf->mark(8);
  mine_out = mine;
  fs_out = (uint32_t)fsel;
  cs_out = (uint32_t)(csel + base);
  return sym + c0 + 8 * kb;
}

}  // namespace dlic
