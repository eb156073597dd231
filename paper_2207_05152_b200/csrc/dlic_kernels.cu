// dlic_kernels.cu — the B200 kernels of the DLIC hot path (sm_100a).
//
//   k_enc_mlp   every pixel at once (north_star (b)): window gather (P:63,
//               P:290; fill 0 P:59) -> dense network -> softmax -> Q1
//               table (R5) -> (f_s, c_s) of the true symbol.  Persistent CTAs
//               over 64-pixel tiles; tcgen05 (bf16) or FFMA (fp32) engine.
//   k_rans_enc  one warp per G-row group stream ("at most one [coder
//               instance] per pixel row"; R7): lanes = rows, walks the
//               wavefront in reverse (t desc, r desc), ballot/popc word
//               emission.
//   k_container / k_copy  header + prefix-sum stream compaction (a6).
//   k_dec_prep  parses container framing on the device (batch decode).
//   k_decode    persistent per-unit wavefront decoder: one
//               cluster of nc CTAs x 64 slots; every front: fresh taps from a
//               shared-memory ring -> same network (layer 1 over the older
//               taps issued a front early) -> Q1 search -> publish pixel
//               (DSMEM mirror) -> cluster barrier; the rANS step runs one
//               front late inside the next front's network.
#include <cstdint>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include "dlic_device.cuh"
#include "dlic_internal.h"
#include "dlic_stream.cuh"
#include "dlic_x3.cuh"



namespace dlic {

// decoder: the rANS warp publishes a front's slots on an mbarrier that each
// row thread waits on right before its symbol search (1), or on named barrier
// 7 that all 16 row warps sync on after the network (0).  With 1 the column
// groups whose logits half lands first start their softmax at once (C2
// decode 10.92 -> 10.50 ms).  The 12-bit engine keeps barrier 7 either way
// (its head has no early half; its key is read before the second pass).
#ifndef DLIC_SLOT_MBAR
#define DLIC_SLOT_MBAR 1
#endif

// Decoded-pixel ring, column-major so the 32 lanes of a warp (consecutive
// rows) touch distinct shared-memory banks: byte (bank, pos, ringrow) at
// bank*RING_BANK + pos*RING_ROWS + ringrow.  ringrow = 8 + slot-in-CTA; rows
// 0..7 mirror the previous CTA's last 8 slots (halo).  bank = pass parity of
// the READER's row (the wrap-around halo, written by the last CTA for the
// first CTA's next pass, flips it).  Column c lives at pos c & 31 and, for
// c & 31 < 8, also at pos 32 + (c & 31), so a window (dc in [-6, 2]) never
// wraps: it is read from pos cb + dc with cb = (c & 31) < 6 ? (c & 31) + 32 :
// (c & 31).  Out-of-image taps read zeros that the writers keep in place: the
// ring starts zeroed, a row clears its right pad (columns W, W+1) when it
// ends and the left pad (pos 26..31) of its slot's next row in the other bank.
constexpr int RING_ROWS = ROWS + 8;                           // own 64 slots + 8 halo rows
constexpr int RING_COLS = 40;                                 // 32-column ring + copies of 0..7
constexpr uint32_t RING_BANK = (uint32_t)RING_COLS * RING_ROWS;  // 2880
constexpr uint32_t RING_BYTES = 2u * RING_BANK;               // 5760
constexpr uint32_t F32_BUF_BYTES = (NOUT + HID) * ROWS * 4u;          // 98304
constexpr uint32_t F32_X_BYTES = NXSLOT * NGRP * ROWS * 4u;          // 7168
constexpr uint32_t MAX_DYN_SMEM = 232448 - 2048;                     // 227 KB minus static (fallback, see dec_smem_limit)

// bias region in shared memory: biases + fresh-tap table (+ the 3D taps'
// weights for volume plans)
__host__ __device__ inline uint32_t bias_bytes(uint32_t w3d) { return BIAS_BYTES + (w3d ? W3D_BYTES : 0u); }
// `precision` here is the ENGINE: 0 fp32 FFMA, 1 bf16 P100K (resident
// weights), 2 bf16 P350K (streamed weights, dlic_stream.cuh)
size_t enc_smem_bytes(uint32_t precision, uint32_t w3d) {
  if (precision == 4) return TcX3::SMEM;
  if (precision == 3) return TcStream12::SMEM;
  if (precision == 2) return TcStream::SMEM;
  return precision == 1 ? WIMG_BYTES + bias_bytes(w3d) : F32_BUF_BYTES + F32_X_BYTES;
}
static uint32_t cursor_bytes(uint32_t ngroups) { return (ngroups * 4u + 15u) & ~15u; }
// 3D decoder (bf16): lower-layer taps of each slot for the current and the
// next step, [2][ROWS][3] words (filled by the rANS warp)
constexpr uint32_t T3_BYTES = 2u * ROWS * 3u * 4u;
size_t dec_smem_bytes(uint32_t precision, uint32_t max_groups, uint32_t w3d) {
  return enc_smem_bytes(precision, w3d) + RING_BYTES * (precision == 3 ? 2u : 1u) + 16 + 3 * cursor_bytes(max_groups) +
         (w3d && precision == 1 ? T3_BYTES : 0u);  // (engine index, see enc_smem_bytes)
}
// dynamic shared memory a decoder block may use: the device's opt-in limit
// per block minus k_decode's static shared memory (queried once; the
// constant is the fallback when no device is visible)
size_t dec_smem_limit();

// ------------------------------------------------------------ engine setup
template <int PREC>
struct EngineSel;
template <>
struct EngineSel<1> {
  using T = TcEngine;
};
template <>
struct EngineSel<0> {
  using T = Fp32Engine;
};
template <>
struct EngineSel<2> {
  using T = TcStream;
};
template <>
struct EngineSel<3> {
  using T = TcStream12;
};
template <>
struct EngineSel<4> {
  using T = TcX3;
};
// decoded pixel storage: 12-bit alphabet (engine 3) in u16, else u8
template <int PREC>
using PixT = std::conditional_t<PREC == 3, uint16_t, uint8_t>;
template <int PREC>
__host__ __device__ constexpr int pix_bits() { return PREC == 3 ? 12 : 8; }
// v / 2^BITS exactly (v < 2^BITS): 1 + v/2^BITS has v in the top mantissa bits
template <int BITS>
__device__ __forceinline__ float unit_of(uint32_t v) {
  return __fadd_rn(__uint_as_float(0x3F800000u | (v << (23 - BITS))), -1.0f);
}
// a fresh tap as layer-1's epilogue takes it: v / 2^bits as a bf16 operand
// (exact for 8-bit pixels; 12-bit pixels are rounded like the MMA's taps)
template <int PREC>
__device__ __forceinline__ float fresh_in(uint32_t v) {
  const float x = unit_of<pix_bits<PREC>()>(v);
  if constexpr (PREC == 3) return __bfloat162float(__float2bfloat16_rn(x));
  return x;
}

__device__ __forceinline__ void load_smem(uint8_t* dst, const void* src, uint32_t bytes) {
  const int4* s4 = reinterpret_cast<const int4*>(src);
  int4* d4 = reinterpret_cast<int4*>(dst);
  for (uint32_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) d4[i] = __ldg(s4 + i);
}

// Shared setup of both engines at kernel start (all threads).  Returns the
// end of the engine's shared-memory region.
template <int PREC>
__device__ __forceinline__ uint8_t* engine_setup(typename EngineSel<PREC>::T& eng, uint8_t* smem, const DevWeights& w,
                                                 uint64_t* bar, uint32_t* tslot, uint32_t w3d) {  // bar: 2 mbarriers
  if constexpr (PREC >= 2) {  // streamed engines: layer 1 | ring | biases | full[S] empty[S] (| dfull[2] dfree[2])
    using E = typename EngineSel<PREC>::T;
    using Cfg = E;
    load_smem(smem + E::L1_O, w.wimg, E::L1_BYTES);
    load_smem(smem + E::BIAS_O, w.bias, E::BIAS_BYTES);
    const uint32_t bars = smem_u32(smem + E::BARS_O);
    if (threadIdx.x < 32) tmem_alloc(smem_u32(tslot), TM_COLS);
    if (threadIdx.x == 0) {
      mbar_init(smem_u32(bar), 1);
      mbar_init(smem_u32(bar + 1), NTHREADS / 32);  // layer-1 input ready (row warps)
      for (int i = 0; i < 2 * Cfg::S; ++i) mbar_init(bars + 8u * (uint32_t)i, 1);
      if constexpr (E::HEAD) {
        for (int i = 0; i < 2; ++i) {
          mbar_init(bars + 8u * (2 * Cfg::S + i), 1);                 // dfull[b]: tcgen05.commit
          mbar_init(bars + 8u * (2 * Cfg::S + 2 + i), NTHREADS / 32);  // dfree[b]: the row warps
        }
      }
      fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    eng.tmem = *tslot;
    eng.bias = reinterpret_cast<const float*>(smem + E::BIAS_O);
    eng.b0 = eng.bias;
    eng.bar = smem_u32(bar);
    eng.bar2 = eng.bar;
    eng.phase = 0;
    eng.ring = smem_u32(smem + E::RING_O);
    eng.l1s = smem_u32(smem + E::L1_O);
    eng.full0 = bars;
    eng.empty0 = bars + 8u * Cfg::S;
    eng.dfull0 = bars + 8u * (2 * Cfg::S);
    eng.dfree0 = bars + 8u * (2 * Cfg::S + 2);
    eng.wstream = w.wimg;
    eng.aready = smem_u32(bar + 1);
    return smem + E::SMEM;
  } else if constexpr (PREC == 1) {
    load_smem(smem, w.wimg, WIMG_BYTES);
    load_smem(smem + WIMG_BYTES, w.bias, bias_bytes(w3d));
    if (threadIdx.x < 32) tmem_alloc(smem_u32(tslot), TM_COLS);
    if (threadIdx.x == 0) {
      mbar_init(smem_u32(bar), 1);
      fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    eng.tmem = *tslot;
    eng.wsmem = smem_u32(smem);
    eng.bias = reinterpret_cast<const float*>(smem + WIMG_BYTES);
    eng.b0 = eng.bias;
    eng.bar = smem_u32(bar);
    eng.phase = 0;
    return smem + WIMG_BYTES + bias_bytes(w3d);
  } else {
    eng.buf0 = reinterpret_cast<float*>(smem);
    eng.buf1 = eng.buf0 + NOUT * ROWS;
    eng.xbuf = reinterpret_cast<uint32_t*>(smem + F32_BUF_BYTES);
    eng.w = w.w32;
    eng.b0 = nullptr;
    eng.k0 = w3d ? KIN3 : KIN;
    return smem + F32_BUF_BYTES + F32_X_BYTES;
  }
}

template <int PREC>
__device__ __forceinline__ void engine_teardown(typename EngineSel<PREC>::T& eng) {
  if constexpr (PREC >= 1) {
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(eng.tmem, TM_COLS);
  }
}

// Feed this thread's share of the window inputs (encoder; the decoder has its
// own ring gather).  bf16: thread u = 2j + h owns K positions [10u, +10) in
// the kpos_tap order; get(dr, dc) returns the pixel value of that window
// offset (0 fill).  fp32: the same taps, stored at their R1 index.
__device__ __forceinline__ void tap_of(int u, int i, int& dr, int& dc) {
  if (i < 9) {
    dr = u - 8;
    dc = i - 6;
  } else {
    dr = 0;
    dc = u - 6;
  }
}
template <int PREC, class Eng, class Get>
__device__ __forceinline__ void feed(const Eng& eng, Get get, const uint32_t (*t3)[3] = nullptr) {
  const int u = 2 * col_grp() + half_id();
  constexpr int SHIFT = 23 - pix_bits<PREC>();
  if constexpr (PREC >= 1) {
    // v/2^bits exactly: (1 + v/2^bits) has v in the top mantissa bits; minus 1 is exact.
    const f2 m1 = f2_make(-1.0f, -1.0f);
    uint32_t a[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      int dr0, dc0, dr1, dc1;
      tap_of(u, 2 * q, dr0, dc0);
      tap_of(u, 2 * q + 1, dr1, dc1);
      const uint32_t v0 = get(dr0, dc0);
      const uint32_t v1 = (q < 4 || u < 6) ? get(dr1, dc1) : 0u;
      float x0, x1;
      f2_split(f2_add(f2_bits(0x3F800000u | (v0 << SHIFT), 0x3F800000u | (v1 << SHIFT)), m1), x0, x1);
      a[q] = pack_bf16(x0, x1);
    }
    eng.put_input(a);
  } else {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      int dr, dc;
      tap_of(u, i, dr, dc);
      if (i < 9 || u < 6)
        eng.put_input(i < 9 ? 9 * u + i : 72 + u, __fadd_rn(__uint_as_float(0x3F800000u | (get(dr, dc) << 15)), -1.0f));
    }
    if (t3) {  // 3D window: lower-layer tap u at input 78 + u, thread 0 also tap 8
      const uint32_t v = ((*t3)[u >> 2] >> (8 * (u & 3))) & 0xFFu;
      eng.put_input(KIN + u, __fadd_rn(__uint_as_float(0x3F800000u | (v << 15)), -1.0f));
      if (u == 0) eng.put_input(KIN + 8, __fadd_rn(__uint_as_float(0x3F800000u | ((*t3)[2] & 0xFFu) << 15), -1.0f));
    }
  }
}

// v/256 exactly (v < 256)
__device__ __forceinline__ float u8_unit(uint32_t v) {
  return __fadd_rn(__uint_as_float(0x3F800000u | (v << 15)), -1.0f);
}

// ------------------------------------------------------------ encoder MLP
// Persistent CTAs over 64-pixel tiles of the units' raster order.  Thread
// (row, j, h): pixel = tile*64 + row; (j, h) owns inputs [20j+10h, +10),
// hidden columns [32j+16h, +16) and logits [64j+32h, +32) (dlic_device.cuh).
// PREC 2 (P350K, TcStream): one more warp streams the weights and issues the
// MMAs (TcStream::issue_tiles); the row warps run the same code as PREC 0.
__host__ __device__ constexpr int enc_block(int prec) { return prec >= 2 ? NTHREADS + 64 : NTHREADS; }
template <int PREC>
__global__ void __launch_bounds__(enc_block(PREC), 1)
    k_enc_mlp(Plan p, DevWeights w, const uint8_t* __restrict__ imgs, uint32_t* __restrict__ fc,
              float* __restrict__ dbg_logits, float* __restrict__ dbg_probs, uint16_t* __restrict__ dbg_freqs) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar[3];  // 0 MMA completion, 2 spare (engine)
  __shared__ uint32_t tslot;
  __shared__ uint32_t s_nq[2];  // 12-bit: the tile's pass-2 chunk count, (tile ordinal << 8 | n), by tile parity
  if (threadIdx.x < 2) s_nq[threadIdx.x] = 0u;
  const int row = tile_row();
  using Pix = PixT<PREC>;
  constexpr int BITS = pix_bits<PREC>();
  const Pix* const imgp = reinterpret_cast<const Pix*>(imgs);
  typename EngineSel<PREC>::T eng;
  engine_setup<PREC>(eng, smem, w, bar, &tslot, p.w3d);
  if constexpr (PREC == 3) eng.nq2s = s_nq;  // (engine_setup's barrier orders the zeroing above)
  // tiles of units [u_lo, u_lo + u_cnt) (global tile index = tbase + k)
  const uint64_t tbase = (uint64_t)p.u_lo * p.tiles_per_unit;
  const uint64_t total = (uint64_t)p.u_cnt * p.tiles_per_unit;
  const bool dbg = dbg_logits || dbg_probs || dbg_freqs;
  if constexpr (PREC >= 2) {
    if (threadIdx.x >= NTHREADS) {  // weight stream + MMA issuer: one network per tile of this CTA
      // (the row warps take the one-tile-at-a-time loop: with 17 warps a
      // thread has 96 registers, too few to hold a tile's logits across the
      // next tile's network)
      const uint64_t n = total > blockIdx.x ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
      uint64_t pt = 0;
      int pk = 0;
      int tlen = EngineSel<PREC>::T::CPN;  // chunks of the current tile (12-bit: 80 + 2 x its pass-2 chunks)
      auto next = [&](int& c) -> bool {  // every tile's network chunks, in order
        if (pt >= n) return false;
        if constexpr (PREC == 3) {
          if (pk == CH_HID12 + H12_STREAM) {  // the tile's pass 2 starts: its length, published before start_l0
            mbar_wait(eng.aready, (uint32_t)pt & 1u);
            tlen = CH_HID12 + H12_STREAM + 2 * (int)(s_nq[pt & 1u] & 0xFFu);
          }
        }
        c = pk;
        if (++pk == tlen) {
          pk = 0;
          ++pt;
          tlen = EngineSel<PREC>::T::CPN;
        }
        return true;
      };
      eng.prof = p.prof != 0;
      eng.mode = p.prof;
      if (threadIdx.x < NTHREADS + 32) {
        eng.issue_tiles(n);  // warp 16: MMA issuer
      } else {
        eng.produce_all(next);  // warp 17: weight-stream producer
        if (eng.prof && lane_id() == 0) atomicAdd(&g_sprof[1], eng.pw[1]);
      }
      engine_teardown<PREC>(eng);
      return;
    }
  }

  // this thread's pixel of a tile (64 consecutive pixels of a unit in raster
  // order).  The pipelined loop walks its tiles in order, so the unit (and
  // its divisions) is recomputed only when a tile starts a new unit.
  struct Px {
    bool valid;
    int r, c, uw, uh, z, sym;
    const Pix* img;
    uint64_t gi, fci;
  };
  uint32_t cu = 0xFFFFFFFFu;  // cached unit
  Unit cun;
  auto pixel = [&](uint64_t tile) -> Px {
    Px x;
    const uint32_t t32 = (uint32_t)tile;  // < 2^32 tiles (checked by the planner)
    const uint32_t u = t32 / p.tiles_per_unit;
    const uint32_t kt = t32 - u * p.tiles_per_unit;
    if (u != cu) {
      cu = u;
      cun = unit_info(p, u);
      if (w.b1img) eng.b0 = w.b1img + (uint64_t)(cun.img / p.depth) * HID;  // the tile's image's metadata-folded layer-1 bias
    }
    const uint32_t q = kt * (uint32_t)ROWS + (uint32_t)row;
    x.valid = q < cun.w * cun.h;
    x.r = x.valid ? (int)(q / cun.w) : 0;
    x.c = x.valid ? (int)(q - (uint32_t)x.r * cun.w) : 0;
    x.uw = (int)cun.w;
    x.uh = (int)cun.h;
    x.z = (int)(cun.img % p.depth);
    x.img = imgp + (uint64_t)cun.img * p.W * p.H + (uint64_t)cun.y0 * p.W + cun.x0;
    x.sym = 0;  // loaded by load_sym() when needed (its L2 latency off the tile start)
    x.gi = (uint64_t)cun.img * p.W * p.H + (uint64_t)(cun.y0 + x.r) * p.W + (cun.x0 + x.c);
    x.fci = cun.fc_off + q;
    return x;
  };
  auto load_sym = [&](Px& x) {
    if (x.valid) x.sym = (int)__ldg(x.img + (uint64_t)x.r * p.W + x.c);
  };
  // L1 prefetch of a tile's window rows (its 10 taps + the target), issued a
  // tile ahead so the feed's loads hit L1 (no registers held)
  auto prefetch_px = [&](const Px& x) {
    if (!x.valid) return;
    const int u = 2 * col_grp() + half_id();
    const int rr = max(x.r + u - 8, 0);
    const Pix* a = x.img + (int64_t)rr * p.W + max(x.c - 6, 0);
    asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(x.img + (int64_t)x.r * p.W + x.c));
  };
  auto getter = [&](const Px& x) {
    return [&x, &p](int dr, int dc) -> uint32_t {  // branch-free: invalid taps load the target and mask
      const int rr = x.r + dr, cc = x.c + dc;
      const bool ok = x.valid && rr >= 0 && (unsigned)cc < (unsigned)x.uw;
      const uint32_t v = __ldg(x.img + (ok ? (int64_t)rr * p.W + cc : (int64_t)x.r * p.W + x.c));
      return ok ? v : 0u;
    };
  };
  // 3D window: the 3x3 box of the previous slice (same unit; fill 0 outside it, below slice 0)
  auto lower = [&](const Px& x, uint32_t (&t3)[3]) {
    t3[0] = t3[1] = t3[2] = 0u;
    for (int k = 0; k < 9; ++k) {
      const int rr = x.r + k / 3 - 1, cc = x.c + k % 3 - 1;
      const bool ok = x.valid && x.z > 0 && rr >= 0 && rr < x.uh && cc >= 0 && cc < x.uw;
      const uint32_t v = ok ? (uint32_t)__ldg(x.img - (uint64_t)p.W * p.H + (int64_t)rr * p.W + cc) : 0u;
      t3[k >> 2] |= v << (8 * (k & 3));
    }
  };
  auto feed_x = [&](const Px& x, auto& get) {
    if (p.w3d) {
      uint32_t t3[3];
      lower(x, t3);
      feed<PREC>(eng, get, &t3);
    } else {
      feed<PREC>(eng, get);
    }
  };

  if (dbg || PREC >= 2) {  // debug exports (and P350K, P12): one tile at a time
    uint32_t kt = 0;  // this CTA's tile ordinal
#pragma unroll 1
    for (uint64_t tile = tbase + blockIdx.x; tile < tbase + total; tile += gridDim.x, ++kt) {
      const long long c0 = clock64();
      Px x = pixel(tile);
      load_sym(x);
      auto get = getter(x);
      feed_x(x, get);
      uint32_t nq2 = (uint32_t)H12_NCH;
      if constexpr (PREC == 3) {
        // the second head pass only needs the chunks up to the tile's largest
        // true symbol (c_s sums the f of the symbols below s; the f of each
        // chunk are the decoder's): count published for the issuer and the
        // producer before start_l0, read back after a row-warp barrier
        const uint32_t mq = dbg ? (uint32_t)H12_NCH : (x.valid ? (uint32_t)x.sym / (uint32_t)H12_CN + 1u : 1u);
        const uint32_t wq = __reduce_max_sync(0xFFFFFFFFu, mq);
        if (lane_id() == 0) atomicMax(&s_nq[kt & 1u], (kt << 8) | wq);
        row_sync();
        nq2 = s_nq[kt & 1u] & 0xFFu;
      }
      eng.start_l0();
      const long long c1 = clock64();
      eng.run_rest(fresh_in<PREC>(get(0, -1)), fresh_in<PREC>(get(-1, 2)), [](int) {});
      const long long c2 = clock64();
      if constexpr (PREC == 3) {  // 12-bit head (R17): (f_s | c_s << 16) from the owning thread
        Q12Dbg dd{x.valid && dbg_logits ? dbg_logits + x.gi * H12_N : nullptr,
                   x.valid && dbg_probs ? dbg_probs + x.gi * H12_N : nullptr,
                   x.valid && dbg_freqs ? dbg_freqs + x.gi * H12_N : nullptr};
        bool mine;
        uint32_t fs, cs;
        q12_row<true>(eng, (uint32_t)x.sym, mine, fs, cs, []() {}, dbg ? &dd : nullptr, nq2);
        if (x.valid && mine) fc[x.fci] = fs | (cs << 16);
        if (p.prof && threadIdx.x == 0) {
          atomicAdd(&g_sprof[5], (unsigned long long)(c1 - c0));
          atomicAdd(&g_sprof[6], (unsigned long long)(c2 - c1));
          atomicAdd(&g_sprof[7], (unsigned long long)(clock64() - c2));
        }
        continue;
      }
      const uint32_t v = q1_encode(eng, x.sym, (x.valid && dbg_probs) ? dbg_probs + x.gi * NOUT : nullptr,
                                   (x.valid && dbg_freqs) ? dbg_freqs + x.gi * NOUT : nullptr, dbg_freqs != nullptr);
      if constexpr (PREC == 2) {
        if (p.prof && threadIdx.x == 0) {
          atomicAdd(&g_sprof[5], (unsigned long long)(c1 - c0));
          atomicAdd(&g_sprof[6], (unsigned long long)(c2 - c1));
          atomicAdd(&g_sprof[7], (unsigned long long)(clock64() - c2));
        }
      }
      if (dbg_logits) {  // raw logits (bias added) of this thread's 32 columns
        uint32_t lv[32];
        eng.ld32(lv);
        if (x.valid)
          for (int i = 0; i < 32; ++i) {
            const int cc = 64 * col_grp() + 32 * half_id() + i;
            float l = __uint_as_float(lv[i]);
            if constexpr (PREC == 1) l = __fadd_rn(l, eng.bias[BIAS_OFF_LAST + cc]);
            if constexpr (PREC == 2 || PREC == 4) l = __fadd_rn(l, eng.bias[EngineSel<PREC>::T::LAST_BIAS + cc]);
            dbg_logits[x.gi * NOUT + cc] = l;
          }
      }
      if (x.valid && threadIdx.x < ROWS * 2 && half_id() == 0) fc[x.fci] = v;
    }
    engine_teardown<PREC>(eng);
    return;
  }

  // Software pipeline over this CTA's tiles: the softmax -> Q1' stages of
  // tile k run in the MMA waits of tile k+1's network (its logits are in
  // registers once loaded, which frees the accumulator columns).  The thread
  // whose columns hold the true symbol writes (f_s | c_s << 16).
  auto write_fc = [&](const Px& x, const Q1Work<true>& qw) {
    const int c0 = 64 * col_grp() + 32 * half_id();
    if (x.valid && x.sym >= c0 && x.sym < c0 + 32) {
      float fsv = qw.fs;
      if (x.sym == NOUT - 1) fsv += qw.r.R;
      fc[x.fci] = (uint32_t)fsv | ((uint32_t)(q1_base(qw.r) + qw.cs_local) << 16);
    }
  };
  // each CTA takes a contiguous range of tiles: consecutive 64-pixel tiles
  // share most of their 9-row windows, which then hit L1
  const uint64_t per = (total + gridDim.x - 1) / gridDim.x;
  const uint64_t tend = tbase + min(total, per * (blockIdx.x + 1));
  uint64_t tile = tbase + per * blockIdx.x;
  if (tile < tend) {
    Px cur = pixel(tile);
    {
      auto get = getter(cur);
      feed_x(cur, get);
      eng.start_l0();
      if (tile + 1 < tend) prefetch_px(pixel(tile + 1));
      eng.run_rest(u8_unit(get(0, -1)), u8_unit(get(-1, 2)), [](int) {});
      load_sym(cur);
    }
#pragma unroll 1
    for (;;) {
      uint32_t v[32];
      eng.ld32(v);  // tile's logits
      Q1Work<true> qw;
      const uint64_t nxt = tile + 1;
      if (nxt < tend) {
        Px nx = pixel(nxt);
        auto get = getter(nx);
        if constexpr (PREC == 0) quad_sync();  // fp32: the logits buffer also holds the inputs
        feed_x(nx, get);
        eng.start_l0();
        // tile k's softmax -> Q1' stages in the MMA waits of tile k+1's
        // layers 2-6 (the last, N=256, has the longest wait); tile k+2's
        // window is prefetched into L1 meanwhile
        eng.run_rest(u8_unit(get(0, -1)), u8_unit(get(-1, 2)), [&](int l) {
          if (l == 1) {
            qw.s1a(eng, v);
            qw.template s1b<0, 8>(v);
          } else if (l == 2) {
            qw.template s1b<8, 16>(v);
            qw.s1c();
          } else if (l == 3) {
            qw.x1(eng);
            load_sym(nx);
          } else if (l == 4) {
            qw.sA(eng, v, cur.sym, nullptr);
          } else {
            qw.x2(eng);
            write_fc(cur, qw);
            if (nxt + 1 < tend) prefetch_px(pixel(nxt + 1));
          }
        });
        cur = nx;
        tile = nxt;
      } else {
        qw.s1a(eng, v);
        qw.template s1b<0, 16>(v);
        qw.s1c();
        qw.x1(eng);
        qw.sA(eng, v, cur.sym, nullptr);
        qw.x2(eng);
        write_fc(cur, qw);
        break;
      }
    }
  }
  engine_teardown<PREC>(eng);
}

// ------------------------------------------------------------ encoder MLP, two tiles in flight
// bf16 production encoder.  The tensor core would idle in every epilogue and
// softmax of a single tile chain, so each CTA keeps two 64-pixel tiles in
// flight (slot a, slot b) and a dedicated issuer warp (warp 16) alternates
// their MMAs: while the 16 row warps run the epilogue of a's layer l, b's
// layer l runs on the tensor core, and vice versa.  TMEM map (512 columns):
//   [0,128)   a: hidden accumulator      [0,256) logits of a and of b
//   [256,320) a: A operand (layer-1 input in its first 40 columns)
//   [320,448) b: hidden accumulator      [448,512) b: A operand
// The logits of the two slots share [0,256): b's last layer is issued after
// a's logits are in registers, and the next a's first layer after b's.
// Row warps arrive on named barrier 8 + s when slot s's next MMA may go;
// the issuer commits each layer to mma[s].  Exchanges go through shared
// memory (one region per slot).  Every row sees exactly the decoder's
// per-row instruction sequence (same engine code, same Q1Work stages), so
// the tables stay bit-identical (R8).
constexpr int ENC_PP_THREADS = NTHREADS + 32;
constexpr uint32_t ENC_PP_XS_BYTES = 2u * NXS_SMEM * NGRP * ROWS * 4u;
using EngA = TcEngineT<0, 256, 256, true>;
using EngB = TcEngineT<320, 448, 448, true>;

size_t enc_pp_smem_bytes(uint32_t w3d) { return WIMG_BYTES + bias_bytes(w3d) + ENC_PP_XS_BYTES; }

// DBG: parity tap of this production kernel -- per pixel (image raster order)
// the biased logits, the probabilities the quantiser used and the integer
// table, written from inside the same instruction sequence (R8), so tests can
// compare the production encoder itself with the oracle.
template <bool DBG, bool W3D>
__global__ void __launch_bounds__(ENC_PP_THREADS, 1)
    k_enc_pp(Plan p, DevWeights w, const uint8_t* __restrict__ imgs, uint32_t* __restrict__ fc,
             unsigned long long* __restrict__ prof, float* __restrict__ dbg_logits, float* __restrict__ dbg_probs,
             uint16_t* __restrict__ dbg_freqs) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[2];  // mma[0], mma[1] (tcgen05.commit)
  __shared__ uint32_t tslot;
  load_smem(smem, w.wimg, WIMG_BYTES);
  load_smem(smem + WIMG_BYTES, w.bias, bias_bytes(W3D));
  if (threadIdx.x < 32) tmem_alloc(smem_u32(&tslot), TM_COLS);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    mbar_init(smem_u32(&bars[1]), 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  EngA ea;
  EngB eb;
  uint32_t* xsb = reinterpret_cast<uint32_t*>(smem + WIMG_BYTES + bias_bytes(W3D));
  ea.tmem = eb.tmem = tslot;
  ea.wsmem = eb.wsmem = smem_u32(smem);
  ea.bias = eb.bias = reinterpret_cast<const float*>(smem + WIMG_BYTES);
  ea.b0 = eb.b0 = ea.bias;
  ea.bar = smem_u32(&bars[0]);
  eb.bar = smem_u32(&bars[1]);
  ea.phase = eb.phase = 0;
  ea.xs = xsb;
  eb.xs = xsb + NXS_SMEM * NGRP * ROWS;

  // tiles of units [u_lo, u_lo + u_cnt), contiguous ranges per CTA
  const uint64_t tbase = (uint64_t)p.u_lo * p.tiles_per_unit;
  const uint64_t total = (uint64_t)p.u_cnt * p.tiles_per_unit;
  const uint64_t per = (total + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = tbase + per * blockIdx.x;
  const uint64_t tend = tbase + min(total, per * (blockIdx.x + 1));
  const uint32_t ntl = t0 < tend ? (uint32_t)(tend - t0) : 0u;  // tiles of this CTA
  const uint32_t npairs = (ntl + 1) / 2;

  if (threadIdx.x >= NTHREADS) {
    // ================================================ issuer warp
    // (the whole warp runs the loop converged; one elected lane issues, the
    // per-layer descriptors are compile-time constants + the TMEM/smem bases)
    unsigned long long idle = 0, t0c = prof ? clock64() : 0;
#pragma unroll 1
    for (uint32_t k = 0; k < npairs; ++k) {
#pragma unroll
      for (int l = 0; l < NLAYER; ++l) {
        const unsigned long long c0 = prof ? clock64() : 0;
        asm volatile("bar.sync 8, %0;" ::"n"(ENC_PP_THREADS) : "memory");  // slot a ready
        ea.issue_warp(l);
        const unsigned long long c1 = prof ? clock64() : 0;
        asm volatile("bar.sync 9, %0;" ::"n"(ENC_PP_THREADS) : "memory");  // slot b ready
        if (prof) idle += clock64() - c1;
        eb.issue_warp(l);
        (void)c0;
      }
    }
    if (prof && threadIdx.x == NTHREADS) {
      atomicAdd(prof + 8, idle);
      atomicAdd(prof + 9, clock64() - t0c);
      atomicAdd(prof + 10, (unsigned long long)npairs);
    }
  } else {
    // ================================================ 16 row warps
    const int row = tile_row();
    const uint32_t lane = lane_id();
    // Feed cursor: this thread's pixel in the next tile to feed.  Tiles are
    // fed in order (t0, t0+1, ...), so the pixel advances by 64 raster
    // positions per tile without divisions; unit geometry is reloaded only
    // when a tile starts a new unit.
    uint32_t fu = 0, fkt = 0, fw = 1, fwh = 0;
    int fr = 0, fcol = 0;
    const uint8_t* fimg = imgs;
    uint64_t ffc = 0;
    uint64_t fgi = 0;  // DBG: image-raster index of the unit's pixel (0, 0)
    const float* fb0 = ea.bias;  // layer-1 biases of the cursor's image
    uint32_t fh = 1, fz = 0;     // W3D: unit height, slice index in its volume
    auto set_unit = [&](uint32_t u) {
      const Unit un = unit_info(p, u);
      fu = u;
      fkt = 0;
      fw = un.w;
      fwh = un.w * un.h;
      fr = (int)((uint32_t)row / un.w);
      fcol = row - fr * (int)un.w;
      fimg = imgs + (uint64_t)un.img * p.W * p.H + (uint64_t)un.y0 * p.W + un.x0;
      ffc = un.fc_off;
      fgi = (uint64_t)un.img * p.W * p.H + (uint64_t)un.y0 * p.W + un.x0;
      if (w.b1img) fb0 = w.b1img + (uint64_t)(un.img / p.depth) * HID;
      fh = un.h;
      fz = un.img % p.depth;
    };
    if (t0 < tend) {
      const uint32_t u0 = (uint32_t)(t0 / p.tiles_per_unit);
      set_unit(u0);
      fkt = (uint32_t)(t0 - (uint64_t)u0 * p.tiles_per_unit);
      const uint32_t q = fkt * (uint32_t)ROWS + (uint32_t)row;
      fr = (int)(q / fw);
      fcol = (int)(q - (uint32_t)fr * fw);
    }
    auto advance = [&]() {
      if (++fkt == p.tiles_per_unit) {
        if (fu + 1 < p.n_img * p.upi) set_unit(fu + 1);  // else stays past the end (fkt == tiles_per_unit)
      } else {
        fcol += ROWS;
        if (fw >= (uint32_t)ROWS) {
          if (fcol >= (int)fw) {
            fcol -= (int)fw;
            ++fr;
          }
        } else {
          const int k = fcol / (int)fw;
          fr += k;
          fcol -= k * (int)fw;
        }
      }
    };
    // what a tile's softmax needs later: the output index and the true
    // symbol (-1 for a pixel outside the unit)
    struct Px {
      uint64_t fci;
      int sym;
      uint64_t gi;     // DBG only
      uint32_t t3[3];  // W3D only: the 3x3 box of the slice below (R13), bytes row-major
    };
    // the cursor's tile -> layer-1 input of a slot; fresh taps, symbol.
    // Thread u = 2j + h reads window row dr = u - 8 (taps dc = -6..2) and,
    // for u < 6, the target-row tap dc = u - 6 (kpos_tap order).
    const int gu = 2 * col_grp() + half_id();
    auto feed_px = [&](auto& eng, bool live, float& xa, float& xb) -> Px {
      const uint32_t q = fkt * (uint32_t)ROWS + (uint32_t)row;
      const bool valid = live && q < fwh;
      const int rr = fr + gu - 8;
      const uint8_t* rp = fimg + (int64_t)rr * p.W + fcol;  // window row, column c
      const uint8_t* tp = fimg + (int64_t)fr * p.W + fcol;  // target row, column c
      uint32_t tv[10];
      if (valid && rr >= 0 && fcol >= 6 && fcol + 2 < (int)fw) {
#pragma unroll
        for (int i = 0; i < 9; ++i) tv[i] = __ldg(rp + i - 6);
      } else {
#pragma unroll
        for (int i = 0; i < 9; ++i) {
          const int cc = fcol + i - 6;
          tv[i] = (valid && rr >= 0 && cc >= 0 && cc < (int)fw) ? (uint32_t)__ldg(rp + i - 6) : 0u;
        }
      }
      tv[9] = (valid && gu < 6 && fcol + gu - 6 >= 0) ? (uint32_t)__ldg(tp + gu - 6) : 0u;
      const f2 m1 = f2_make(-1.0f, -1.0f);
      uint32_t a[5];
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        float x0, x1;
        f2_split(f2_add(f2_bits(0x3F800000u | (tv[2 * k] << 15), 0x3F800000u | (tv[2 * k + 1] << 15)), m1), x0,
                 x1);
        a[k] = pack_bf16(x0, x1);
      }
      eng.put_input(a);
      eng.b0 = fb0;  // the slot's layer-1 bias until its next feed
      // fresh taps (0,-1) and (-1,+2)
      xa = u8_unit((valid && fcol >= 1) ? (uint32_t)__ldg(tp - 1) : 0u);
      xb = u8_unit((valid && fr >= 1 && fcol + 2 < (int)fw) ? (uint32_t)__ldg(tp - p.W + 2) : 0u);
      Px o;
      o.fci = ffc + q;
      o.sym = valid ? (int)__ldg(tp) : -1;
      o.gi = fgi + (uint64_t)fr * p.W + (uint64_t)fcol;
      if constexpr (W3D) {  // same unit of the previous slice (fill 0 outside it and below slice 0)
        const uint8_t* lp = fimg - (uint64_t)p.W * p.H;
        o.t3[0] = o.t3[1] = o.t3[2] = 0u;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          const int rr = fr + k / 3 - 1, cc = fcol + k % 3 - 1;
          const bool ok = valid && fz > 0 && rr >= 0 && rr < (int)fh && cc >= 0 && cc < (int)fw;
          const uint32_t v = ok ? (uint32_t)__ldg(lp + (int64_t)rr * p.W + cc) : 0u;
          o.t3[k >> 2] |= v << (8 * (k & 3));
        }
      }
      if (live) advance();
      return o;
    };
    // L1 prefetch of this thread's window row `ahead` tiles past the cursor
    // (a hint: the address is clamped into the unit image, row wrap ignored)
    auto prefetch_ahead = [&](int ahead) {
      if (fkt + (uint32_t)ahead >= p.tiles_per_unit) return;
      const int cc = min(fcol + ahead * ROWS, (int)fw - 1);
      const int rr = max(fr + gu - 8, 0);
      asm volatile("prefetch.global.L1 [%0];" ::"l"(fimg + (int64_t)rr * p.W + max(cc - 6, 0)));
    };
    // slot s's next MMA may go: named barrier 8 + s (the 16 row warps
    // arrive, the issuer warp syncs)
    auto signal = [&](int slot) {
      tc_wait_st();
      tc_fence_before();
      if (slot == 0) asm volatile("bar.arrive 8, %0;" ::"n"(ENC_PP_THREADS) : "memory");
      else asm volatile("bar.arrive 9, %0;" ::"n"(ENC_PP_THREADS) : "memory");
    };
    auto write_fc = [&](const Px& x, const Q1Work<true>& qw) {
      const int c0 = 64 * col_grp() + 32 * half_id();
      if (x.sym >= c0 && x.sym < c0 + 32) {
        float fsv = qw.fs;
        if (x.sym == NOUT - 1) fsv += qw.r.R;
        fc[x.fci] = (uint32_t)fsv | ((uint32_t)(q1_base(qw.r) + qw.cs_local) << 16);
      }
    };

    // one tile's softmax -> Q1' -> (f_s, c_s), logits in v
    auto finish = [&](auto& eng, uint32_t (&v)[32], const Px& x) {
      Q1Work<true> qw;
      qw.s1a(eng, v);
      const int c0 = 64 * col_grp() + 32 * half_id();
      if constexpr (DBG) {  // biased logits of this thread's 32 columns
        if (dbg_logits && x.sym >= 0)
          for (int i = 0; i < 32; ++i) dbg_logits[x.gi * NOUT + c0 + i] = __uint_as_float(v[i]);
      }
      qw.template s1b<0, 16>(v);
      qw.s1c();
      qw.x1(eng);
      qw.sA(eng, v, x.sym, DBG && dbg_probs && x.sym >= 0 ? dbg_probs + x.gi * NOUT : nullptr);
      qw.x2(eng);
      if constexpr (DBG) {
        if (dbg_freqs && x.sym >= 0) q1_store_freqs(v, qw.r, dbg_freqs + x.gi * NOUT);
      }
      write_fc(x, qw);
    };
    if (npairs > 0) {
      float xaA, xbA, xaB, xbB;
      Px A = feed_px(ea, true, xaA, xbA);
      signal(0);
      Px B = feed_px(eb, ntl > 1, xaB, xbB);
      signal(1);
      float2 bq[8];
      const bool pon = prof != nullptr && threadIdx.x == 0;
      unsigned long long pt = pon ? clock64() : 0;
      auto pmark = [&](int i) {
        if (pon) {
          const unsigned long long n = clock64();
          atomicAdd(prof + i, n - pt);
          pt = n;
        }
      };
#pragma unroll 1
      for (uint32_t k = 0; k < npairs; ++k) {
        // layers 1..5 of a and b alternating on the tensor core; each
        // epilogue releases that slot's next layer.  Layer 1 adds the fresh
        // taps in its epilogue (same split as the decoder).
        ea.load_bias(0, bq);
        if constexpr (W3D) add_w3d(ea.bias, A.t3, bq);
        ea.wait_mma();
        ea.template epilogue<true>(bq, xaA, xbA);
        signal(0);
        eb.load_bias(0, bq);
        if constexpr (W3D) add_w3d(eb.bias, B.t3, bq);
        eb.wait_mma();
        eb.template epilogue<true>(bq, xaB, xbB);
        signal(1);
        pmark(0);
#pragma unroll 1
        for (int l = 1; l < NLAYER - 1; ++l) {
          ea.load_bias(l, bq);
          pmark(6);
          ea.wait_mma();
          pmark(7);
          ea.template epilogue<false>(bq, 0.0f, 0.0f);
          pmark(11);
          signal(0);  // l = 4: a's last layer (logits -> [0,256))
          pmark(12);
          if (l == 2) prefetch_ahead(0);
          if (l == 3) prefetch_ahead(1);
          eb.load_bias(l, bq);
          pmark(6);
          eb.wait_mma();
          pmark(7);
          eb.template epilogue<false>(bq, 0.0f, 0.0f);
          pmark(11);
          if (l < NLAYER - 2) signal(1);
          pmark(12);
        }
        const bool more = k + 1 < npairs;
        {
          // a's logits -> registers; b's last layer may then overwrite [0,256)
          uint32_t v[32];
          ea.wait_mma();
          ea.ld32(v);
          signal(1);
          pmark(1);
          finish(ea, v, A);  // overlaps b's last layer
          pmark(2);
        }
        if (more) A = feed_px(ea, true, xaA, xbA);  // a's A operand is free: its last layer is done
        pmark(3);
        {
          uint32_t v[32];
          eb.wait_mma();
          eb.ld32(v);
          const Px Bc = B;
          if (more) {
            signal(0);  // next a's layer 1: input written, b's logits out of [0,256)
            B = feed_px(eb, 2 * k + 3 < ntl, xaB, xbB);
            signal(1);
          }
          pmark(4);
          finish(eb, v, Bc);  // overlaps the next pair's layer 1
          pmark(5);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tslot, TM_COLS);
}

// ------------------------------------------------------------ rANS encoder
// One warp per stream.  Lane i = row r0+i of the group.  Fronts walked in
// reverse (LIFO); within a front rows descending = lanes descending, so
// lane i's emitted word goes after those of lanes > i.  Words are written
// backwards from the end of the stream's scratch region so the region tail is
// already in decoder order (t asc, r asc).
__global__ void __launch_bounds__(128) k_rans_enc(Plan p, const uint32_t* __restrict__ fc,
                                                  uint16_t* __restrict__ scratch, uint32_t* __restrict__ words) {
  const uint32_t s = p.s_lo + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const uint32_t lane = threadIdx.x & 31;
  if (s >= p.s_lo + p.s_cnt) return;  // warp-uniform
  uint32_t u, g;
  stream_info(p, s, u, g);
  const Unit un = unit_info(p, u);
  const uint32_t r0 = g * p.G;
  const uint32_t nr = min(p.G, un.h - r0);
  uint16_t* region = scratch + (uint64_t)s * p.cap_words;
  const uint32_t cap = p.cap_words;
  const bool lane_ok = lane < nr;
  const int r = (int)(r0 + lane);
  const uint32_t* frow = fc + un.fc_off + (uint64_t)r * un.w;
  uint32_t x = RANS_L;
  uint32_t n = 0;
  const int t_hi = 3 * (int)(r0 + nr - 1) + (int)un.w - 1;
  const int t_lo = 3 * (int)r0;
  // Software pipeline: the (f, c) of the next 16 steps of this lane are
  // independent loads (its row read backwards), issued together; the 16
  // dependent encode steps then run from registers.
  // The next chunk's loads are issued before the current chunk's steps (two
  // register buffers), so a chunk never starts on an L2 round trip.
  constexpr int CH = 16;
  auto load_chunk = [&](int t0, uint32_t (&fcv)[CH]) {
#pragma unroll
    for (int s = 0; s < CH; ++s) {
      const int c = t0 - s - 3 * r;
      const bool act = lane_ok && t0 - s >= t_lo && c >= 0 && c < (int)un.w;
      fcv[s] = act ? __ldg(frow + c) : 0u;  // 0 = inactive (f >= 1 for real pixels)
    }
  };
  uint32_t cur[CH], nxt[CH];
  load_chunk(t_hi, cur);
#pragma unroll 1
  for (int t0 = t_hi; t0 >= t_lo; t0 -= CH) {
    if (t0 - CH >= t_lo) load_chunk(t0 - CH, nxt);
#pragma unroll
    for (int s = 0; s < CH; ++s) {
      const bool act = cur[s] != 0u;
      const uint32_t f = act ? (cur[s] & 0xFFFFu) : 1u, cum = cur[s] >> 16;
      const bool emit = act && (x >> 16) >= f;  // x >= f * 2^16  (renormalise first, R6)
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, emit);
      if (emit) {
        const uint32_t kk = n + __popc(m >> lane >> 1);  // lanes above emit first
        region[cap - 1 - kk] = (uint16_t)(x & 0xFFFFu);
        x >>= 16;
      }
      n += __popc(m);
      if (act) x = ((x / f) << 16) + (x % f) + cum;
    }
#pragma unroll
    for (int s = 0; s < CH; ++s) cur[s] = nxt[s];
  }
  if (lane_ok) {
    region[2 * lane] = (uint16_t)(x >> 16);
    region[2 * lane + 1] = (uint16_t)(x & 0xFFFFu);
  }
  if (lane == 0) words[s] = 2 * nr + n;
}

// ------------------------------------------------------------ container
struct Sha {
  uint8_t b[32];
};

__device__ __forceinline__ void put_u16(uint8_t* o, uint32_t v) {
  o[0] = (uint8_t)v;
  o[1] = (uint8_t)(v >> 8);
}
__device__ __forceinline__ void put_u32(uint8_t* o, uint32_t v) {
  o[0] = (uint8_t)v;
  o[1] = (uint8_t)(v >> 8);
  o[2] = (uint8_t)(v >> 16);
  o[3] = (uint8_t)(v >> 24);
}

// Header (version 2) + the prefix sum of the stream
// sizes = each stream's byte offset.  payload_only (unit-range calls): no
// header, offsets relative to the payload start, streams [s_lo, s_lo + s_cnt).
__global__ void k_container(Plan p, Sha sha, const uint32_t* __restrict__ words, uint8_t* __restrict__ out,
                            uint64_t stride, uint64_t* __restrict__ sizes, uint64_t* __restrict__ dst,
                            int payload_only, const float* __restrict__ meta) {
  const uint32_t img = blockIdx.x;  // container index (a volume = depth slices)
  uint8_t* o = out + (uint64_t)img * stride;
  if (payload_only) {
    if (threadIdx.x == 0) {
      uint64_t off = 0;
      for (uint32_t s = p.s_lo; s < p.s_lo + p.s_cnt; ++s) {
        dst[s] = off;
        off += 2ull * words[s];
      }
      sizes[0] = off;
    }
    return;
  }
  if (threadIdx.x == 0) {
    o[0] = 'D';
    o[1] = 'L';
    o[2] = 'I';
    o[3] = 'C';
    o[4] = (uint8_t)CONTAINER_VERSION;
    o[5] = (uint8_t)p.precision;
    o[6] = p.w3d ? 2 : 1;  // window id (R1; 2 = the 3D window R13, a volume)
    o[7] = p.bits == 12 ? 12 : 0;  // alphabet (R15; 0 = 8-bit)
    put_u32(o + 8, p.W);
    put_u32(o + 12, p.H);
    put_u16(o + 16, p.hdr_tw);
    put_u16(o + 18, p.hdr_th);
    put_u16(o + 20, p.G);
    put_u16(o + 22, NUMERICS_REV);  // arithmetic revision of the tables (decode must match)
    for (int i = 0; i < 32; ++i) o[24 + i] = sha.b[i];
    put_u32(o + 56, p.spc);
    uint64_t off = p.hdr_bytes;
    // metadata block after the size table: u32 n, f32 raw reals
    uint8_t* mb = o + HDR_FIXED + 4u * p.spc;
    put_u32(mb, p.n_meta);
    for (uint32_t k = 0; k < p.n_meta; ++k) put_u32(mb + 4 + 4 * k, __float_as_uint(meta[(uint64_t)img * p.n_meta + k]));
    for (uint32_t s = 0; s < p.spc; ++s) {
      const uint32_t sz = 2u * words[(uint64_t)img * p.spc + s];
      put_u32(o + HDR_FIXED + 4 * s, sz);
      dst[(uint64_t)img * p.spc + s] = off;
      off += sz;
    }
    sizes[img] = off;
  }
}

__global__ void __launch_bounds__(128) k_copy(Plan p, const uint32_t* __restrict__ words,
                                              const uint16_t* __restrict__ scratch,
                                              const uint64_t* __restrict__ dst, uint8_t* __restrict__ out,
                                              uint64_t stride) {
  const uint32_t s = p.s_lo + blockIdx.x;
  uint32_t u, g;
  stream_info(p, s, u, g);
  const Unit un = unit_info(p, u);
  const uint32_t nr = min(p.G, un.h - g * p.G);
  const uint32_t nw = words[s], ns = 2 * nr, ne = nw - ns;
  const uint16_t* region = scratch + (uint64_t)s * p.cap_words;
  uint16_t* o = reinterpret_cast<uint16_t*>(out + (uint64_t)(un.img / p.depth) * stride + dst[s]);
  for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x)
    o[i] = i < ns ? region[i] : region[p.cap_words - ne + (i - ns)];
}

// ------------------------------------------------------------ table-driven rANS decode
// Parity tap for the coder alone: every pixel's full integer table is given
// (north_star "when the oracle is fed the same integer tables"), so groups are
// independent; one warp per stream mirrors k_rans_enc in decoder order.
__global__ void __launch_bounds__(128) k_rans_dec_tables(Plan p, const uint8_t* __restrict__ bits,
                                                         const uint32_t* __restrict__ sbase,
                                                         const uint32_t* __restrict__ slen,
                                                         const uint16_t* __restrict__ tables,
                                                         uint8_t* __restrict__ out, int32_t* __restrict__ status) {
  const uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (s >= p.n_img * p.spi) return;
  uint32_t u, g;
  stream_info(p, s, u, g);
  const Unit un = unit_info(p, u);
  const uint32_t r0 = g * p.G, nr = min(p.G, un.h - r0);
  const uint16_t* sw = reinterpret_cast<const uint16_t*>(bits + sbase[s]);
  const uint32_t sl = slen[s];
  const bool lane_ok = lane < nr;
  const int r = (int)(r0 + lane);
  int err = 0;
  uint32_t x = 0;
  if (lane_ok) {
    if (2 * lane + 1 < sl) x = ((uint32_t)sw[2 * lane] << 16) | sw[2 * lane + 1];
    else err = 8;
  }
  uint32_t cur = 2 * nr;
  const int t_hi = 3 * (int)(r0 + nr - 1) + (int)un.w - 1;
#pragma unroll 1
  for (int t = 3 * (int)r0; t <= t_hi; ++t) {
    const int c = t - 3 * r;
    const bool act = lane_ok && c >= 0 && c < (int)un.w;
    bool need = false;
    if (act) {
      const uint64_t gi = (uint64_t)un.img * p.W * p.H + (uint64_t)(un.y0 + r) * p.W + un.x0 + c;
      const uint16_t* tab = tables + gi * NOUT;
      const uint32_t slot = x & 0xFFFFu;
      uint32_t cum = 0, fsel = 0, csel = 0;
      int sym = 0;
      for (int i = 0; i < NOUT; ++i) {
        const uint32_t f = __ldg(tab + i);
        if (slot - cum < f) {
          sym = i;
          fsel = f;
          csel = cum;
        }
        cum += f;
      }
      if (cum != 65536u || fsel == 0) err = 9;
      x = fsel * (x >> 16) + slot - csel;
      need = x < RANS_L;
      out[gi] = (uint8_t)sym;
    }
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, need);
    if (need) {
      const uint32_t wi = cur + __popc(m & ((1u << lane) - 1u));
      if (wi < sl) x = (x << 16) | sw[wi];
      else err = 8;
    }
    cur += __popc(m);
  }
  if (lane_ok && x != RANS_L) err = err ? err : 6;
  if (lane == 0 && cur != sl) err = err ? err : 6;
  if (err) atomicMax(status + un.img / p.depth, err);
}

cudaError_t launch_rans_dec_tables(const Plan& p, const uint8_t* d_bits, const uint32_t* d_sbase,
                                   const uint32_t* d_slen, const uint16_t* d_tables, uint8_t* d_out,
                                   int32_t* d_status, cudaStream_t st) {
  const uint32_t ns = p.n_img * p.spi;  // == n_cont * spc
  k_rans_dec_tables<<<(ns + 3) / 4, 128, 0, st>>>(p, d_bits, d_sbase, d_slen, d_tables, d_out, d_status);
  return cudaGetLastError();
}

// ------------------------------------------------------------ decode prep
__device__ __forceinline__ uint32_t get_u32(const uint8_t* b) {
  return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
}
__device__ __forceinline__ uint32_t get_u16(const uint8_t* b) { return (uint32_t)b[0] | ((uint32_t)b[1] << 8); }

__global__ void k_dec_prep(Plan p, const uint8_t* __restrict__ bits, const uint64_t* __restrict__ cont_off,
                           const uint64_t* __restrict__ cont_len, uint32_t* __restrict__ sbase,
                           uint32_t* __restrict__ slen, int32_t* __restrict__ status, int check_numerics) {
  const uint32_t img = blockIdx.x * blockDim.x + threadIdx.x;  // container index
  if (img >= p.n_cont) return;
  const uint8_t* b = bits + cont_off[img];
  const uint64_t len = cont_len[img];  // required: every read below stays inside [b, b + len)
  int err = 0;
  if (len < HDR_FIXED || b[0] != 'D' || b[1] != 'L' || b[2] != 'I' || b[3] != 'C') err = 6;
  else if (b[4] != CONTAINER_VERSION || b[6] != (p.w3d ? 2 : 1) || b[7] != (p.bits == 12 ? 12 : 0) ||
           (check_numerics && get_u16(b + 22) != NUMERICS_REV))
    err = 5;
  else if (get_u32(b + 8) != p.W || get_u32(b + 12) != p.H || get_u16(b + 16) != p.hdr_tw ||
           get_u16(b + 18) != p.hdr_th || get_u16(b + 20) != p.G || b[5] != p.precision ||
           get_u32(b + 56) != p.spc || p.hdr_bytes > len || get_u32(b + HDR_FIXED + 4u * p.spc) != p.n_meta)
    err = 2;
  uint64_t off = p.hdr_bytes;
  for (uint32_t s = 0; s < p.spc; ++s) {
    uint32_t sz = err ? 0u : get_u32(b + HDR_FIXED + 4 * s);
    if ((sz & 1u) || off + sz > len) {
      err = 6;
      sz = 0;
    }
    sbase[(uint64_t)img * p.spc + s] = (uint32_t)off;
    slen[(uint64_t)img * p.spc + s] = err ? 0u : sz / 2;
    off += sz;
  }
  if (off != len && !err) err = 6;
  status[img] = err;
}

// ------------------------------------------------------------ decoder
// One cluster of nc CTAs per unit; slot S = rank*64 + row holds rows
// r = S (mod 64*nc) in turn.  A CTA has 16 row warps (the network, softmax and
// symbol search of its 64 slots, 8 threads per row, as the encoder) and one
// rANS warp (lane l owns the rANS lanes of CTA rows l and l + 32).
//
// (Warp 0 is the rANS warp, warps 1-16 the row warps.)
// Per front t, row warps: the two fresh taps -> network (layer 1 over
// the 76 older taps was issued during front t-1; the next front's older taps
// are gathered in an MMA wait) -> wait for the rANS warp's slots of front t ->
// softmax / Q1' / search -> the finder thread publishes the pixel (ring, the
// next CTA's halo via DSMEM, zero pads, HBM) and (f_s, c_s) for the rANS warp
// -> cluster barrier (the next front's layer-1 MMA is issued between its
// arrive and wait).
// rANS warp: apply front t-1's steps (state update, renormalisation words
// from registers prefetched a front earlier, one ballot per 32-row half, group
// cursors) -> start rows beginning at front t -> publish the slots x & 0xFFFF
// (named barrier 7: arrive) -> prefetch the words front t's steps may read ->
// cluster barrier.  Its work overlaps the row warps' network entirely.
constexpr int DEC_THREADS = NTHREADS + 32;

// bf16: one more warp (the 18th) only issues the network's MMAs (run_rest_ws)
// bf16: + the MMA issuer warp; streamed engines: + the weight producer warp
__host__ __device__ constexpr int dec_block(int prec) {
  return prec >= 2 ? DEC_THREADS + 64 : prec == 1 ? DEC_THREADS + 32 : DEC_THREADS;
}

template <int PREC, bool PROF, bool W3D>
__global__ void __launch_bounds__(dec_block(PREC), 1)
    k_decode(Plan p, DevWeights w, const uint8_t* __restrict__ bits, const uint64_t* __restrict__ cont_off,
             const uint32_t* __restrict__ sbase, const uint32_t* __restrict__ slen, uint8_t* __restrict__ out,
             int32_t* __restrict__ status, unsigned long long* __restrict__ prof, uint32_t* __restrict__ sync) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar[3];  // 0 MMA completion, 1 a_ready (16 row warps), 2 spare
  __shared__ uint32_t tslot;
  __shared__ uint32_t s_tick;   // 3D: this cluster's unit ticket (rank 0's copy is authoritative)
  __shared__ uint32_t s_lower;  // 3D: steps the slice below has published (a lower bound)
  __shared__ uint32_t s_slot[ROWS];  // the row's rANS slot x & 0xFFFF (rANS warp -> the row's 8 threads)
  __shared__ uint64_t s_sbar;        // DLIC_SLOT_MBAR: front t's slots published (phase t)
  __shared__ uint2 s_res[ROWS];      // (f_s, c_s) of the decoded symbol (finder -> rANS warp, next front)
  const uint32_t lane = lane_id();
  const uint32_t NC = p.nc, NS = ROWS * NC;
  const uint32_t ns_shift = 6u + (uint32_t)(__ffs((int)NC) - 1);
  // optional phase profile (thread 0 of each CTA), see Prof in dlic_device.cuh:
  // 0 top 1 gather 2 put 3 mlp 4 pass1 5 exchanges 6 pass2 7 passA 8 search 9 rans 10 barrier
  Prof pf;
  pf.on = PROF && threadIdx.x == DLIC_PROF_TID;  // a row thread
  const uint32_t rank = NC > 1 ? cluster_rank() : 0u;
  // Volumes (3D wavefront): the unit of slice z waits for the same
  // unit of slice z-1, so units are handed out in order through a ticket:
  // a cluster only ever waits for clusters that were dispatched before it.
  // sync[0] = ticket, sync[1 + u] = steps unit u has published.
  auto unit_of_cluster = [&]() -> uint32_t {
    if (!W3D) return blockIdx.x / NC;
    if (rank == 0 && threadIdx.x == 0) s_tick = atomicAdd(sync, 1u);
    if (NC > 1) {
      cluster_sync_all();
      uint32_t v;
      asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(map_cluster(smem_u32(&s_tick), 0)) : "memory");
      cluster_sync_all();  // rank 0's ticket read by every CTA before anyone moves on
      return v;
    }
    __syncthreads();
    return s_tick;
  };
  const uint32_t u = p.u_lo + unit_of_cluster();
  const Unit un = unit_info(p, u);
  const uint32_t DEPTH = W3D ? p.depth : 1u;  // images per container (2D: 1, compile-time)
  const int zsl = W3D ? (int)(un.img % DEPTH) : 0;  // slice index in its volume
  uint32_t* const my_done = W3D ? sync + 1 + u : nullptr;
  const uint32_t* const lower_done = W3D && zsl > 0 ? sync + 1 + (u - p.upi) : nullptr;
  if (W3D && threadIdx.x == 0) s_lower = 0;

  using Pix = PixT<PREC>;
  constexpr int BITS = pix_bits<PREC>();
  typename EngineSel<PREC>::T eng;
  Pix* ring = reinterpret_cast<Pix*>(engine_setup<PREC>(eng, smem, w, bar, &tslot, p.w3d));
  if constexpr (PREC == 1 || PREC == 4) eng.bar2 = smem_u32(&bar[2]);  // the decoder's logits halves (P350K: none, measured slower)
  if (w.b1img) {  // the unit's image's metadata-folded layer-1 bias
    if constexpr (PREC == 1) {
      __syncthreads();  // engine_setup's bias copy is complete
      float* b1 = const_cast<float*>(eng.bias);
      for (uint32_t i = threadIdx.x; i < (uint32_t)HID; i += blockDim.x) b1[i] = w.b1img[(uint64_t)(un.img / DEPTH) * HID + i];
    } else {
      eng.b0 = w.b1img + (uint64_t)(un.img / DEPTH) * HID;
    }
  }
  uint32_t* cursor = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(ring + RING_BYTES) + 16);  // 16 zero bytes after the ring
  uint32_t* s_sbase = cursor + ((un.ngroups + 3u) & ~3u);                   // per-group stream table
  uint32_t* s_slen = s_sbase + ((un.ngroups + 3u) & ~3u);
  uint32_t* s_t3 = s_slen + ((un.ngroups + 3u) & ~3u);  // W3D bf16: [2][ROWS][3]
  for (uint32_t i = threadIdx.x; i < RING_BYTES * sizeof(Pix) / 16; i += blockDim.x)
    reinterpret_cast<int4*>(ring)[i] = make_int4(0, 0, 0, 0);
  const uint32_t G = p.G;
  const uint32_t g_shift = (uint32_t)(__ffs((int)G) - 1);
  for (uint32_t g = threadIdx.x; g < un.ngroups; g += blockDim.x) {
    if ((((G * g) & (NS - 1)) >> 6) == rank) cursor[g] = 2u * min(G, un.h - G * g);
    s_sbase[g] = sbase[un.first_stream + g];
    s_slen[g] = slen[un.first_stream + g];
  }
  const uint32_t a_ready = smem_u32(&bar[1]);
  // named barrier 7 (16 row warps sync, the rANS warp arrives): slots ready
  if (threadIdx.x == 0) {
    mbar_init(a_ready, NTHREADS / 32);
    mbar_init(smem_u32(&bar[2]), 1);  // second MMA-completion barrier (DEC_NSPLIT)
    mbar_init(smem_u32(&s_sbar), 1);  // the rANS warp's lane 0, once per front
    fence_mbar_init();
  }
  if (NC > 1) cluster_sync_all();
  else __syncthreads();

  const uint8_t* cbase = bits + cont_off[un.img / DEPTH];
  const int uw = (int)un.w, uh = (int)un.h;
  const int T = uw + 3 * (uh - 1);
  int err = 0;
  // geometry of slot S at front t: row r (active if decoded on front t), column c
  auto slot_rc = [&](uint32_t S, int t, int& r, int& c) -> bool {
    const int rlo = t - uw + 1 > 0 ? (t - uw + 3) / 3 : 0;
    const int rhi = min(uh - 1, t / 3);
    r = 0;
    c = 0;
    if (rlo > rhi) return false;
    r = rlo + (int)((S + NS - ((uint32_t)rlo & (NS - 1))) & (NS - 1));
    c = t - 3 * r;
    return r <= rhi;
  };
  // 3D (bf16): the rANS warp loads the 3x3 box of the slice below for each of
  // its CTA's 64 slots one step ahead into s_t3[step & 1] (its own slack:
  // after publishing the step's slots), waiting first until the slice below
  // has published the steps it needs (its pixels up to 4 steps past the
  // slot's, stored one step after decoding: done >= step + 5).  L2 loads
  // (.cg): this SM may hold stale L1 lines of the slice below.
  const uint8_t* lower_img = out + (uint64_t)(un.img - (zsl > 0 ? 1u : 0u)) * p.W * p.H +
                             (uint64_t)un.y0 * p.W + un.x0;
  auto wait_lower = [&](int need) {
    if (!lower_done) return;
    for (long long spins = 0;; ++spins) {
      uint32_t v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(lower_done) : "memory");
      if ((int)v >= need) break;
      if (spins > (1ll << 26)) {  // watchdog: corrupt, never a hang
        err = 6;
        break;
      }
    }
  };
  auto lower_box = [&](int r, int c, bool act, uint32_t (&t)[3]) {
    t[0] = t[1] = t[2] = 0u;
    if (!lower_done || !act) return;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int rr = r + k / 3 - 1, cc = c + k % 3 - 1;
      const bool ok = rr >= 0 && rr < uh && cc >= 0 && cc < uw;
      const uint32_t v = ok ? (uint32_t)__ldcg(lower_img + (int64_t)rr * p.W + cc) : 0u;
      t[k >> 2] |= v << (8 * (k & 3));
    }
  };
  auto fill_t3 = [&](int t) {  // rANS warp: both 32-slot halves at step t
    wait_lower(t + 5);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      int r, c;
      const bool act = slot_rc(rank * ROWS + 32u * hf + lane, t, r, c);
      uint32_t tt[3];
      lower_box(r, c, act, tt);
      uint32_t* d = s_t3 + ((uint32_t)(t & 1) * ROWS + 32u * hf + lane) * 3u;
      d[0] = tt[0];
      d[1] = tt[1];
      d[2] = tt[2];
    }
  };
  if constexpr (W3D && PREC == 1) {
    if (threadIdx.x < 32) fill_t3(0);
    __syncthreads();
  }
  auto front_end = [&]() {
    if (NC > 1) cluster_sync_all();
    else __syncthreads();
  };

  if (threadIdx.x < 32) {
    // ======================================================= rANS warp
    // (warp 0: the lowest issue priority on its SMSP -- the scheduler favours
    // the highest warp id -- as its work has a whole front of slack)
    // Lanes of my group among the warp's lanes for one 32-row half: rows are
    // 32-aligned per pass, so a group is all active lanes of my pass parity
    // (G = 32) or a G-aligned lane range of them.
    auto group_mask = [&](bool act, uint32_t bk, uint32_t am, uint32_t bm) -> uint32_t {
      if (!act) return 0u;
      const uint32_t same = am & (bk ? bm : ~bm);
      return G >= 32 ? same : same & (((1u << G) - 1u) << (lane & ~(G - 1u)));
    };
    uint32_t xs[2] = {0u, 0u};                // states of CTA rows lane, lane + 32
    uint32_t pw[2][2] = {{0u, 0u}, {0u, 0u}};  // prefetched words [half][pass parity]
    uint32_t fl[2] = {0u, 0u}, cur[2] = {0u, 0u}, sl[2] = {0u, 0u};
    // apply the step of front t (rows of half hf): x' = f*(x>>16) + slot - c,
    // renormalised with words in decoder order within each group
    auto apply = [&](int hf, int t) {
      int r, c;
      const bool act = slot_rc(rank * ROWS + 32u * hf + lane, t, r, c);
      const uint32_t g = (uint32_t)r >> g_shift;
      const uint32_t bk = ((uint32_t)r >> ns_shift) & 1u;
      bool need = false;
      uint32_t x = xs[hf];
      if (act) {
        const uint2 fc = s_res[32 * hf + lane];  // written by the thread that found the symbol
        x = fc.x * (x >> 16) + (x & 0xFFFFu) - fc.y;
        need = x < RANS_L;
      }
      const uint32_t am = __ballot_sync(0xFFFFFFFFu, act);
      const uint32_t bm = __ballot_sync(0xFFFFFFFFu, bk != 0);
      const uint32_t nm = __ballot_sync(0xFFFFFFFFu, need);
      const uint32_t gm = group_mask(act, bk, am, bm);
      const uint32_t readers = nm & gm;
      const uint32_t rk = __popc(readers & ((1u << lane) - 1u));
      const uint32_t src = G == 32 ? rk : (fl[hf] + rk) & 31u;
      const uint32_t w0 = __shfl_sync(0xFFFFFFFFu, pw[hf][0], src);
      const uint32_t w1 = __shfl_sync(0xFFFFFFFFu, pw[hf][1], src);
      if (need) {
        if (cur[hf] + rk < sl[hf]) x = (x << 16) | (G == 32 && bk == 1 ? w1 : w0);
        else err = 8;
      }
      if (act && lane == (uint32_t)(__ffs(gm) - 1)) cursor[g] = cur[hf] + __popc(readers);
      if (act && c == uw - 1 && x != RANS_L) err = 6;  // end-of-lane invariant
      xs[hf] = x;
    };
    // prefetch the words the steps of front t may read (registers; the L2
    // latency hides behind a whole front -- the cluster barrier invalidates L1)
    //  G = 32: lanes hold words cur..cur+31 of the group of each pass parity
    //  G < 32: each lane holds the word it reads if every earlier row of its
    //          group reads one
    auto prefetch = [&](int hf, int t) {
      int r, c;
      const bool act = slot_rc(rank * ROWS + 32u * hf + lane, t, r, c);
      const uint32_t g = (uint32_t)r >> g_shift;
      const uint32_t bk = ((uint32_t)r >> ns_shift) & 1u;
      uint32_t sb = 0;
      sl[hf] = 0;
      cur[hf] = 0;
      pw[hf][0] = pw[hf][1] = 0;
      if (act) {
        sb = s_sbase[g];
        sl[hf] = s_slen[g];
        cur[hf] = cursor[g];
      }
      const uint32_t am = __ballot_sync(0xFFFFFFFFu, act);
      const uint32_t bm = __ballot_sync(0xFFFFFFFFu, bk != 0);
      if (G == 32) {
#pragma unroll
        for (uint32_t b = 0; b < 2; ++b) {
          const uint32_t mb = am & (b ? bm : ~bm);
          if (mb) {
            const uint32_t s0 = (uint32_t)__ffs(mb) - 1u;
            const uint32_t sbb = __shfl_sync(0xFFFFFFFFu, sb, s0);
            const uint32_t slb = __shfl_sync(0xFFFFFFFFu, sl[hf], s0);
            const uint32_t cub = __shfl_sync(0xFFFFFFFFu, cur[hf], s0);
            const uint16_t* swb = reinterpret_cast<const uint16_t*>(cbase + sbb);
            const uint32_t idx = cub + lane;
            pw[hf][b] = idx < slb ? (uint32_t)__ldg(swb + idx) : 0u;
          }
        }
      } else {
        const uint32_t gm = group_mask(act, bk, am, bm);
        fl[hf] = gm ? (uint32_t)__ffs(gm) - 1u : lane;
        const uint32_t idx = cur[hf] + (lane - fl[hf]);
        const uint16_t* swm = reinterpret_cast<const uint16_t*>(cbase + sb);
        pw[hf][0] = (act && idx < sl[hf]) ? (uint32_t)__ldg(swm + idx) : 0u;
      }
    };
#pragma unroll 1
    for (int t = 0; t < T; ++t) {
      if (t > 0) {
        // the words front t-1's steps may read: loaded here, after the
        // barrier (the L2 latency is in this warp's slack, not in its arrive)
        prefetch(0, t - 1);
        prefetch(1, t - 1);
        __syncwarp();  // cursor reads before apply's cursor updates
        apply(0, t - 1);
        apply(1, t - 1);
        __syncwarp();  // cursor updates before the prefetch reads them
      }
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {  // rows starting at front t: flushed state (hi, lo)
        int r, c;
        if (slot_rc(rank * ROWS + 32u * hf + lane, t, r, c) && c == 0) {
          const uint32_t g = (uint32_t)r >> g_shift;
          const uint16_t* sw = reinterpret_cast<const uint16_t*>(cbase + s_sbase[g]);
          const uint32_t i = 2u * ((uint32_t)r - G * g);
          if (i + 1 < s_slen[g]) xs[hf] = ((uint32_t)__ldg(sw + i) << 16) | (uint32_t)__ldg(sw + i + 1);
          else err = 8;
        }
        s_slot[32 * hf + lane] = xs[hf] & 0xFFFFu;
      }
      if constexpr (DLIC_SLOT_MBAR && PREC != 3) {  // slots of front t published (12-bit: named barrier 7)
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&s_sbar));
      } else {
        asm volatile("bar.arrive 7, %0;" ::"n"(DEC_THREADS) : "memory");
      }
      if constexpr (W3D && PREC == 1) {
        if (t + 1 < T) fill_t3(t + 1);
      }
      front_end();
      if (W3D && lane == 0) {
        // the cluster barrier released every pixel store of steps <= t - 1
        // (each is stored in the step after it is decoded): publish them
        if (rank == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(my_done), "r"((uint32_t)t) : "memory");
        if (PREC == 0 && lower_done) {  // fp32: progress of the slice below, for the row warps
          uint32_t v;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(lower_done) : "memory");
          *(volatile uint32_t*)&s_lower = v;
        }
      }
    }
    if (T > 0) {  // the last front's steps
      prefetch(0, T - 1);
      prefetch(1, T - 1);
      __syncwarp();
      apply(0, T - 1);
      apply(1, T - 1);
    }
    __syncthreads();  // (1) cursors final
  } else if (PREC >= 2 && threadIdx.x >= DEC_THREADS + 32) {
    // ======================================================= weight-stream producer warp
    // the chunks of every front this CTA has an active row on, in the
    // issuer's order: front t's rest after barrier t-1, then up to S-1 chunks
    // of front t+1 before barrier t (they only need front t's last stages,
    // whose MMAs complete on their own)
    if constexpr (PREC >= 2) {
      auto any_t = [&](int t) -> bool {  // (as the issuer's)
        const int rlo = t - uw + 1 > 0 ? (t - uw + 3) / 3 : 0;
        const int rhi = min(uh - 1, t / 3);
        if (rlo > rhi) return false;
        const uint32_t m = (uint32_t)rlo & (NS - 1), b = rank * ROWS;
        const uint32_t d = m - b < (uint32_t)ROWS ? 0u : ((b - m) & (NS - 1));
        return rlo + (int)d <= rhi;
      };
      constexpr int CPN = EngineSel<PREC>::T::CPN;
      constexpr int LA = EngineSel<PREC>::T::S - 1 < CPN ? EngineSel<PREC>::T::S - 1 : CPN;
      if (any_t(0))
        for (int k = 0; k < CPN; ++k) eng.produce_one(k);
#pragma unroll 1
      for (int t = 0; t < T; ++t) {
        const bool an = any_t(t + 1);
        int done = 0;
        if (an)
          for (; done < LA; ++done) eng.produce_one(done);
        if (NC > 1) {
          cluster_arrive_relaxed();
          cluster_wait();
        } else {
          __syncthreads();
        }
        if (an)
          for (int k = done; k < CPN; ++k) eng.produce_one(k);
      }
    }
    __syncthreads();  // (1) cursors final
  } else if (PREC >= 1 && threadIdx.x >= DEC_THREADS) {
    // ======================================================= MMA issuer warp (bf16)
    if constexpr (PREC >= 1) {
      uint32_t aph = 0;
      auto any_t = [&](int t) -> bool {  // does any slot of this CTA hold an active row at front t
        const int rlo = t - uw + 1 > 0 ? (t - uw + 3) / 3 : 0;
        const int rhi = min(uh - 1, t / 3);
        if (rlo > rhi) return false;
        const uint32_t m = (uint32_t)rlo & (NS - 1), b = rank * ROWS;
        const uint32_t d = m - b < (uint32_t)ROWS ? 0u : ((b - m) & (NS - 1));
        return rlo + (int)d <= rhi;
      };
      // layer 1 of front t over the 76 early taps, once every row warp has
      // written them and loaded the previous logits (a_ready)
      auto issue_l0 = [&](bool a) {
        if (a) {
          mbar_wait(a_ready, aph);
          if constexpr (PREC >= 2) {
            eng.issue_l0();
          } else {
            eng.issue_slices(0, 0, KPAD / 16, TcEngine::dcol_of(0));
            eng.commit_both();
          }
        }
        aph ^= 1u;  // every row warp arrives once per front
      };
      issue_l0(any_t(0));
      unsigned long long ip[3] = {0, 0, 0};  // PROF: network issue, arrive->l0, l0->wait done
#pragma unroll 1
      for (int t = 0; t < T; ++t) {
        const long long i0 = PROF ? clock64() : 0;
        if (any_t(t)) {
          if constexpr (PREC >= 2) eng.issue_network();
          else eng.dec_issue_network();
        }
        const bool an = any_t(t + 1);
        const long long i1 = PROF ? clock64() : 0;
        long long i2 = 0;
        if (NC > 1) {
          if constexpr (PREC >= 2) cluster_arrive_relaxed();
          else cluster_arrive();
          issue_l0(an);
          if (PROF) i2 = clock64();
          cluster_wait();
        } else {
          issue_l0(an);
          if (PROF) i2 = clock64();
          __syncthreads();
        }
        if (PROF) {
          ip[0] += i1 - i0;
          ip[1] += i2 - i1;
          ip[2] += clock64() - i2;
        }
      }
      if (PROF && lane == 0) {
        atomicAdd(prof + 26, ip[0]);
        atomicAdd(prof + 27, ip[1]);
        atomicAdd(prof + 28, ip[2]);
      }
    }
    __syncthreads();  // (1) cursors final
  } else {
    // ======================================================= row warps
    const int row = tile_row();
    const uint32_t S = rank * ROWS + (uint32_t)row;
    Pix* oimg = reinterpret_cast<Pix*>(out) + (uint64_t)un.img * p.W * p.H + (uint64_t)un.y0 * p.W + un.x0;
    const uint32_t ring_s = smem_u32(ring);
    const uint32_t halo_base = NC > 1 ? map_cluster(ring_s, (rank + 1) % NC) : ring_s;
    const uint32_t halo_flip = rank == NC - 1 ? 1u : 0u;  // wrap-around halo feeds the next pass
    // gather: thread u = 2j + h reads window row dr = u - 8 at ringrow row + u
    // and (u < 6) the target-row tap dc = u - 6 at ringrow row + 8 (kpos_tap)
    const int gu = 2 * col_grp() + half_id();
    const int g9 = gu < 6 ? (8 - gu) + (gu - 6) * RING_ROWS : 0;
    int pix = 0;
    // ring base of slot (r, c): window cell (dr, dc) of the K order at
    // bp + (dc)*RING_ROWS for dr = u - 8, tap 9 at bp + g9 (see the ring notes)
    auto ring_at = [&](int r, int c) -> const Pix* {
      const uint32_t col = (uint32_t)c & 31u;
      const uint32_t cb = col < 6u ? col + 32u : col;
      return ring + (((uint32_t)r >> ns_shift) & 1u) * RING_BANK + cb * RING_ROWS + (uint32_t)row;
    };
    // Early part of a front (one front ahead): the 76 taps decoded before the
    // preceding front -> layer-1 input (the two fresh taps' weights are zero in
    // the MMA image; fp32: overwritten by run_rest).
    // 3D window: the 3x3 box of the slice below for the next step's pixel,
    // loaded in that step's predecessor (layer-3 MMA wait) once the slice
    // below has published the steps it needs (its pixels up to step t+5 of
    // this slice's clock: the box reaches (r+1, c+1), 4 steps after (r, c);
    // pixels are stored one step after they are decoded).  L2 loads (.cg):
    // this SM may hold stale L1 lines of the slice below.
    uint32_t t3[3] = {0u, 0u, 0u}, t3n[3] = {0u, 0u, 0u};
    auto load_lower = [&](int rn, int cn, bool act, int need) {  // fp32 engine: the row warps load directly
      t3n[0] = t3n[1] = t3n[2] = 0u;
      if (!lower_done || !act) return;
      if ((int)*(volatile uint32_t*)&s_lower < need) {
        const long long w0 = PROF ? clock64() : 0;
        if (PROF && pf.on) atomicAdd(prof + 24, 1ull);  // waits (profiled thread)
        for (long long spins = 0;; ++spins) {
          uint32_t v;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(lower_done) : "memory");
          if ((int)v >= need) {
            if (PROF && pf.on) atomicAdd(prof + 25, (unsigned long long)(clock64() - w0));
            break;
          }
          if (spins > (1ll << 26)) {  // watchdog: corrupt, never a hang
            err = 6;
            break;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const int rr = rn + k / 3 - 1, cc = cn + k % 3 - 1;
        const bool ok = rr >= 0 && rr < uh && cc >= 0 && cc < uw;
        const uint32_t v = ok ? (uint32_t)__ldcg(lower_img + (int64_t)rr * p.W + cc) : 0u;
        t3n[k >> 2] |= v << (8 * (k & 3));
      }
    };
    auto early_put = [&](int r, int c) {
      const Pix* bp = ring_at(r, c) + gu;
      uint32_t tv[10];
#pragma unroll
      for (int i = 0; i < 9; ++i) tv[i] = bp[(i - 6) * RING_ROWS];
      tv[9] = bp[g9];
      if constexpr (PREC >= 1) {
        const f2 m1 = f2_make(-1.0f, -1.0f);
        uint32_t a[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          float x0, x1;
          f2_split(f2_add(f2_bits(0x3F800000u | (tv[2 * q] << (23 - BITS)), 0x3F800000u | (tv[2 * q + 1] << (23 - BITS))),
                          m1),
                   x0, x1);
          a[q] = pack_bf16(x0, x1);
        }
        eng.put_input(a);
      } else {
#pragma unroll
        for (int i = 0; i < 10; ++i)
          if (i < 9 || gu < 6) eng.put_input(i < 9 ? 9 * gu + i : 72 + gu, u8_unit(tv[i]));
        if (W3D) {  // the lower-layer taps enter the fp32 network as inputs 78..86
          eng.put_input(KIN + gu, u8_unit((t3n[gu >> 2] >> (8 * (gu & 3))) & 0xFFu));
          if (gu == 0) eng.put_input(KIN + 8, u8_unit(t3n[2] & 0xFFu));
        }
      }
    };
    // does any slot of this CTA hold an active row at front t (uniform)
    auto cta_any = [&](int t) -> bool {
      const int rlo = t - uw + 1 > 0 ? (t - uw + 3) / 3 : 0;
      const int rhi = min(uh - 1, t / 3);
      if (rlo > rhi) return false;
      const uint32_t m = (uint32_t)rlo & (NS - 1), b = rank * ROWS;
      const uint32_t d = m - b < (uint32_t)ROWS ? 0u : ((b - m) & (NS - 1));
      return rlo + (int)d <= rhi;
    };
    // early part of front t+1 once this thread is done with the network's
    // output of front t: gather -> layer-1 input; each warp then arrives on
    // a_ready, which the MMA issuer waits on before issuing layer 1
    // (issue_early).  bf16: the layer-1 input has its own TMEM columns
    // (TM_A0), so the gather runs during the network; the signal only has to
    // follow this thread's load of the logits (the MMA overwrites them).
    // fp32: the input shares the logits buffer.
    auto early_gather = [&](int rn, int cn) {
      if constexpr (PREC >= 1) early_put(rn, cn);
    };
    auto early_signal = [&](int rn, int cn) {
      if constexpr (PREC >= 1) {
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_ready);
      } else {
        quad_sync();  // the row's logits are loaded: its buffer columns are free
        early_put(rn, cn);
      }
    };
    auto issue_early = [&](bool) {};  // bf16: the issuer warp issues layer 1

    // Front range [rlo, rhi] of active rows, kept incrementally (no
    // divisions): t = 3*q3 + m3, W = 3*qw + mw, rhi = min(H-1, q3),
    // rlo = t >= W-1 ? q3 - qw + 1 - (m3 < mw) : 0 = ceil((t - W + 1) / 3).
    const int qw = uw / 3, mw = uw - 3 * (uw / 3);
    int q3 = 0, m3 = 0;  // of front t + 1 inside the loop
    auto range = [&](int t, int q, int m, int& rlo, int& rhi) {
      rhi = min(uh - 1, q);
      rlo = t >= uw - 1 ? q - qw + 1 - (m < mw ? 1 : 0) : 0;
    };
    auto slot_at = [&](int t, int rlo, int rhi, int& r, int& c) -> bool {
      r = 0;
      c = 0;
      if (rlo > rhi) return false;
      r = rlo + (int)((S + NS - ((uint32_t)rlo & (NS - 1))) & (NS - 1));
      c = t - 3 * r;
      return r <= rhi;
    };
    auto any_at = [&](int rlo, int rhi) -> bool {
      if (rlo > rhi) return false;
      const uint32_t m = (uint32_t)rlo & (NS - 1), b = rank * ROWS;
      const uint32_t d = m - b < (uint32_t)ROWS ? 0u : ((b - m) & (NS - 1));
      return rlo + (int)d <= rhi;
    };
    int r, c;
    bool active = slot_rc(S, 0, r, c);
    bool any = cta_any(0);
    if constexpr (W3D && PREC == 0) {  // step 0's lower taps (later steps load theirs a step ahead)
      load_lower(r, c, active, 5);
      t3[0] = t3n[0];
      t3[1] = t3n[1];
      t3[2] = t3n[2];
    }
    early_gather(r, c);
    early_signal(r, c);
    issue_early(any);
    // front t+1 (used by front t's early gather); advanced in the end-of-front
    // barrier window, off the critical path
    int rn, cn;
    bool active_n, any_n;
    {
      int rlo, rhi;
      if (++m3 == 3) {
        m3 = 0;
        ++q3;
      }
      range(1, q3, m3, rlo, rhi);
      active_n = slot_at(1, rlo, rhi, rn, cn);
      any_n = any_at(rlo, rhi);
    }
    uint32_t fpo = (uint32_t)(ring_at(r, c) - ring) + 8u;  // the front's fresh-tap ring position
    Pix* optr = nullptr;  // deferred pixel store
    int opix = 0;
    if (pf.on) pf.t = clock64();
#pragma unroll 1
    for (int t = 0; t < T; ++t) {
      bool pub = false;
      pf.mark(0);
      if (any) {
        // the fresh taps (0,-1) and (-1,+2), decoded on front t-1
        const Pix* fp = ring + fpo;
        const float xa = fresh_in<PREC>(fp[-RING_ROWS]);
        const float xb = fresh_in<PREC>(fp[2 * RING_ROWS - 1]);
        pf.mark(1);
        // network; the previous front's pixel goes to HBM in the layer-2 MMA
        // wait, the next front's early gather in the layer-3 MMA wait
        if constexpr (PREC >= 1) {
          eng.run_rest_ws(xa, xb, [&](int l) {
            if (l == 1 && optr) *optr = (Pix)opix;
            if (l == 2) early_gather(rn, cn);
          }, [&](auto& bq) {
            if constexpr (W3D && PREC == 1) {  // this step's lower taps (s_t3, written by the rANS warp last step)
              const uint32_t* q = s_t3 + ((uint32_t)(t & 1) * ROWS + (uint32_t)row) * 3u;
              const uint32_t tt[3] = {q[0], q[1], q[2]};
              add_w3d(eng.bias, tt, bq);
            }
          });
        } else {
          eng.run_rest(xa, xb, [&](int l) {
            if (l == 1 && optr) *optr = (Pix)opix;
            if constexpr (W3D) { if (l == 2) load_lower(rn, cn, active_n, t + 6); }
          }, PROF ? &pf : nullptr);
        }
        pf.mark(3);
        // this front's slot of my row (the rANS warp's): DLIC_SLOT_MBAR waits
        // for it only at the symbol search, so the column groups whose
        // logits land first start their softmax at once
        auto my_slot = [&]() -> uint32_t {
          if constexpr (DLIC_SLOT_MBAR && PREC != 3) mbar_wait(smem_u32(&s_sbar), (uint32_t)t & 1u);
          return s_slot[row];
        };
        if (!DLIC_SLOT_MBAR || PREC == 3) asm volatile("bar.sync 7, %0;" ::"n"(DEC_THREADS) : "memory");
        pf.mark(6);  // profile: time spent waiting for the rANS warp's slots
        uint32_t fs, cs;
        bool mine;
        int sym;
        if constexpr (PREC == 3) sym = q12_row<false>(eng, my_slot(), mine, fs, cs, [&]() { early_signal(rn, cn); });
        else sym = q1_decode(eng, my_slot, mine, fs, cs, [&]() { early_signal(rn, cn); }, &pf);
        // the thread that found the symbol publishes it: own ring, the
        // successor's halo through DSMEM for the CTA's last 8 rows, zero
        // pads, and (f_s, c_s) for the rANS warp (applied next front)
        pub = mine && active;
        pix = sym;
        if (pub) {
          s_res[row] = make_uint2(fs, cs);
          const uint32_t bank = ((uint32_t)r >> ns_shift) & 1u;
          const uint32_t col = (uint32_t)c & 31u;
          Pix* rp = ring + (uint32_t)row + 8u;
          rp[bank * RING_BANK + col * RING_ROWS] = (Pix)sym;
          if (col < 8u) rp[bank * RING_BANK + (col + 32u) * RING_ROWS] = (Pix)sym;
          const bool halo = row >= ROWS - 8;
          const uint32_t hb = bank ^ halo_flip;
          const uint32_t hrow = (uint32_t)(row - (ROWS - 8));
          auto hput = [&](uint32_t b, uint32_t pos, uint32_t v) {
            const uint32_t off = b * RING_BANK + pos * RING_ROWS + hrow;
            if (NC > 1) {
              if constexpr (sizeof(Pix) == 2) st_cluster_u16(halo_base + 2u * off, v);
              else st_cluster_u8(halo_base + off, v);
            } else {
              ring[off] = (Pix)v;
            }
          };
          if (halo) {
            hput(hb, col, (uint32_t)sym);
            if (col < 8u) hput(hb, col + 32u, (uint32_t)sym);
          }
          if (c == uw - 1) {  // row end: right pad (columns W, W+1) of this row
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const uint32_t pc = (uint32_t)(uw + e) & 31u;
              rp[bank * RING_BANK + pc * RING_ROWS] = 0;
              if (pc < 8u) rp[bank * RING_BANK + (pc + 32u) * RING_ROWS] = 0;
              if (halo) {
                hput(hb, pc, 0u);
                if (pc < 8u) hput(hb, pc + 32u, 0u);
              }
            }
          }
          // left pad (pos 26..31) of the slot's next row, in the other bank:
          // after the previous occupant's readers are done (front 3r + 23 at
          // the latest, W <= 3*NS) and well before the next row's early gather
          if (c == min(24, uw - 1)) {
#pragma unroll
            for (uint32_t pc = 26; pc < 32; ++pc) {
              rp[(bank ^ 1u) * RING_BANK + pc * RING_ROWS] = 0;
              if (halo) hput(hb ^ 1u, pc, 0u);
            }
          }
        }
        pf.mark(9);
      } else {
        if (!DLIC_SLOT_MBAR || PREC == 3) asm volatile("bar.sync 7, %0;" ::"n"(DEC_THREADS) : "memory");  // in step
        if (optr) *optr = (Pix)opix;
        if constexpr (W3D && PREC == 0) load_lower(rn, cn, active_n, t + 6);
        early_gather(rn, cn);
        early_signal(rn, cn);
      }
      // end-of-front barrier; the next front's layer-1 MMA is issued between
      // its arrive and wait.  (A point-to-point variant -- halo writers
      // arriving remotely on a successor mbarrier -- measured slower.)
      int rn2, cn2;
      bool active_n2, any_n2;
      uint32_t fpo_n;
      if (NC > 1) {
        cluster_arrive();
        issue_early(any_n);
        fpo_n = (uint32_t)(ring_at(rn, cn) - ring) + 8u;
        {  // front t+2's geometry while the cluster arrives
          int rlo, rhi;
          if (++m3 == 3) {
            m3 = 0;
            ++q3;
          }
          range(t + 2, q3, m3, rlo, rhi);
          active_n2 = slot_at(t + 2, rlo, rhi, rn2, cn2);
          any_n2 = any_at(rlo, rhi);
        }
        cluster_wait();
      } else {
        issue_early(any_n);
        fpo_n = (uint32_t)(ring_at(rn, cn) - ring) + 8u;
        int rlo, rhi;
        if (++m3 == 3) {
          m3 = 0;
          ++q3;
        }
        range(t + 2, q3, m3, rlo, rhi);
        active_n2 = slot_at(t + 2, rlo, rhi, rn2, cn2);
        any_n2 = any_at(rlo, rhi);
        __syncthreads();
      }
      // the pixel's HBM store: issued in the next front's layer-2 MMA wait (off
      // the post-barrier critical path; the barrier's release never waits for it)
      optr = pub ? oimg + (uint64_t)r * p.W + c : nullptr;
      opix = pix;
      pf.mark(10);
      r = rn;
      c = cn;
      active = active_n;
      any = any_n;
      t3[0] = t3n[0];
      t3[1] = t3n[1];
      t3[2] = t3n[2];
      rn = rn2;
      cn = cn2;
      active_n = active_n2;
      any_n = any_n2;
      fpo = fpo_n;
    }
    if (optr) *optr = (Pix)opix;  // the last front's pixel
    __syncthreads();  // (1) cursors final
  }
  if (pf.on) {
    for (int kk = 0; kk < 11; ++kk) atomicAdd(prof + kk, pf.acc[kk]);
    for (int kk = 0; kk < 4; ++kk) atomicAdd(prof + 16 + kk, pf.acc2[kk]);
  }
  for (uint32_t g = threadIdx.x; g < un.ngroups; g += blockDim.x) {
    if ((((G * g) & (NS - 1)) >> 6) == rank && cursor[g] != slen[un.first_stream + g]) err = 6;
  }
  if (err) atomicMax(status + un.img / DEPTH, err);
  engine_teardown<PREC>(eng);
  if (NC > 1) cluster_sync_all();  // keep DSMEM alive until every CTA is done
  else if (W3D) __syncthreads();
  if (W3D && rank == 0 && threadIdx.x == 0)  // every pixel of the unit is stored (the barrier released them)
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(my_done), "r"(0x7FFFFFFFu) : "memory");
}

// ------------------------------------------------------------ metadata -> layer-1 bias
// One thread per (image, hidden unit): out = b1 + sum_k m'_k W1[78 + k] (see
// dlic_internal.h); the per-image constant part of layer 1 (P:210 metadata
// features are the same for every pixel of an image).
__device__ __forceinline__ float bf16_rn(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__global__ void k_meta_bias(uint32_t n_img, uint32_t n_meta, const float* __restrict__ meta,
                            const uint8_t* __restrict__ bits, const uint64_t* __restrict__ cont_off,
                            uint32_t meta_off, const float* __restrict__ range, const float* __restrict__ wmeta,
                            const float* __restrict__ b1, uint32_t precision, float* __restrict__ out) {
  const uint32_t i = blockIdx.x, n = threadIdx.x;
  if (i >= n_img || n >= (uint32_t)HID) return;
  float acc = 0.0f;
  for (uint32_t k = 0; k < n_meta; ++k) {
    const float lo = range[2 * k], hi = range[2 * k + 1];
    // raw real: from the host-supplied array (encode) or re-read from the
    // container's metadata block (decode)
    const float raw = bits ? __uint_as_float(get_u32(bits + cont_off[i] + meta_off + 4u * k))
                           : meta[(uint64_t)i * n_meta + k];
    const float m = __fdiv_rn(__fsub_rn(raw, lo), __fsub_rn(hi, lo));
    const float wv = wmeta[k * HID + n];
    if (precision == 1) acc = __fadd_rn(acc, __fmul_rn(bf16_rn(m), bf16_rn(wv)));  // exact product
    else acc = __fmaf_rn(m, wv, acc);
  }
  out[(uint64_t)i * HID + n] = __fadd_rn(b1[n], acc);
}

cudaError_t launch_meta_bias(uint32_t n_img, uint32_t n_meta, const float* d_meta, const uint8_t* d_bits,
                             const uint64_t* d_cont_off, uint32_t meta_off, const float* d_range,
                             const float* d_wmeta, const float* d_b1, uint32_t precision, float* d_out,
                             cudaStream_t st) {
  k_meta_bias<<<n_img, HID, 0, st>>>(n_img, n_meta, d_meta, d_bits, d_cont_off, meta_off, d_range, d_wmeta, d_b1,
                                     precision, d_out);
  return cudaGetLastError();
}

// ------------------------------------------------------------ launchers
template <class K>
static cudaError_t set_smem(K kern, size_t bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

cudaError_t launch_enc_mlp(const Plan& p, const DevWeights& w, const uint8_t* d_imgs, uint32_t* d_fc,
                           float* dbg_logits, float* dbg_probs, uint16_t* dbg_freqs, cudaStream_t st,
                           int num_sms) {
  const uint64_t total = (uint64_t)p.u_cnt * p.tiles_per_unit;
  const uint32_t grid = (uint32_t)(total < (uint64_t)num_sms ? total : (uint64_t)num_sms);
  const size_t sm = enc_smem_bytes(p.engine, p.w3d);
  if (p.engine >= 2) {  // P350K / P12: streamed weights, one tile chain per CTA (+ debug exports)
    auto kern = p.engine == 4 ? k_enc_mlp<4> : p.engine == 3 ? k_enc_mlp<3> : k_enc_mlp<2>;
    cudaError_t e = set_smem(kern, sm);
    if (e != cudaSuccess) return e;
    const bool prof = getenv("DLIC_PROF_STREAM") != nullptr;
    Plan pp = p;
    if (prof) {
      pp.prof = 1u | (uint32_t)atoi(getenv("DLIC_PROF_STREAM"));
      unsigned long long z[8] = {};
      cudaMemcpyToSymbolAsync(g_sprof, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
    }
    kern<<<grid, enc_block(p.engine), sm, st>>>(pp, w, d_imgs, d_fc, dbg_logits, dbg_probs, dbg_freqs);
    if (prof) {
      unsigned long long h[8];
      cudaMemcpyFromSymbolAsync(h, g_sprof, sizeof(h), 0, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const double ns = (double)h[4], cpn = p.engine == 4 ? TcX3::CPN : p.engine == 3 ? CH_NET12 : CH_NET;
      fprintf(stderr, "[stream prof] per chunk (issuer, cycles): data wait %.0f  stage wait %.0f  epilogue wait %.0f  "
              "total %.0f  (chunks %llu) | per tile (row thread 0): feed %.0f network %.0f q1 %.0f\n", h[0] / ns,
              h[1] / ns, h[2] / ns, h[3] / ns, h[4], h[5] / (ns / cpn), h[6] / (ns / cpn), h[7] / (ns / cpn));
    }
  } else if (p.engine == 1 && (dbg_logits || dbg_probs || dbg_freqs)) {
    // parity tap: the production kernel with its debug exports
    const size_t sp = enc_pp_smem_bytes(p.w3d);
    auto k = p.w3d ? k_enc_pp<true, true> : k_enc_pp<true, false>;
    cudaError_t e = set_smem(k, sp);
    if (e != cudaSuccess) return e;
    k<<<grid, ENC_PP_THREADS, sp, st>>>(p, w, d_imgs, d_fc, nullptr, dbg_logits, dbg_probs, dbg_freqs);
  } else if (p.engine == 1) {
    const size_t sp = enc_pp_smem_bytes(p.w3d);
    auto kp = p.w3d ? k_enc_pp<false, true> : k_enc_pp<false, false>;
    cudaError_t e = set_smem(kp, sp);
    if (e != cudaSuccess) return e;
    static unsigned long long* d_prof = nullptr;
    const bool prof = getenv("DLIC_PROF_ENC") != nullptr;
    if (prof && !d_prof) cudaMalloc(&d_prof, 16 * 8);
    if (prof) cudaMemsetAsync(d_prof, 0, 16 * 8, st);
    kp<<<grid, ENC_PP_THREADS, sp, st>>>(p, w, d_imgs, d_fc, prof ? d_prof : nullptr, nullptr, nullptr, nullptr);
    if (prof) {
      unsigned long long h[16];
      cudaMemcpyAsync(h, d_prof, 16 * 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const double np = (double)h[10];
      fprintf(stderr, "[enc prof] cycles per pair (thread 0): layer0 %.0f a-logits %.0f finish-a %.0f feed-a %.0f "
              "b-logits+feed-b %.0f finish-b %.0f | layers1-4 (8 epilogues): bias %.0f mma-wait %.0f epilogue %.0f "
              "signal %.0f | issuer: total %.0f waiting for b %.0f\n", h[0] / np, h[1] / np,
              h[2] / np, h[3] / np, h[4] / np, h[5] / np, h[6] / np, h[7] / np, h[11] / np, h[12] / np, h[9] / np,
              h[8] / np);
    }
  } else {
    cudaError_t e = set_smem(k_enc_mlp<0>, sm);
    if (e != cudaSuccess) return e;
    k_enc_mlp<0><<<grid, NTHREADS, sm, st>>>(p, w, d_imgs, d_fc, dbg_logits, dbg_probs, dbg_freqs);
  }
  return cudaGetLastError();
}

cudaError_t launch_rans_enc(const Plan& p, const uint32_t* d_fc, uint16_t* d_scratch, uint32_t* d_words,
                            cudaStream_t st) {
  if (p.s_cnt == 0) return cudaSuccess;
  k_rans_enc<<<(p.s_cnt + 3) / 4, 128, 0, st>>>(p, d_fc, d_scratch, d_words);
  return cudaGetLastError();
}

cudaError_t launch_container(const Plan& p, const uint8_t* model_sha, const uint32_t* d_words,
                             const uint16_t* d_scratch, uint8_t* d_out, uint64_t out_stride, uint64_t* d_sizes,
                             uint64_t* d_stream_dst, cudaStream_t st, bool payload_only, const float* d_meta) {
  Sha sha;
  for (int i = 0; i < 32; ++i) sha.b[i] = model_sha ? model_sha[i] : 0;
  k_container<<<payload_only ? 1u : p.n_cont, 32, 0, st>>>(p, sha, d_words, d_out, out_stride, d_sizes,
                                                           d_stream_dst, payload_only ? 1 : 0, d_meta);
  if (p.s_cnt > 0) k_copy<<<p.s_cnt, 128, 0, st>>>(p, d_words, d_scratch, d_stream_dst, d_out, out_stride);
  return cudaGetLastError();
}

cudaError_t launch_dec_prep(const Plan& p, const uint8_t* d_bits, const uint64_t* d_cont_off,
                            const uint64_t* d_cont_len, uint32_t* d_sbase, uint32_t* d_slen, int32_t* d_status,
                            cudaStream_t st, bool check_numerics) {
  k_dec_prep<<<(p.n_cont + 63) / 64, 64, 0, st>>>(p, d_bits, d_cont_off, d_cont_len, d_sbase, d_slen, d_status,
                                                 check_numerics ? 1 : 0);
  return cudaGetLastError();
}

template <int PREC, bool PROF>
static cudaError_t launch_decode_t(const Plan& p, const DevWeights& w, const uint8_t* d_bits,
                                   const uint64_t* d_cont_off, const uint32_t* d_sbase, const uint32_t* d_slen,
                                   uint8_t* d_imgs, int32_t* d_status, cudaStream_t st,
                                   unsigned long long* prof, uint32_t* d_sync) {
  const size_t sm = dec_smem_bytes(PREC, p.gpt > p.gpl ? p.gpt : p.gpl, p.w3d);
  auto kern = k_decode<PREC, PROF, false>;
  if constexpr (PREC < 2) {  // (P350K: no volumes)
    if (p.w3d) kern = k_decode<PREC, PROF, true>;
  }
  cudaError_t e = set_smem(kern, sm);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.u_cnt * p.nc);
  cfg.blockDim = dim3(dec_block(PREC));
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  if (p.nc > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.nc;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p, w, d_bits, d_cont_off, d_sbase, d_slen, d_imgs, d_status,
                            prof, d_sync);
}

size_t dec_smem_limit() {
  static size_t lim = 0;
  if (!lim) {
    int dev = 0, optin = 0;
    cudaFuncAttributes fa = {};
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess &&
        cudaFuncGetAttributes(&fa, k_decode<1, false, false>) == cudaSuccess && optin > (int)fa.sharedSizeBytes)
      lim = (size_t)optin - fa.sharedSizeBytes;
    else
      lim = MAX_DYN_SMEM;
    cudaGetLastError();
  }
  return lim;
}

template <int PREC>
static int max_clusters_t(uint32_t nc, size_t sm) {
  if (set_smem(k_decode<PREC, false, false>, sm) != cudaSuccess) return 0;
  if (nc > 8 && cudaFuncSetAttribute(k_decode<PREC, false, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                    cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nc);
  cfg.blockDim = dim3(dec_block(PREC));
  cfg.dynamicSmemBytes = sm;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nc;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_decode<PREC, false, false>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int dec_max_active_clusters(uint32_t engine, uint32_t nc, size_t smem) {
  if (engine == 4) return max_clusters_t<4>(nc, smem);
  if (engine == 3) return max_clusters_t<3>(nc, smem);
  if (engine == 2) return max_clusters_t<2>(nc, smem);
  return engine == 1 ? max_clusters_t<1>(nc, smem) : max_clusters_t<0>(nc, smem);
}

cudaError_t launch_decode(const Plan& p, const DevWeights& w, const uint8_t* d_bits, const uint64_t* d_cont_off,
                          const uint32_t* d_sbase, const uint32_t* d_slen, uint8_t* d_imgs, int32_t* d_status,
                          cudaStream_t st, unsigned long long* prof, uint32_t* d_sync) {
  if (p.engine == 4)
    return launch_decode_t<4, false>(p, w, d_bits, d_cont_off, d_sbase, d_slen, d_imgs, d_status, st, prof, d_sync);
  if (p.engine == 3)
    return launch_decode_t<3, false>(p, w, d_bits, d_cont_off, d_sbase, d_slen, d_imgs, d_status, st, prof, d_sync);
  if (p.engine == 2) {
    if (prof)
      return launch_decode_t<2, true>(p, w, d_bits, d_cont_off, d_sbase, d_slen, d_imgs, d_status, st, prof, d_sync);
    return launch_decode_t<2, false>(p, w, d_bits, d_cont_off, d_sbase, d_slen, d_imgs, d_status, st, prof, d_sync);
  }
  if (prof) {
    if (p.precision == 1)
      return launch_decode_t<1, true>(p, w, d_bits, d_cont_off, d_sbase, d_slen, d_imgs, d_status, st, prof, d_sync);
    return launch_decode_t<0, true>(p, w, d_bits, d_cont_off, d_sbase, d_slen, d_imgs, d_status, st, prof, d_sync);
  }
  if (p.precision == 1)
    return launch_decode_t<1, false>(p, w, d_bits, d_cont_off, d_sbase, d_slen, d_imgs, d_status, st, prof, d_sync);
  return launch_decode_t<0, false>(p, w, d_bits, d_cont_off, d_sbase, d_slen, d_imgs, d_status, st, prof, d_sync);
}

}  // namespace dlic
