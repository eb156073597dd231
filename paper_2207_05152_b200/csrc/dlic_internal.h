// dlic_internal.h — host-side view of the kernels (no torch, no CUDA types
// beyond cudaStream_t) shared by dlic_api.cpp and dlic_kernels.cu.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace dlic {

// Uniform tiling of n equal-size images into independent units (reading Q16).
// Untiled = one unit per image (tw = W, th = H).
struct Plan {
  uint32_t W, H, tw, th, ntx, nty, G, n_img;
  uint32_t upi;        // units per image = ntx * nty
  uint32_t gpt, gpl;   // groups per full-height tile / per last-row tile
  uint32_t spi;        // streams per image
  uint32_t cap_words;  // scratch words per stream (2G + G*tw)
  uint32_t hdr_bytes;  // HDR_FIXED + 4*spi
  uint32_t precision;
  uint32_t tiles_per_unit;  // ceil(tw*th / 64) 64-pixel MLP tiles
  uint32_t nc;              // CTAs per decode cluster (slots = 64*nc >= ceil(tw/3))
  uint32_t hdr_tw, hdr_th;  // tile fields as written in the header (0,0 = untiled)
  uint64_t max_container;   // hdr_bytes + per-stream worst case
  // unit range of this launch: units [u_lo, u_lo + u_cnt) of the batch, i.e.
  // streams [s_lo, s_lo + s_cnt) (the whole batch unless a *_units call)
  uint32_t u_lo, u_cnt, s_lo, s_cnt;
  uint32_t n_meta;  // metadata reals per container (block: 4 + 4 n_meta bytes after the size table)
  // volumes (§8(f) f2): `depth` consecutive images (slices) form one volume
  // and one container (window id 2, slice-major streams); 2D: depth 1
  uint32_t depth, n_cont, spc;  // slices per container, containers, streams per container
  uint32_t w3d;                 // 3D window (R13): 9 taps from the slice below
  // the network engine the kernels instantiate: 0 fp32 FFMA (P100K), 1 bf16
  // tcgen05 with resident weights (P100K), 2 bf16 tcgen05 with weights
  // streamed from L2 (P350K, dlic_stream.cuh).  The header keeps `precision`.
  uint32_t engine;
  uint32_t bits;  // alphabet: 8 (u8 pixels) or 12 (u16 pixels, engine 3; container byte 7 = 12)
  uint32_t prof;  // diagnostics only (DLIC_PROF_STREAM): issuer cycle counters
};

constexpr uint32_t HDR_FIXED = 60;  // container header bytes before the size table (version 2)
constexpr uint32_t CONTAINER_VERSION = 2;

struct Unit {
  uint32_t img, x0, y0, w, h, first_stream, ngroups;
  uint64_t fc_off;
};

__host__ __device__ inline Unit unit_info(const Plan& p, uint32_t u) {
  Unit r;
  r.img = u / p.upi;
  const uint32_t k = u % p.upi, tx = k % p.ntx, ty = k / p.ntx;
  r.x0 = tx * p.tw;
  r.y0 = ty * p.th;
  r.w = (p.W - r.x0 < p.tw) ? p.W - r.x0 : p.tw;
  r.h = (p.H - r.y0 < p.th) ? p.H - r.y0 : p.th;
  r.ngroups = (r.h + p.G - 1) / p.G;
  r.first_stream = r.img * p.spi + ty * p.ntx * p.gpt + tx * r.ngroups;
  r.fc_off = (uint64_t)r.img * p.W * p.H + (uint64_t)ty * p.th * p.W + (uint64_t)tx * p.tw * r.h;
  return r;
}

// global stream index -> (unit, group)
__host__ __device__ inline void stream_info(const Plan& p, uint32_t s, uint32_t& u, uint32_t& g) {
  const uint32_t img = s / p.spi, sp = s % p.spi;
  const uint32_t full = (p.nty - 1) * p.ntx * p.gpt;
  uint32_t tx, ty;
  if (sp < full) {
    ty = sp / (p.ntx * p.gpt);
    const uint32_t rem = sp % (p.ntx * p.gpt);
    tx = rem / p.gpt;
    g = rem % p.gpt;
  } else {
    ty = p.nty - 1;
    const uint32_t rem = sp - full;
    tx = rem / p.gpl;
    g = rem % p.gpl;
  }
  u = img * p.upi + ty * p.ntx + tx;
}

// weights as uploaded at model load
struct DevWeights {
  const uint8_t* wimg;  // bf16 core-matrix image, WIMG_BYTES (P350K: the SWIMG_BYTES slice stream)
  const float* bias;    // BIAS_TOTAL floats
  const float* w32;     // fp32 blob (f32_off layout)
  // per-image layer-1 bias with the metadata inputs folded in ([n_img][HID]
  // fp32, k_meta_bias), or null (no metadata: the model's own b1)
  const float* b1img;
};

// Metadata inputs -> per-image layer-1 bias: out[i][n] = b1[n] +
// sum_k m'_ik W1[78 + k][n], m' = (m - min) / (max - min) in binary32; bf16
// path: m' and W rounded to bf16 (exact products), sum in fp32 k ascending,
// then + b1; fp32 path: the same with fp32 operands (fma chain).
// raw reals from d_meta[i][k] (encode), or, when d_bits is set, from the
// metadata block of container i at d_bits + d_cont_off[i] + meta_off (decode)
cudaError_t launch_meta_bias(uint32_t n_img, uint32_t n_meta, const float* d_meta, const uint8_t* d_bits,
                             const uint64_t* d_cont_off, uint32_t meta_off, const float* d_range,
                             const float* d_wmeta, const float* d_b1, uint32_t precision, float* d_out,
                             cudaStream_t st);

struct Timing;  // optional CUDA-event timing, owned by the API layer

// --- launchers (return cudaGetLastError() of the launch)
cudaError_t launch_enc_mlp(const Plan& p, const DevWeights& w, const uint8_t* d_imgs, uint32_t* d_fc,
                           float* dbg_logits, float* dbg_probs, uint16_t* dbg_freqs, cudaStream_t st,
                           int num_sms);
cudaError_t launch_rans_enc(const Plan& p, const uint32_t* d_fc, uint16_t* d_scratch, uint32_t* d_words,
                            cudaStream_t st);
cudaError_t launch_container(const Plan& p, const uint8_t* model_sha, const uint32_t* d_words,
                             const uint16_t* d_scratch, uint8_t* d_out, uint64_t out_stride,
                             uint64_t* d_sizes, uint64_t* d_stream_dst, cudaStream_t st, bool payload_only = false,
                             const float* d_meta = nullptr);
cudaError_t launch_dec_prep(const Plan& p, const uint8_t* d_bits, const uint64_t* d_cont_off,
                            const uint64_t* d_cont_len, uint32_t* d_sbase, uint32_t* d_slen,
                            int32_t* d_status, cudaStream_t st, bool check_numerics = true);
cudaError_t launch_decode(const Plan& p, const DevWeights& w, const uint8_t* d_bits, const uint64_t* d_cont_off,
                          const uint32_t* d_sbase, const uint32_t* d_slen, uint8_t* d_imgs, int32_t* d_status,
                          cudaStream_t st, unsigned long long* prof = nullptr, uint32_t* d_sync = nullptr);
// volumes: d_sync = zeroed u32 [1 + units] (unit ticket + per-unit progress; sync_words)
inline size_t sync_words(const Plan& p) { return p.w3d ? 1u + (size_t)p.u_lo + p.u_cnt : 0u; }

cudaError_t launch_rans_dec_tables(const Plan& p, const uint8_t* d_bits, const uint32_t* d_sbase,
                                   const uint32_t* d_slen, const uint16_t* d_tables, uint8_t* d_out,
                                   int32_t* d_status, cudaStream_t st);

// how many decode clusters of nc CTAs (dynamic smem `smem`) the device can
// co-schedule (cudaOccupancyMaxActiveClusters); 0 = the launch cannot run
// (engine: Plan::engine)
int dec_max_active_clusters(uint32_t engine, uint32_t nc, size_t smem);
size_t dec_smem_bytes(uint32_t engine, uint32_t max_groups, uint32_t w3d = 0);
size_t dec_smem_limit();
size_t enc_smem_bytes(uint32_t engine, uint32_t w3d = 0);

}  // namespace dlic
