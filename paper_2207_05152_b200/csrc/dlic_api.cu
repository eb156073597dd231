// dlic_api.cpp — the C-ABI of libdlic.so (include/dlic.h).
//
// Host side only: model parsing and SHA-256, weight packing
// into the tcgen05 shared-memory image, planning (units, groups, decode
// cluster size), the container framing, scratch
// management and kernel launches.  Every pixel-level step runs in the CUDA
// kernels of dlic_kernels.cu; there is no CPU fallback.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dlic.h"
#include "dlic_device.cuh"
#include "dlic_internal.h"
#include "dlic_stream.cuh"
#include "dlic_x3.cuh"
#include "sha256.h"

using namespace dlic;

struct dlic_model {
  int device = 0;
  std::vector<uint8_t> blob;  // the "DLICMDL1" bytes
  uint8_t sha[32];
  std::vector<uint32_t> dims;
  bool p100k = false;  // topology the GPU engines run (see dlic_model_load)
  bool p350k = false;  // 78 -> 256 x5 -> 256 (§8(f) f1): bf16 only, streamed weights (engine 2)
  bool p12 = false;    // 78 -> 256 x5 -> 4096 (§8(f) f3, 12-bit pixels): bf16 only (engine 3)
  uint32_t n_meta = 0;
  bool in3d = false;   // 87 window inputs: the 3D window (R13)
  uint8_t* d_wimg = nullptr;
  float* d_bias = nullptr;
  float* d_w32 = nullptr;
  float* d_wmeta = nullptr;  // metadata rows of W1 [n_meta][HID] fp32
  float* d_range = nullptr;  // (min, max) per metadata feature
  uint8_t* d_x3img = nullptr;  // fp32 path on tcgen05 (engine 4): hi/lo bf16 limbs (dlic_x3.cuh)
  float* d_x3bias = nullptr;
  DevWeights dw(const float* b1img = nullptr, uint32_t engine = 1) const {
    if (engine == 4) return DevWeights{d_x3img, d_x3bias, d_w32, b1img};
    return DevWeights{d_wimg, d_bias, d_w32, b1img};
  }
};

namespace {

thread_local std::string g_err;
thread_local bool g_timing = false;

dlic_status fail(dlic_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      return fail(e_ == cudaErrorMemoryAllocation ? DLIC_E_OUT_OF_MEMORY : DLIC_E_CUDA,  \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                   \
    }                                                                                    \
  } while (0)

// ---------------------------------------------------------------- timing
struct EvPair {
  cudaEvent_t a = nullptr, b = nullptr;
  bool used = false;
};
thread_local std::map<std::string, EvPair> g_ev;
void ev_begin(const char* name, cudaStream_t st) {
  if (!g_timing) return;
  EvPair& e = g_ev[name];
  if (!e.a) {
    cudaEventCreate(&e.a);
    cudaEventCreate(&e.b);
  }
  cudaEventRecord(e.a, st);
}
void ev_end(const char* name, cudaStream_t st) {
  if (!g_timing) return;
  EvPair& e = g_ev[name];
  cudaEventRecord(e.b, st);
  e.used = true;
}

// ---------------------------------------------------------------- device info
int num_sms(int dev) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> l(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  cache[dev] = n;
  return n;
}

dlic_status check_device(int dev) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(DLIC_E_CUDA, "no CUDA device");
  if (dev < 0 || dev >= n) return fail(DLIC_E_INVALID_ARG, "bad cuda_device");
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) return fail(DLIC_E_CUDA, "libdlic kernels are built for sm_100a (B200)");
  CUDA_TRY(cudaSetDevice(dev));
  static std::once_flag once[64];
  if (dev < 64)
    std::call_once(once[dev], [dev] {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
    });
  return DLIC_OK;
}

cudaStream_t my_stream() {
  thread_local cudaStream_t s = nullptr;
  thread_local int dev = -1;
  int cur = 0;
  cudaGetDevice(&cur);
  if (!s || dev != cur) {
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    dev = cur;
  }
  return s;
}

// host copy between a user buffer and pinned staging: large copies (batches
// of images or containers, tens to hundreds of MB) are split across host
// threads -- one thread's memcpy runs at a fraction of the host's memory
// bandwidth and would dominate the end-to-end time of the batch calls
void par_memcpy(void* dst, const void* src, size_t n) {
  constexpr size_t MIN_SPLIT = 8u << 20;
  const unsigned hw = std::thread::hardware_concurrency();
  const unsigned nt = (unsigned)std::min<size_t>(std::min(hw ? hw : 1u, 16u), n / MIN_SPLIT);
  if (nt <= 1) {
    memcpy(dst, src, n);
    return;
  }
  const size_t chunk = ((n + nt - 1) / nt + 63) & ~(size_t)63;
  std::vector<std::thread> th;
  th.reserve(nt - 1);
  for (unsigned i = 1; i < nt; ++i) {
    const size_t a = std::min(n, (size_t)i * chunk), b = std::min(n, a + chunk);
    if (b > a) th.emplace_back([=]() { memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a); });
  }
  memcpy(dst, src, std::min(n, chunk));
  for (auto& t : th) t.join();
}

// pinned staging buffers (per thread, grown on demand)
struct Pinned {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t n) {
    if (n > cap) {
      if (p) cudaFreeHost(p);
      cap = std::max(n, (size_t)1 << 20);
      if (cudaMallocHost(&p, cap) != cudaSuccess) {
        p = nullptr;
        cap = 0;
      }
    }
    return p;
  }
};
thread_local Pinned g_pin_in, g_pin_out;

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// stream-ordered scratch freed at scope exit
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  template <class T>
  cudaError_t alloc(T** out, size_t bytes) {
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 16, st);
    if (e == cudaSuccess) ptrs.push_back(p);
    *out = reinterpret_cast<T*>(p);
    return e;
  }
};

// ---------------------------------------------------------------- model parsing
uint32_t rd32(const uint8_t* p) { return p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24); }
uint16_t rd16(const uint8_t* p) { return (uint16_t)(p[0] | (p[1] << 8)); }

struct ParsedModel {
  std::vector<uint32_t> dims;
  std::vector<std::vector<float>> W, b;
  std::vector<uint32_t> pool;        // pooling group after each layer (0 = none)
  std::vector<float> meta_range;     // (min, max) per metadata feature
};

dlic_status parse_model(const uint8_t* d, size_t len, ParsedModel& pm, uint8_t sha_out[32]) {
  if (!d || len < 8 + 2 + 2 + 32 || memcmp(d, "DLICMDL1", 8) != 0) return fail(DLIC_E_CORRUPT_MODEL, "model magic");
  uint8_t h[32];
  sha256(d, len - 32, h);
  if (memcmp(h, d + len - 32, 32) != 0) return fail(DLIC_E_CORRUPT_MODEL, "model SHA-256 mismatch");
  const size_t body = len - 32;
  size_t off = 8;
  const uint32_t nl = rd16(d + off);
  off += 2;
  if (nl == 0 || nl > 64) return fail(DLIC_E_CORRUPT_MODEL, "layer count");
  for (uint32_t l = 0; l < nl; ++l) {
    if (off + 10 > body) return fail(DLIC_E_CORRUPT_MODEL, "truncated layer header");
    const uint32_t in = rd32(d + off), outd = rd32(d + off + 4);
    const uint32_t g = d[off + 9];
    off += 10;
    if (l > 0) {  // dims chain after the previous layer's pooling
      const uint32_t gp = pm.pool.back() ? pm.pool.back() : 1u;
      if (pm.dims.back() % gp != 0 || pm.dims.back() / gp != in)
        return fail(DLIC_E_CORRUPT_MODEL, "layer dims do not chain");
    }
    if (l == 0) pm.dims.push_back(in);
    pm.dims.push_back(outd);
    pm.pool.push_back(g);
    const size_t nw = (size_t)in * outd;
    if (in == 0 || outd == 0 || off + 4 * (nw + outd) > body) return fail(DLIC_E_CORRUPT_MODEL, "truncated weights");
    std::vector<float> w(nw), bb(outd);
    memcpy(w.data(), d + off, 4 * nw);
    off += 4 * nw;
    memcpy(bb.data(), d + off, 4 * outd);
    off += 4 * outd;
    pm.W.push_back(std::move(w));
    pm.b.push_back(std::move(bb));
  }
  if (off + 2 > body) return fail(DLIC_E_CORRUPT_MODEL, "truncated meta");
  const uint32_t nmeta = rd16(d + off);
  if (off + 2 + 8 * (size_t)nmeta > body) return fail(DLIC_E_CORRUPT_MODEL, "truncated metadata ranges");
  for (uint32_t k = 0; k < 2 * nmeta; ++k) {
    float v;
    memcpy(&v, d + off + 2 + 4 * k, 4);
    pm.meta_range.push_back(v);
  }
  off += 2 + 8 * (size_t)nmeta;
  if (off != body) return fail(DLIC_E_CORRUPT_MODEL, "model length");
  if (sha_out) memcpy(sha_out, h, 32);
  return DLIC_OK;
}

uint16_t bf16_bits(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}

// Fold a pooled network into the engines' shape: average pooling of g units
// after layer l is linear, so layer l+1 with K = 128/g inputs becomes an
// equivalent layer with K = 128 whose row k is W[k / g] / g (exact in fp32 and
// bf16: g is a power of two).  Returns false for topologies outside the engines.
static bool engine_weights(const ParsedModel& pm, std::vector<std::vector<float>>& W, uint32_t& n_meta,
                           bool& in3d) {
  if (pm.W.size() != (size_t)NLAYER) return false;
  n_meta = (uint32_t)(pm.meta_range.size() / 2);
  if (n_meta > DLIC_MAX_META) return false;
  const uint32_t kwin = pm.dims[0] - n_meta;  // window inputs: 78 (2D) or 87 (3D)
  if (kwin != (uint32_t)KIN && kwin != (uint32_t)KIN3) return false;
  in3d = kwin == (uint32_t)KIN3;
  for (int l = 0; l < NLAYER; ++l)
    if (pm.dims[l + 1] != (uint32_t)layer_n(l)) return false;  // outputs 128 x5, 256
  if (pm.pool[NLAYER - 1] != 0) return false;
  W.assign(NLAYER, {});
  W[0] = pm.W[0];
  for (int l = 1; l < NLAYER; ++l) {
    const uint32_t g = pm.pool[l - 1] ? pm.pool[l - 1] : 1u;
    if (g & (g - 1)) return false;  // powers of two only (exact 1/g)
    const uint32_t N = (uint32_t)layer_n(l);
    W[l].resize((size_t)HID * N);
    for (uint32_t k = 0; k < (uint32_t)HID; ++k)
      for (uint32_t n = 0; n < N; ++n) W[l][(size_t)k * N + n] = pm.W[l][(size_t)(k / g) * N + n] / (float)g;
  }
  return true;
}

// P350K (reading R4): 78 window inputs -> 256 x5 -> 256 logits; P12
// (R16): the same hidden stack -> 4096 logits (12-bit pixels).  No pooling,
// no metadata.
static bool is_stream_model(const ParsedModel& pm, uint32_t nout) {
  if (pm.W.size() != (size_t)NLAYER || !pm.meta_range.empty() || pm.dims[0] != (uint32_t)KIN) return false;
  for (int l = 0; l < NLAYER; ++l)
    if (pm.dims[l + 1] != (l == NLAYER - 1 ? nout : (uint32_t)SH) || pm.pool[l] != 0) return false;
  return true;
}

// The P350K slice stream (dlic_stream.cuh): 85 K=16 slices of 8 KB, layer 1
// first (K in the engine's kpos_tap order, the fresh taps zero), each in the
// UMMA no-swizzle K-major core-matrix layout of an N=256 operand; biases
// [5][256] + [256] and the fresh-tap table (bf16-rounded, float4 per pair).
// P12: layers 1-5 as P350K's, then the head: for each 128-column chunk q,
// K = 256 in 16 slices of N = 128 (4 KB, the same core-matrix layout with
// N = 128), two 32 KB stream chunks (K-slices 0-7, 8-15) after layer 5's.
// Biases: [5][256], the fresh table at SB_FRESH, the 4096 head biases at
// SB12_HEAD.
static dlic_status upload_p12(dlic_model* m, const ParsedModel& pm) {
  std::vector<uint8_t> img(SWIMG12_BYTES, 0);
  for (int l = 0; l < NLAYER - 1; ++l) {
    const int K = l == 0 ? KPAD : SH;
    for (int k = 0; k < K; ++k)
      for (int n = 0; n < SH; ++n) {
        const int kt = l == 0 ? kpos_tap(k) : k;
        const bool fresh = l == 0 && (kt == TAP_FA || kt == TAP_FB);
        const float v = kt >= 0 && kt < (l == 0 ? KIN : SH) && !fresh ? pm.W[l][(size_t)kt * SH + n] : 0.0f;
        const uint16_t u = bf16_bits(v);
        const int kk = k / 16, kl = k % 16;
        const size_t a = (size_t)s_slice(l, kk) * SL_BYTES + (size_t)(kl / 8) * (SH / 8) * 128 +
                         (size_t)(n / 8) * 128 + (n % 8) * 16 + (kl % 8) * 2;
        memcpy(&img[a], &u, 2);
      }
  }
  const size_t head0 = SL1_BYTES + (size_t)CH_HID12 * CH_BYTES;
  for (int k = 0; k < SH; ++k)
    for (int n = 0; n < H12_N; ++n) {
      const int q = n / H12_CN, nl = n % H12_CN, kk = k / 16, kl = k % 16;
      const uint16_t u = bf16_bits(pm.W[NLAYER - 1][(size_t)k * H12_N + n]);
      const size_t a = head0 + (size_t)(2 * q + kk / H12_CH_SL) * CH_BYTES + (size_t)(kk % H12_CH_SL) * H12_SL_BYTES +
                       (size_t)(kl / 8) * (H12_CN / 8) * 128 + (size_t)(nl / 8) * 128 + (nl % 8) * 16 + (kl % 8) * 2;
      memcpy(&img[a], &u, 2);
    }
  std::vector<float> bias(SBIAS12_BYTES / 4, 0.0f);
  for (int l = 0; l < NLAYER - 1; ++l)
    for (int n = 0; n < SH; ++n) bias[(size_t)l * SH + n] = pm.b[l][n];
  for (int n = 0; n < H12_N; ++n) bias[SB12_HEAD + n] = pm.b[NLAYER - 1][n];
  for (int n = 0; n < SH; ++n) {
    const size_t q = SB_FRESH + 4 * (size_t)(n / 2) + (n & 1);
    const uint32_t ua = (uint32_t)bf16_bits(pm.W[0][(size_t)TAP_FA * SH + n]) << 16;
    const uint32_t ub = (uint32_t)bf16_bits(pm.W[0][(size_t)TAP_FB * SH + n]) << 16;
    memcpy(&bias[q], &ua, 4);
    memcpy(&bias[q + 2], &ub, 4);
  }
  CUDA_TRY(cudaMalloc(&m->d_wimg, SWIMG12_BYTES));
  CUDA_TRY(cudaMalloc(&m->d_bias, bias.size() * 4));
  CUDA_TRY(cudaMemcpy(m->d_wimg, img.data(), SWIMG12_BYTES, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(m->d_bias, bias.data(), bias.size() * 4, cudaMemcpyHostToDevice));
  return DLIC_OK;
}

static dlic_status upload_p350k(dlic_model* m, const ParsedModel& pm) {
  std::vector<uint8_t> img(SWIMG_BYTES, 0);
  for (int l = 0; l < NLAYER; ++l) {
    const int K = l == 0 ? KPAD : SH;
    for (int k = 0; k < K; ++k)
      for (int n = 0; n < SH; ++n) {
        const int kt = l == 0 ? kpos_tap(k) : k;
        const bool fresh = l == 0 && (kt == TAP_FA || kt == TAP_FB);
        const float v = kt >= 0 && kt < (l == 0 ? KIN : SH) && !fresh ? pm.W[l][(size_t)kt * SH + n] : 0.0f;
        const uint16_t u = bf16_bits(v);
        const int kk = k / 16, kl = k % 16;
        const size_t a = (size_t)s_slice(l, kk) * SL_BYTES + (size_t)(kl / 8) * (SH / 8) * 128 +
                         (size_t)(n / 8) * 128 + (n % 8) * 16 + (kl % 8) * 2;
        memcpy(&img[a], &u, 2);
      }
  }
  std::vector<float> bias(SBIAS_BYTES / 4, 0.0f);
  for (int l = 0; l < NLAYER; ++l)
    for (int n = 0; n < SH; ++n) bias[(size_t)l * SH + n] = pm.b[l][n];
  auto bf16f = [](float v) {
    const uint32_t u = (uint32_t)bf16_bits(v) << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
  };
  for (int n = 0; n < SH; ++n) {
    const size_t q = SB_FRESH + 4 * (size_t)(n / 2) + (n & 1);
    bias[q] = bf16f(pm.W[0][(size_t)TAP_FA * SH + n]);
    bias[q + 2] = bf16f(pm.W[0][(size_t)TAP_FB * SH + n]);
  }
  CUDA_TRY(cudaMalloc(&m->d_wimg, SWIMG_BYTES));
  CUDA_TRY(cudaMalloc(&m->d_bias, bias.size() * 4));
  CUDA_TRY(cudaMemcpy(m->d_wimg, img.data(), SWIMG_BYTES, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(m->d_bias, bias.data(), bias.size() * 4, cudaMemcpyHostToDevice));
  return DLIC_OK;
}

// The fp32 path's tensor-core image (dlic_x3.cuh): every weight as bf16 hi =
// bf16_rn(w) and lo = bf16_rn(w - hi).  Layer 1 resident: 5 K-slices x {hi,
// lo} (N=128, kpos_tap K order, fresh taps zero); then 12 stream chunks of 32
// KB: layers 2-5 as 2 chunks of 4 K-slices x {hi, lo} (N=128), the logits
// layer as 4 chunks of 2 K-slices x {hi, lo} (N=256).  Biases fp32: [5][128],
// [256], fresh table {wa[n], wa[n+1], wb[n], wb[n+1]} (fp32, exact).
static dlic_status upload_x3(dlic_model* m, const ParsedModel& pm) {
  std::vector<uint8_t> img(X3_WIMG_BYTES, 0);
  auto limbs = [](float w, uint16_t& hi, uint16_t& lo) {
    hi = bf16_bits(w);
    const uint32_t hu = (uint32_t)hi << 16;
    float hf;
    memcpy(&hf, &hu, 4);
    lo = bf16_bits(w - hf);
  };
  // element (n, k) of a K=16 slice of an N-wide operand at slice base `a`
  auto put = [&](size_t a, int N, int n, int kl, uint16_t u) {
    memcpy(&img[a + (size_t)(kl / 8) * (N / 8) * 128 + (size_t)(n / 8) * 128 + (n % 8) * 16 + (kl % 8) * 2], &u, 2);
  };
  for (int k = 0; k < KPAD; ++k)
    for (int n = 0; n < HID; ++n) {
      const int kt = kpos_tap(k);
      const bool fresh = kt == TAP_FA || kt == TAP_FB;
      const float w = kt >= 0 && kt < KIN && !fresh ? pm.W[0][(size_t)kt * HID + n] : 0.0f;
      uint16_t hi, lo;
      limbs(w, hi, lo);
      const int kk = k / 16;
      put((size_t)(2 * kk) * X3_SL, HID, n, k % 16, hi);
      put((size_t)(2 * kk + 1) * X3_SL, HID, n, k % 16, lo);
    }
  for (int l = 1; l < NLAYER; ++l) {
    const int N = layer_n(l);
    const bool last = l == NLAYER - 1;
    const size_t sl = last ? X3_SL_LAST : X3_SL;
    const int per = last ? 2 : 4;  // K-slices per chunk
    const size_t c0 = X3_L1_BYTES + (size_t)(l - 1) * 2 * CH_BYTES;  // layers 2-5: 2 chunks each
    for (int k = 0; k < HID; ++k)
      for (int n = 0; n < N; ++n) {
        uint16_t hi, lo;
        limbs(pm.W[l][(size_t)k * N + n], hi, lo);
        const int kk = k / 16, cl = kk / per, i = kk % per;
        const size_t base = c0 + (size_t)cl * CH_BYTES + (size_t)(2 * i) * sl;
        put(base, N, n, k % 16, hi);
        put(base + sl, N, n, k % 16, lo);
      }
  }
  std::vector<float> bias(X3_BIAS_BYTES / 4, 0.0f);
  for (int l = 0; l < NLAYER - 1; ++l)
    for (int n = 0; n < HID; ++n) bias[(size_t)l * HID + n] = pm.b[l][n];
  for (int n = 0; n < NOUT; ++n) bias[X3_B_LAST + n] = pm.b[NLAYER - 1][n];
  for (int n = 0; n < HID; ++n) {
    const size_t q = X3_B_FRESH + 4 * (size_t)(n / 2) + (n & 1);
    bias[q] = pm.W[0][(size_t)TAP_FA * HID + n];
    bias[q + 2] = pm.W[0][(size_t)TAP_FB * HID + n];
  }
  CUDA_TRY(cudaMalloc(&m->d_x3img, X3_WIMG_BYTES));
  CUDA_TRY(cudaMalloc(&m->d_x3bias, bias.size() * 4));
  CUDA_TRY(cudaMemcpy(m->d_x3img, img.data(), X3_WIMG_BYTES, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(m->d_x3bias, bias.data(), bias.size() * 4, cudaMemcpyHostToDevice));
  return DLIC_OK;
}

dlic_status upload_model(dlic_model* m, const ParsedModel& pm_in) {
  m->dims = pm_in.dims;
  std::vector<std::vector<float>> Wf;
  uint32_t n_meta = 0;
  bool in3d = false;
  if (is_stream_model(pm_in, (uint32_t)NOUT)) {
    m->p350k = true;
    return upload_p350k(m, pm_in);
  }
  if (is_stream_model(pm_in, (uint32_t)H12_N)) {
    m->p12 = true;
    return upload_p12(m, pm_in);
  }
  m->p100k = engine_weights(pm_in, Wf, n_meta, in3d);
  if (!m->p100k) return DLIC_OK;  // loadable; GPU engines refuse it at encode/decode
  m->n_meta = n_meta;
  m->in3d = in3d;
  const uint32_t kwin = in3d ? (uint32_t)KIN3 : (uint32_t)KIN;  // metadata rows follow the window rows
  ParsedModel pm = pm_in;
  pm.W = Wf;  // pooling folded; W1 keeps its KIN + n_meta rows (the packers below read rows < KIN)
  // bf16 UMMA image: layer l, element (n, k) of B = W^T at
  // (k/8)*(N/8)*128 + (n/8)*128 + (n%8)*16 + (k%8)*2   (K-major, no swizzle)
  std::vector<uint8_t> img(WIMG_BYTES, 0);
  for (int l = 0; l < NLAYER; ++l) {
    const int K = layer_k(l), N = layer_n(l), Kr = l == 0 ? KIN : K;  // W1's metadata rows: d_wmeta
    for (int k = 0; k < K; ++k)
      for (int n = 0; n < N; ++n) {
        const int kt = l == 0 ? kpos_tap(k) : k;  // layer 1: the engine's K order
        const bool fresh = l == 0 && (kt == TAP_FA || kt == TAP_FB);  // applied in the epilogue
        const float v = kt >= 0 && kt < Kr && !fresh ? pm.W[l][(size_t)kt * N + n] : 0.0f;
        const uint16_t u = bf16_bits(v);
        const size_t a = wimg_off(l) + (size_t)(k / 8) * (N / 8) * 128 + (size_t)(n / 8) * 128 + (n % 8) * 16 + (k % 8) * 2;
        memcpy(&img[a], &u, 2);
      }
  }
  std::vector<float> bias(BIAS_TOTAL + FRESH_FLOATS + (in3d ? W3D_WORDS : 0));
  for (int l = 0; l < NLAYER; ++l)
    for (int n = 0; n < layer_n(l); ++n) bias[(l < NLAYER - 1 ? l * HID : BIAS_OFF_LAST) + n] = pm.b[l][n];
  // fresh-tap weights (bf16-rounded like the MMA image), float4 per pair n, n+1
  auto bf16f = [](float v) {
    const uint32_t u = (uint32_t)bf16_bits(v) << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
  };
  for (int n = 0; n < HID; ++n) {
    const size_t q = FRESH_OFF + 4 * (size_t)(n / 2) + (n & 1);
    bias[q] = bf16f(pm.W[0][(size_t)TAP_FA * HID + n]);
    bias[q + 2] = bf16f(pm.W[0][(size_t)TAP_FB * HID + n]);
  }
  if (in3d) {  // lower-layer (3D) tap weights, bf16 pairs: word k*64 + n/2 = (W[78+k][n], W[78+k][n+1])
    for (int k = 0; k < 9; ++k)
      for (int n = 0; n < HID; n += 2) {
        const uint32_t lo = bf16_bits(pm.W[0][(size_t)(KIN + k) * HID + n]);
        const uint32_t hi = bf16_bits(pm.W[0][(size_t)(KIN + k) * HID + n + 1]);
        const uint32_t u = lo | (hi << 16);
        memcpy(&bias[W3D_OFF + (size_t)k * (HID / 2) + n / 2], &u, 4);
      }
  }
  // fp32 blob: layer 0 has the window rows (78 or 87), the others as packed
  std::vector<float> w32(f32_off(NLAYER) + (in3d ? (size_t)(KIN3 - KIN) * HID : 0));
  size_t o32 = 0;
  for (int l = 0; l < NLAYER; ++l) {
    const int K = l == 0 ? (int)kwin : f32_k(l), N = layer_n(l);
    memcpy(&w32[o32], pm.W[l].data(), 4 * (size_t)K * N);
    memcpy(&w32[o32 + (size_t)K * N], pm.b[l].data(), 4 * (size_t)N);
    o32 += (size_t)K * N + N;
  }
  if (n_meta) {  // metadata rows of W1 and their normalisation constants
    std::vector<float> wm((size_t)n_meta * HID);
    for (uint32_t k = 0; k < n_meta; ++k)
      for (int n = 0; n < HID; ++n) wm[(size_t)k * HID + n] = pm.W[0][(size_t)(kwin + k) * HID + n];
    CUDA_TRY(cudaMalloc(&m->d_wmeta, wm.size() * 4));
    CUDA_TRY(cudaMalloc(&m->d_range, pm.meta_range.size() * 4));
    CUDA_TRY(cudaMemcpy(m->d_wmeta, wm.data(), wm.size() * 4, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(m->d_range, pm.meta_range.data(), pm.meta_range.size() * 4, cudaMemcpyHostToDevice));
  }
  if (!in3d) {  // the fp32 path's bf16x3 image (engine 4; volumes keep the FFMA engine)
    dlic_status s = upload_x3(m, pm);
    if (s != DLIC_OK) return s;
  }
  CUDA_TRY(cudaMalloc(&m->d_wimg, WIMG_BYTES));
  CUDA_TRY(cudaMalloc(&m->d_bias, bias.size() * 4));
  CUDA_TRY(cudaMalloc(&m->d_w32, w32.size() * 4));
  CUDA_TRY(cudaMemcpy(m->d_wimg, img.data(), WIMG_BYTES, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(m->d_bias, bias.data(), bias.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(m->d_w32, w32.data(), w32.size() * 4, cudaMemcpyHostToDevice));
  return DLIC_OK;
}

// ---------------------------------------------------------------- planning
dlic_status make_plan(uint32_t W, uint32_t H, uint32_t n, const dlic_opts* o, Plan& p,
                      const dlic_model* m = nullptr) {
  dlic_opts d = {DLIC_PREC_BF16, 32, 0, 0, 0, nullptr, 0};
  if (o) d = *o;
  if (d.group_rows == 0) d.group_rows = 32;
  if (d.n_meta > DLIC_MAX_META) return fail(DLIC_E_INVALID_ARG, "more than DLIC_MAX_META metadata reals");
  if (W == 0 || H == 0 || n == 0) return fail(DLIC_E_INVALID_ARG, "empty image or batch");
  if (W > 65535 * 16 || H > 65535 * 16) return fail(DLIC_E_INVALID_ARG, "image too large");
  if (d.precision > 1) return fail(DLIC_E_INVALID_ARG, "precision must be 0 (fp32) or 1 (bf16)");
  if (32 % d.group_rows != 0) return fail(DLIC_E_INVALID_ARG, "GPU path supports group_rows in {1,2,4,8,16,32}");
  const bool tiled = d.tile_w != 0 && d.tile_h != 0;
  if (tiled && (d.tile_w > 65535 || d.tile_h > 65535)) return fail(DLIC_E_INVALID_ARG, "tile too large");
  p = Plan{};
  p.W = W;
  p.H = H;
  p.n_img = n;
  p.G = d.group_rows;
  p.precision = d.precision;
  p.engine = d.precision;
  p.bits = 8;
  if (m && (m->p350k || m->p12)) {  // §8(f) f1 / f3: the streamed bf16 engines only
    if (d.precision != DLIC_PREC_BF16)
      return fail(DLIC_E_UNSUPPORTED_MODEL, "the 78->256x5->256/4096 models run in bf16 only");
    if (d.volume_depth > 0 || d.n_meta > 0)
      return fail(DLIC_E_UNSUPPORTED_MODEL, "the streamed-weight engines have no volume or metadata inputs");
    p.engine = m->p12 ? 3 : 2;
    p.bits = m->p12 ? 12 : 8;
  }
  if (m && m->p100k && d.precision == DLIC_PREC_FP32 && d.volume_depth == 0)
    p.engine = 4;  // fp32 on the tensor cores (bf16x3, dlic_x3.cuh); volumes keep the FFMA engine
  p.tw = tiled ? std::min(d.tile_w, W) : W;
  p.th = tiled ? std::min(d.tile_h, H) : H;
  p.hdr_tw = tiled ? d.tile_w : 0;
  p.hdr_th = tiled ? d.tile_h : 0;
  p.ntx = (W + p.tw - 1) / p.tw;
  p.nty = (H + p.th - 1) / p.th;
  p.upi = p.ntx * p.nty;
  p.gpt = (p.th + p.G - 1) / p.G;
  const uint32_t hl = H - (p.nty - 1) * p.th;
  p.gpl = (hl + p.G - 1) / p.G;
  p.spi = (p.nty - 1) * p.ntx * p.gpt + p.ntx * p.gpl;
  if (dec_smem_bytes(p.engine, std::max(p.gpt, (H - (p.nty - 1) * p.th + p.G - 1) / p.G),
                     d.volume_depth > 0 ? 1u : 0u) > dec_smem_limit())
    return fail(DLIC_E_INVALID_ARG, "too many row groups per unit for the decoder's shared memory: raise group_rows or tile");
  p.cap_words = 2 * p.G + p.G * p.tw;
  p.n_meta = d.n_meta;
  // volumes: depth slices per container (window id 2); 2D: one image each
  p.w3d = d.volume_depth > 0 ? 1u : 0u;
  p.depth = d.volume_depth > 0 ? d.volume_depth : 1u;
  if (n % p.depth) return fail(DLIC_E_SHAPE_MISMATCH, "image count is not a multiple of volume_depth");
  p.n_cont = n / p.depth;
  if ((uint64_t)p.spi * p.depth >= (1ull << 24)) return fail(DLIC_E_INVALID_ARG, "too many streams per volume");
  p.spc = p.spi * p.depth;
  p.hdr_bytes = HDR_FIXED + 4 * p.spc + 4 + 4 * p.n_meta;  // + the metadata block
  p.u_lo = 0;
  p.u_cnt = n * p.upi;
  p.s_lo = 0;
  p.s_cnt = n * p.spi;
  p.tiles_per_unit = (uint32_t)(((uint64_t)p.tw * p.th + ROWS - 1) / ROWS);
  if ((uint64_t)n * p.upi * p.tiles_per_unit >= (1ull << 32))
    return fail(DLIC_E_INVALID_ARG, "batch too large for one call (>= 2^32 encoder tiles): split it");
  const uint32_t slots = (p.tw + 2) / 3;  // max rows on one front = ceil(tw/3)
  p.nc = 0;
  for (uint32_t nc = 1; nc <= 16; nc *= 2)
    if (slots <= ROWS * nc) {
      p.nc = nc;
      break;
    }
  if (p.nc == 0) return fail(DLIC_E_INVALID_ARG, "unit wider than 3072 px: use tiles (tile_w <= 3072)");
  uint64_t mc = p.hdr_bytes;
  mc += (uint64_t)p.spc * (4ull * p.G + 2ull * p.G * p.tw);
  p.max_container = (mc + 15) & ~15ull;
  return DLIC_OK;
}

dlic_status check_model_gpu(const dlic_model* m) {
  if (!m) return fail(DLIC_E_INVALID_ARG, "null model");
  if (!m->p100k && !m->p350k && !m->p12)
    return fail(DLIC_E_UNSUPPORTED_MODEL, "GPU engines implement (78 + n_meta <= 8)->128x5->256 with optional "
                                          "power-of-two average pooling after hidden layers, and 78->256x5->256");
  return check_device(m->device);
}

// Per-image layer-1 biases with the metadata inputs folded in (k_meta_bias),
// or null when the model has none.  Raw reals from the host array `h_meta`
// ([n_img][n_meta], encode) or from the containers' metadata blocks on the
// device (`d_bits` + `d_cont_off`, decode).
dlic_status meta_bias(const dlic_model* m, const Plan& p, const float* h_meta, const uint8_t* d_bits,
                      const uint64_t* d_cont_off, cudaStream_t st, Scratch& sc, const float** out,
                      float** d_meta_out = nullptr);

// Restrict p to units [lo, hi) of image 0 (unit-range calls).
dlic_status restrict_units(Plan& p, uint32_t lo, uint32_t hi) {
  if (p.n_img != 1 || lo >= hi || hi > p.upi) return fail(DLIC_E_INVALID_ARG, "unit range outside [0, n_units)");
  p.u_lo = lo;
  p.u_cnt = hi - lo;
  p.s_lo = unit_info(p, lo).first_stream;
  p.s_cnt = (hi < p.upi ? unit_info(p, hi).first_stream : p.spi) - p.s_lo;
  return DLIC_OK;
}

// The decode launch for p must be schedulable on this device: a cluster of
// p.nc CTAs with the decoder's shared memory (16-CTA clusters are
// non-portable; checked once per (precision, nc, smem), on the current device).
dlic_status check_schedulable(const Plan& p) {
  static std::mutex mu;
  static std::map<std::tuple<int, uint32_t, uint32_t, size_t>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t sm = dec_smem_bytes(p.engine, std::max(p.gpt, p.gpl), p.w3d);
  const auto key = std::make_tuple(dev, p.engine, p.nc, sm);
  int n;
  {
    std::lock_guard<std::mutex> l(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      n = it->second;
    } else {
      n = dec_max_active_clusters(p.engine, p.nc, sm);
      cache[key] = n;
    }
  }
  if (n <= 0)
    return fail(DLIC_E_INVALID_ARG, "a " + std::to_string(p.nc) +
                                        "-CTA decode cluster cannot be scheduled on this device: use tiles (narrower units)");
  return DLIC_OK;
}

// ---------------------------------------------------------------- header parse
dlic_status peek(const uint8_t* b, size_t len, dlic_header* h, std::vector<uint32_t>* sizes) {
  if (!b || len < HDR_FIXED) return fail(DLIC_E_CORRUPT_CONTAINER, "container shorter than its header");
  if (memcmp(b, "DLIC", 4) != 0) return fail(DLIC_E_CORRUPT_CONTAINER, "container magic");
  if (b[4] != CONTAINER_VERSION || (b[6] != 1 && b[6] != 2))
    return fail(DLIC_E_VERSION_MISMATCH, "container version/window");
  if ((b[7] != 0 && b[7] != 12) || b[5] > 1) return fail(DLIC_E_CORRUPT_CONTAINER, "container alphabet/precision");
  dlic_header o = {};
  o.bits = b[7] == 12 ? 12 : 8;
  o.width = rd32(b + 8);
  o.height = rd32(b + 12);
  o.tile_w = rd16(b + 16);
  o.tile_h = rd16(b + 18);
  o.group_rows = rd16(b + 20);
  o.precision = b[5];
  o.numerics = rd16(b + 22);
  memcpy(o.model_sha256, b + 24, 32);
  o.n_streams = rd32(b + 56);
  if (o.width == 0 || o.height == 0 || o.group_rows == 0) return fail(DLIC_E_CORRUPT_CONTAINER, "header dims");
  if ((uint64_t)HDR_FIXED + 4ull * o.n_streams > len) return fail(DLIC_E_CORRUPT_CONTAINER, "size table");
  o.header_bytes = HDR_FIXED + 4ull * o.n_streams;
  uint64_t tot = 0;
  if (sizes) sizes->resize(o.n_streams);
  for (uint32_t s = 0; s < o.n_streams; ++s) {
    const uint32_t z = rd32(b + HDR_FIXED + 4 * s);
    if (z & 1) return fail(DLIC_E_CORRUPT_CONTAINER, "odd stream size");
    tot += z;
    if (sizes) (*sizes)[s] = z;
  }
  // metadata block: u32 n, f32 raw reals
  if (o.header_bytes + 4 > len) return fail(DLIC_E_CORRUPT_CONTAINER, "metadata block");
  o.n_meta = rd32(b + o.header_bytes);
  if (o.n_meta > DLIC_MAX_META || o.header_bytes + 4 + 4ull * o.n_meta > len)
    return fail(DLIC_E_CORRUPT_CONTAINER, "metadata block");
  for (uint32_t k = 0; k < o.n_meta; ++k) memcpy(&o.meta[k], b + o.header_bytes + 4 + 4 * k, 4);
  o.header_bytes += 4 + 4ull * o.n_meta;
  if (o.header_bytes + tot != len) return fail(DLIC_E_CORRUPT_CONTAINER, "container length");
  o.payload_bytes = tot;
  const bool tiled = o.tile_w && o.tile_h;
  const uint32_t tw = tiled ? std::min<uint32_t>(o.tile_w, o.width) : o.width;
  const uint32_t th = tiled ? std::min<uint32_t>(o.tile_h, o.height) : o.height;
  const uint32_t ntx = (o.width + tw - 1) / tw, nty = (o.height + th - 1) / th;
  const uint64_t spi = (uint64_t)(nty - 1) * ntx * ((th + o.group_rows - 1) / o.group_rows) +
                       (uint64_t)ntx * ((o.height - (nty - 1) * th + o.group_rows - 1) / o.group_rows);
  if (spi == 0 || o.n_streams % spi) return fail(DLIC_E_CORRUPT_CONTAINER, "stream count");
  o.depth = b[6] == 2 ? (uint32_t)(o.n_streams / spi) : 0u;
  if (b[6] == 1 && o.n_streams != spi) return fail(DLIC_E_CORRUPT_CONTAINER, "stream count");
  o.n_units = ntx * nty * (o.depth ? o.depth : 1u);
  *h = o;
  return DLIC_OK;
}

dlic_opts opts_of(const dlic_header& h) {
  dlic_opts o;
  o.precision = h.precision;
  o.group_rows = h.group_rows;
  o.tile_w = h.tile_w;
  o.tile_h = h.tile_h;
  o.n_meta = h.n_meta;
  o.meta = h.meta;  // points into h
  o.volume_depth = h.depth;
  return o;
}

// copy a host buffer to device through pinned staging when needed
cudaError_t h2d(void* dst, const void* src, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (is_pinned(src)) return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st);
  void* pin = g_pin_in.get(n);
  if (!pin) return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st);
  cudaError_t e = cudaStreamSynchronize(st);  // staging buffer may still be in flight
  if (e != cudaSuccess) return e;
  par_memcpy(pin, src, n);
  return cudaMemcpyAsync(dst, pin, n, cudaMemcpyHostToDevice, st);
}

// metadata staging: a pageable copy would block the host mid-pipeline; the
// event marks the buffer's last copy, so reuse waits for that copy only
thread_local Pinned g_pin_meta;
thread_local cudaEvent_t g_pin_meta_ev = nullptr;

dlic_status meta_bias(const dlic_model* m, const Plan& p, const float* h_meta, const uint8_t* d_bits,
                      const uint64_t* d_cont_off, cudaStream_t st, Scratch& sc, const float** out,
                      float** d_meta_out) {
  *out = nullptr;
  if (d_meta_out) *d_meta_out = nullptr;
  if ((p.w3d != 0) != m->in3d)
    return fail(DLIC_E_SHAPE_MISMATCH, m->in3d ? "a 3D-window model codes volumes (opts.volume_depth >= 1)"
                                               : "volumes need a 3D-window model (87 window inputs)");
  if (p.n_meta != m->n_meta)
    return fail(DLIC_E_SHAPE_MISMATCH, "metadata count " + std::to_string(p.n_meta) + " != the model's " +
                                           std::to_string(m->n_meta));
  if (m->n_meta == 0) return DLIC_OK;
  if (!d_bits && !h_meta) return fail(DLIC_E_INVALID_ARG, "the model needs metadata (opts.meta)");
  float* d_out;
  float* d_meta = nullptr;
  CUDA_TRY(sc.alloc(&d_out, 4ull * p.n_cont * HID));
  if (!d_bits) {
    const size_t nb = 4ull * p.n_cont * p.n_meta;
    CUDA_TRY(sc.alloc(&d_meta, nb));
    void* pin = g_pin_meta.get(nb);
    if (pin) {
      if (!g_pin_meta_ev) CUDA_TRY(cudaEventCreateWithFlags(&g_pin_meta_ev, cudaEventDisableTiming));
      else CUDA_TRY(cudaEventSynchronize(g_pin_meta_ev));  // the buffer's previous copy is done
      memcpy(pin, h_meta, nb);
      CUDA_TRY(cudaMemcpyAsync(d_meta, pin, nb, cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaEventRecord(g_pin_meta_ev, st));
    } else {
      CUDA_TRY(cudaMemcpyAsync(d_meta, h_meta, nb, cudaMemcpyHostToDevice, st));
    }
    if (d_meta_out) *d_meta_out = d_meta;
  }
  CUDA_TRY(launch_meta_bias(p.n_cont, p.n_meta, d_meta, d_bits, d_cont_off, HDR_FIXED + 4u * p.spc + 4u, m->d_range,
                            m->d_wmeta, m->d_bias, p.precision, d_out, st));
  *out = d_out;
  return DLIC_OK;
}

// volumes: the decoder's unit ticket + per-unit progress flags (zeroed)
dlic_status alloc_sync(const Plan& p, Scratch& sc, cudaStream_t st, uint32_t** out) {
  *out = nullptr;
  const size_t n = sync_words(p);
  if (!n) return DLIC_OK;
  CUDA_TRY(sc.alloc(out, 4 * n));
  CUDA_TRY(cudaMemsetAsync(*out, 0, 4 * n, st));
  return DLIC_OK;
}

// encode pipeline on device buffers (shared by dlic_encode and the batch API)
dlic_status run_encode(const dlic_model* m, const Plan& p, const uint8_t* d_imgs, uint8_t* d_out, uint64_t stride,
                       uint64_t* d_sizes, cudaStream_t st, Scratch& sc, const float* h_meta,
                       uint32_t** words_out = nullptr) {
  uint32_t* d_fc;
  uint16_t* d_scr;
  uint32_t* d_words;
  uint64_t* d_dst;
  const uint64_t npx = (uint64_t)p.n_img * p.W * p.H;
  const uint64_t ns = (uint64_t)p.n_img * p.spi;
  CUDA_TRY(sc.alloc(&d_fc, 4 * npx));
  CUDA_TRY(sc.alloc(&d_scr, 2ull * p.cap_words * ns));
  CUDA_TRY(sc.alloc(&d_words, 4 * ns));
  CUDA_TRY(sc.alloc(&d_dst, 8 * ns));
  const float* b1img = nullptr;
  float* d_meta = nullptr;  // raw reals, also for the containers' metadata blocks
  dlic_status s = meta_bias(m, p, h_meta, nullptr, nullptr, st, sc, &b1img, &d_meta);
  if (s != DLIC_OK) return s;
  ev_begin("mlp", st);
  CUDA_TRY(launch_enc_mlp(p, m->dw(b1img, p.engine), d_imgs, d_fc, nullptr, nullptr, nullptr, st, num_sms(m->device)));
  ev_end("mlp", st);
  ev_begin("rans_enc", st);
  CUDA_TRY(launch_rans_enc(p, d_fc, d_scr, d_words, st));
  ev_end("rans_enc", st);
  ev_begin("compact", st);
  CUDA_TRY(launch_container(p, m->sha, d_words, d_scr, d_out, stride, d_sizes, d_dst, st, words_out != nullptr, d_meta));
  ev_end("compact", st);
  if (words_out) *words_out = d_words;
  return DLIC_OK;
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

const char* dlic_status_str(dlic_status s) {
  switch (s) {
    case DLIC_OK: return "ok";
    case DLIC_E_INVALID_ARG: return "invalid argument";
    case DLIC_E_SHAPE_MISMATCH: return "shape mismatch";
    case DLIC_E_NONCAUSAL_WINDOW: return "non-causal window";
    case DLIC_E_CORRUPT_MODEL: return "corrupt model";
    case DLIC_E_VERSION_MISMATCH: return "version mismatch";
    case DLIC_E_CORRUPT_CONTAINER: return "corrupt container";
    case DLIC_E_MODEL_HASH_MISMATCH: return "model hash mismatch";
    case DLIC_E_STREAM_UNDERFLOW: return "stream underflow";
    case DLIC_E_SUM_MISMATCH: return "frequency sum mismatch";
    case DLIC_E_ZERO_FREQUENCY: return "zero frequency";
    case DLIC_E_BUFFER_TOO_SMALL: return "buffer too small";
    case DLIC_E_CUDA: return "CUDA error";
    case DLIC_E_OUT_OF_MEMORY: return "out of memory";
    case DLIC_E_UNSUPPORTED_MODEL: return "unsupported model architecture";
  }
  return "unknown status";
}

const char* dlic_last_error(void) { return g_err.c_str(); }

void dlic_free(void* p) { free(p); }

dlic_status dlic_model_blob_check(const void* bytes, size_t len, uint8_t sha_out[32]) {
  ParsedModel pm;
  return parse_model(static_cast<const uint8_t*>(bytes), len, pm, sha_out);
}

dlic_status dlic_model_load(const void* bytes, size_t len, int cuda_device, dlic_model** out) {
  if (!out) return fail(DLIC_E_INVALID_ARG, "null out");
  ParsedModel pm;
  uint8_t sha[32];
  dlic_status s = parse_model(static_cast<const uint8_t*>(bytes), len, pm, sha);
  if (s != DLIC_OK) return s;
  s = check_device(cuda_device);
  if (s != DLIC_OK) return s;
  dlic_model* m = new dlic_model();
  m->device = cuda_device;
  m->blob.assign(static_cast<const uint8_t*>(bytes), static_cast<const uint8_t*>(bytes) + len);
  memcpy(m->sha, sha, 32);
  s = upload_model(m, pm);
  if (s != DLIC_OK) {
    dlic_model_free(m);
    return s;
  }
  *out = m;
  return DLIC_OK;
}

dlic_status dlic_model_from_arrays(uint32_t n_layers, const uint32_t* dims, const float* const* W,
                                   const float* const* b, int cuda_device, dlic_model** out) {
  if (!dims || !W || !b || n_layers == 0 || n_layers > 64) return fail(DLIC_E_INVALID_ARG, "bad arrays");
  std::vector<uint8_t> blob(8);
  memcpy(blob.data(), "DLICMDL1", 8);
  auto put16 = [&](uint32_t v) { blob.push_back((uint8_t)v); blob.push_back((uint8_t)(v >> 8)); };
  auto put32 = [&](uint32_t v) { for (int i = 0; i < 4; ++i) blob.push_back((uint8_t)(v >> (8 * i))); };
  put16(n_layers);
  for (uint32_t l = 0; l < n_layers; ++l) {
    put32(dims[l]);
    put32(dims[l + 1]);
    blob.push_back(l + 1 < n_layers ? 1 : 0);
    blob.push_back(0);
    const uint8_t* wp = reinterpret_cast<const uint8_t*>(W[l]);
    blob.insert(blob.end(), wp, wp + 4ull * dims[l] * dims[l + 1]);
    const uint8_t* bp = reinterpret_cast<const uint8_t*>(b[l]);
    blob.insert(blob.end(), bp, bp + 4ull * dims[l + 1]);
  }
  put16(0);
  uint8_t h[32];
  sha256(blob.data(), blob.size(), h);
  blob.insert(blob.end(), h, h + 32);
  return dlic_model_load(blob.data(), blob.size(), cuda_device, out);
}

void dlic_model_free(dlic_model* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  if (m->d_wimg) cudaFree(m->d_wimg);
  if (m->d_x3img) cudaFree(m->d_x3img);
  if (m->d_x3bias) cudaFree(m->d_x3bias);
  if (m->d_bias) cudaFree(m->d_bias);
  if (m->d_w32) cudaFree(m->d_w32);
  if (m->d_wmeta) cudaFree(m->d_wmeta);
  if (m->d_range) cudaFree(m->d_range);
  delete m;
}

dlic_status dlic_model_sha256(const dlic_model* m, uint8_t out[32]) {
  if (!m || !out) return fail(DLIC_E_INVALID_ARG, "null");
  memcpy(out, m->sha, 32);
  return DLIC_OK;
}

size_t dlic_max_container_bytes(uint32_t width, uint32_t height, const dlic_opts* opts) {
  Plan p;  // one container: one image, or one volume of volume_depth slices
  if (make_plan(width, height, opts && opts->volume_depth ? opts->volume_depth : 1u, opts, p) != DLIC_OK) return 0;
  return p.max_container;
}

dlic_status dlic_peek(const uint8_t* bits, size_t len, dlic_header* out) {
  if (!out) return fail(DLIC_E_INVALID_ARG, "null out");
  return peek(bits, len, out, nullptr);
}

dlic_status dlic_encode(const dlic_model* m, const uint8_t* img, uint32_t width, uint32_t height, size_t row_stride,
                        const dlic_opts* opts, uint8_t** out, size_t* out_len) {
  if (!img || !out || !out_len) return fail(DLIC_E_INVALID_ARG, "null pointer");
  if (row_stride == 0) row_stride = width;
  if (row_stride < width) return fail(DLIC_E_SHAPE_MISMATCH, "row_stride < width");
  dlic_status s = check_model_gpu(m);
  if (s != DLIC_OK) return s;
  Plan p;
  s = make_plan(width, height, 1, opts, p, m);
  if (s != DLIC_OK) return s;
  s = check_schedulable(p);  // never write a container this device cannot decode
  if (s != DLIC_OK) return s;
  cudaStream_t st = my_stream();
  Scratch sc(st);
  uint8_t *d_img, *d_out;
  uint64_t* d_size;
  const size_t pxb = p.bits == 12 ? 2 : 1;  // bytes per pixel (12-bit: u16)
  CUDA_TRY(sc.alloc(&d_img, (size_t)width * height * pxb));
  CUDA_TRY(sc.alloc(&d_out, p.max_container));
  CUDA_TRY(sc.alloc(&d_size, 8));
  if (row_stride == width) {
    CUDA_TRY(h2d(d_img, img, (size_t)width * height * pxb, st));
  } else {
    CUDA_TRY(cudaMemcpy2DAsync(d_img, width * pxb, img, row_stride * pxb, width * pxb, height, cudaMemcpyHostToDevice,
                               st));
  }
  s = run_encode(m, p, d_img, d_out, p.max_container, d_size, st, sc, opts ? opts->meta : nullptr);
  if (s != DLIC_OK) return s;
  uint64_t* hs = static_cast<uint64_t*>(g_pin_out.get(p.max_container + 64));
  if (!hs) return fail(DLIC_E_OUT_OF_MEMORY, "pinned staging");
  CUDA_TRY(cudaMemcpyAsync(hs, d_size, 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const uint64_t n = hs[0];
  if (n > p.max_container) return fail(DLIC_E_CUDA, "container size out of range");
  uint8_t* hb = reinterpret_cast<uint8_t*>(hs) + 64;
  CUDA_TRY(cudaMemcpyAsync(hb, d_out, n, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  uint8_t* res = static_cast<uint8_t*>(malloc(n));
  if (!res) return fail(DLIC_E_OUT_OF_MEMORY, "malloc");
  par_memcpy(res, hb, n);
  *out = res;
  *out_len = n;
  return DLIC_OK;
}

static dlic_status decode_common(const dlic_model* m, const uint8_t* bits, size_t len, const uint16_t* tables,
                                 uint8_t* img, size_t cap, uint32_t unit_lo = 0, uint32_t unit_hi = 0) {
  dlic_header h;
  dlic_status s = peek(bits, len, &h, nullptr);
  if (s != DLIC_OK) return s;
  if (m && memcmp(h.model_sha256, m->sha, 32) != 0)
    return fail(DLIC_E_MODEL_HASH_MISMATCH, "container was coded with another model");
  if (m && h.numerics != NUMERICS_REV)
    return fail(DLIC_E_VERSION_MISMATCH, "container tables come from another arithmetic revision (numerics " +
                                             std::to_string(h.numerics) + ", this build " +
                                             std::to_string(NUMERICS_REV) + ")");
  const uint32_t nsl = h.depth ? h.depth : 1u;  // slices (a volume container holds depth of them)
  const size_t npx = (size_t)h.width * h.height * nsl;
  const size_t pxb = h.bits == 12 ? 2 : 1;  // bytes per pixel (12-bit: u16)
  if (m && h.bits != (m->p12 ? 12u : 8u))
    return fail(DLIC_E_SHAPE_MISMATCH, "container alphabet does not match the model's output layer");
  if (tables && h.bits != 8) return fail(DLIC_E_INVALID_ARG, "table-fed decode is for 8-bit containers");
  if (!img || cap < npx * pxb) return fail(DLIC_E_BUFFER_TOO_SMALL, "image buffer");
  if (m) {
    s = check_model_gpu(m);
  } else {
    int dev = 0;
    cudaGetDevice(&dev);
    s = check_device(dev);
  }
  if (s != DLIC_OK) return s;
  dlic_opts o = opts_of(h);
  Plan p;
  s = make_plan(h.width, h.height, nsl, &o, p, m);
  if (s != DLIC_OK) return s;
  if (p.spc != h.n_streams) return fail(DLIC_E_CORRUPT_CONTAINER, "stream count does not match the header dims");
  const bool part = unit_hi > 0;  // dlic_decode_units: only units [unit_lo, unit_hi)
  if (part && (p.depth > 1 || p.bits != 8)) return fail(DLIC_E_INVALID_ARG, "unit ranges are for 2D 8-bit images");
  if (part) {
    s = restrict_units(p, unit_lo, unit_hi);
    if (s != DLIC_OK) return s;
  }
  if (!tables) {
    s = check_schedulable(p);
    if (s != DLIC_OK) return s;
  }
  cudaStream_t st = my_stream();
  Scratch sc(st);
  uint8_t *d_bits, *d_img;
  uint32_t *d_sbase, *d_slen;
  int32_t* d_status;
  uint64_t* d_meta;  // [0] = container offset (0), [1] = length
  CUDA_TRY(sc.alloc(&d_bits, len));
  CUDA_TRY(sc.alloc(&d_img, npx * pxb));
  CUDA_TRY(sc.alloc(&d_sbase, 4ull * p.spc));
  CUDA_TRY(sc.alloc(&d_slen, 4ull * p.spc));
  CUDA_TRY(sc.alloc(&d_status, 4));
  CUDA_TRY(sc.alloc(&d_meta, 16));
  uint8_t* pin = static_cast<uint8_t*>(g_pin_in.get(len + 16));
  if (!pin) return fail(DLIC_E_OUT_OF_MEMORY, "pinned staging");
  CUDA_TRY(cudaStreamSynchronize(st));
  uint64_t meta[2] = {0, (uint64_t)len};
  memcpy(pin, meta, 16);
  par_memcpy(pin + 16, bits, len);
  CUDA_TRY(cudaMemcpyAsync(d_meta, pin, 16, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_bits, pin + 16, len, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_dec_prep(p, d_bits, d_meta, d_meta + 1, d_sbase, d_slen, d_status, st, tables == nullptr));
  if (part)  // pixels outside the unit range come back untouched (pageable copy: no staging reuse)
    CUDA_TRY(cudaMemcpyAsync(d_img, img, npx * pxb, cudaMemcpyHostToDevice, st));
  if (tables) {
    uint16_t* d_tab;
    const size_t tb = npx * NOUT * 2;
    CUDA_TRY(sc.alloc(&d_tab, tb));
    CUDA_TRY(cudaMemcpyAsync(d_tab, tables, tb, cudaMemcpyHostToDevice, st));
    ev_begin("decode", st);
    CUDA_TRY(launch_rans_dec_tables(p, d_bits, d_sbase, d_slen, d_tab, d_img, d_status, st));
    ev_end("decode", st);
  } else {
    unsigned long long* d_prof = nullptr;
    const bool prof = getenv("DLIC_PROF") != nullptr;
    if (prof) {
      CUDA_TRY(sc.alloc(&d_prof, 300 * 8));
      CUDA_TRY(cudaMemsetAsync(d_prof, 0, 300 * 8, st));
    }
    ev_begin("decode", st);
    const float* b1img = nullptr;  // metadata re-read from the container (device)
    s = meta_bias(m, p, nullptr, d_bits, d_meta, st, sc, &b1img);
    if (s != DLIC_OK) return s;
    uint32_t* d_sync;
    s = alloc_sync(p, sc, st, &d_sync);
    if (s != DLIC_OK) return s;
    CUDA_TRY(launch_decode(p, m->dw(b1img, p.engine), d_bits, d_meta, d_sbase, d_slen, d_img, d_status, st, d_prof, d_sync));
    ev_end("decode", st);
    if (prof) {
      unsigned long long hp[40];
      CUDA_TRY(cudaMemcpyAsync(hp, d_prof, 40 * 8, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      const double ctas = (double)p.n_img * p.upi * p.nc;
      const double T = (double)(p.tw + 3 * (p.th - 1));  // per-slice fronts
      const char* nm[11] = {"top", "gather", "put", "mlp", "pass1", "xchg", "bar7", "passA", "search", "rans",
                            "barrier"};
      fprintf(stderr, "[dlic prof] cycles per front per CTA:");
      for (int k = 0; k < 11; ++k) fprintf(stderr, " %s %.0f", nm[k], hp[k] / ctas / T);
      fprintf(stderr, "\n[dlic prof] sub-phases (pass1 for bf16 decode): ld32 %.0f early-signal %.0f s1a %.0f s1b+s1c %.0f\n", hp[16] / ctas / T, hp[17] / ctas / T, hp[18] / ctas / T, hp[19] / ctas / T);
      if (p.precision == 1)
        fprintf(stderr, "[dlic prof] issuer per front: network issue %.0f  arrive->layer-1 issued %.0f  cluster wait %.0f\n",
                hp[26] / ctas / T, hp[27] / ctas / T, hp[28] / ctas / T);
      if (p.w3d)
        fprintf(stderr, "[dlic prof] 3D: waits for the slice below %.3f per front per CTA, %.0f cycles per wait\n",
                hp[24] / ctas / T, hp[24] ? (double)hp[25] / hp[24] : 0.0);
    }
  }
  uint8_t* ho = static_cast<uint8_t*>(g_pin_out.get(npx * pxb + 64));
  if (!ho) return fail(DLIC_E_OUT_OF_MEMORY, "pinned staging");
  CUDA_TRY(cudaMemcpyAsync(ho, d_status, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(ho + 64, d_img, npx * pxb, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  int32_t stat;
  memcpy(&stat, ho, 4);
  if (stat != 0) return fail((dlic_status)stat, "lane invariant / framing check failed on the device");
  par_memcpy(img, ho + 64, npx * pxb);
  return DLIC_OK;
}

dlic_status dlic_decode(const dlic_model* m, const uint8_t* bits, size_t len, uint8_t* img, size_t img_capacity) {
  if (!m) return fail(DLIC_E_INVALID_ARG, "null model");
  return decode_common(m, bits, len, nullptr, img, img_capacity);
}

dlic_status dlic_rans_decode_tables(const uint8_t* bits, size_t len, const uint16_t* freq_tables, uint8_t* img) {
  if (!freq_tables) return fail(DLIC_E_INVALID_ARG, "null tables");
  dlic_header h;
  dlic_status s = peek(bits, len, &h, nullptr);
  if (s != DLIC_OK) return s;
  return decode_common(nullptr, bits, len, freq_tables, img, (size_t)h.width * h.height * (h.depth ? h.depth : 1u));
}

dlic_status dlic_rans_encode_tables(const uint32_t* fc, uint32_t width, uint32_t height, const dlic_opts* opts,
                                    const uint8_t* model_sha256, uint8_t** out, size_t* out_len) {
  if (!fc || !out || !out_len) return fail(DLIC_E_INVALID_ARG, "null pointer");
  int dev = 0;
  cudaGetDevice(&dev);
  dlic_status s = check_device(dev);
  if (s != DLIC_OK) return s;
  const uint32_t nsl = opts && opts->volume_depth ? opts->volume_depth : 1u;  // a volume: fc[z][r][c]
  const size_t npx = (size_t)width * height * nsl;
  Plan p;
  s = make_plan(width, height, nsl, opts, p);
  if (s != DLIC_OK) return s;
  // tables must be valid: f >= 1 and c + f <= 2^16
  for (size_t i = 0; i < npx; ++i) {
    const uint32_t f = fc[i] & 0xFFFF, c = fc[i] >> 16;
    if (f == 0) return fail(DLIC_E_ZERO_FREQUENCY, "f_s == 0");
    if (c + f > 65536) return fail(DLIC_E_SUM_MISMATCH, "c_s + f_s > 2^16");
  }
  // fc arrives in image raster order; the kernels read it unit by unit
  std::vector<uint32_t> fcu(npx);
  for (uint32_t u = 0; u < p.upi * nsl; ++u) {
    const Unit un = unit_info(p, u);
    const size_t sl = (size_t)un.img * width * height;
    for (uint32_t r = 0; r < un.h; ++r)
      memcpy(&fcu[un.fc_off + (size_t)r * un.w], &fc[sl + (size_t)(un.y0 + r) * width + un.x0], 4ull * un.w);
  }
  cudaStream_t st = my_stream();
  Scratch sc(st);
  uint32_t *d_fc, *d_words;
  uint16_t* d_scr;
  uint64_t *d_dst, *d_size;
  uint8_t* d_out;
  const uint64_t ns = p.spc;
  CUDA_TRY(sc.alloc(&d_fc, 4ull * npx));
  CUDA_TRY(sc.alloc(&d_scr, 2ull * p.cap_words * ns));
  CUDA_TRY(sc.alloc(&d_words, 4 * ns));
  CUDA_TRY(sc.alloc(&d_dst, 8 * ns));
  CUDA_TRY(sc.alloc(&d_size, 8));
  CUDA_TRY(sc.alloc(&d_out, p.max_container));
  CUDA_TRY(cudaMemcpyAsync(d_fc, fcu.data(), 4ull * npx, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_rans_enc(p, d_fc, d_scr, d_words, st));
  float* d_mraw = nullptr;
  if (p.n_meta) {
    if (!opts->meta) return fail(DLIC_E_INVALID_ARG, "opts.n_meta > 0 but opts.meta is null");
    CUDA_TRY(sc.alloc(&d_mraw, 4ull * p.n_meta));
    CUDA_TRY(cudaMemcpyAsync(d_mraw, opts->meta, 4ull * p.n_meta, cudaMemcpyHostToDevice, st));
  }
  CUDA_TRY(launch_container(p, model_sha256, d_words, d_scr, d_out, p.max_container, d_size, d_dst, st, false,
                            d_mraw));
  uint64_t n = 0;
  CUDA_TRY(cudaMemcpyAsync(&n, d_size, 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  uint8_t* res = static_cast<uint8_t*>(malloc(n));
  if (!res) return fail(DLIC_E_OUT_OF_MEMORY, "malloc");
  CUDA_TRY(cudaMemcpyAsync(res, d_out, n, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *out = res;
  *out_len = n;
  return DLIC_OK;
}

dlic_status dlic_debug_mlp(const dlic_model* m, const uint8_t* img, uint32_t width, uint32_t height,
                           const dlic_opts* opts, float* logits, float* probs, uint16_t* freqs, uint32_t* fc) {
  if (!img) return fail(DLIC_E_INVALID_ARG, "null image");
  dlic_status s = check_model_gpu(m);
  if (s != DLIC_OK) return s;
  const uint32_t nsl = opts && opts->volume_depth ? opts->volume_depth : 1u;  // a volume: img holds nsl slices
  Plan p;
  s = make_plan(width, height, nsl, opts, p, m);
  if (s != DLIC_OK) return s;
  cudaStream_t st = my_stream();
  Scratch sc(st);
  const size_t npx = (size_t)width * height * nsl;
  const size_t pxb = p.bits == 12 ? 2 : 1;                 // bytes per pixel
  const size_t nout = p.bits == 12 ? (size_t)H12_N : NOUT;  // table entries per pixel
  uint8_t* d_img;
  uint32_t* d_fc;
  float *d_lg = nullptr, *d_pb = nullptr;
  uint16_t* d_fq = nullptr;
  CUDA_TRY(sc.alloc(&d_img, npx * pxb));
  CUDA_TRY(sc.alloc(&d_fc, 4 * npx));
  if (logits) CUDA_TRY(sc.alloc(&d_lg, 4 * npx * nout));
  if (probs) CUDA_TRY(sc.alloc(&d_pb, 4 * npx * nout));
  if (freqs) CUDA_TRY(sc.alloc(&d_fq, 2 * npx * nout));
  CUDA_TRY(cudaMemcpyAsync(d_img, img, npx * pxb, cudaMemcpyHostToDevice, st));
  const float* b1img = nullptr;
  s = meta_bias(m, p, opts ? opts->meta : nullptr, nullptr, nullptr, st, sc, &b1img);
  if (s != DLIC_OK) return s;
  CUDA_TRY(launch_enc_mlp(p, m->dw(b1img, p.engine), d_img, d_fc, d_lg, d_pb, d_fq, st, num_sms(m->device)));
  if (logits) CUDA_TRY(cudaMemcpyAsync(logits, d_lg, 4 * npx * nout, cudaMemcpyDeviceToHost, st));
  if (probs) CUDA_TRY(cudaMemcpyAsync(probs, d_pb, 4 * npx * nout, cudaMemcpyDeviceToHost, st));
  if (freqs) CUDA_TRY(cudaMemcpyAsync(freqs, d_fq, 2 * npx * nout, cudaMemcpyDeviceToHost, st));
  std::vector<uint32_t> fcu;
  if (fc) {
    fcu.resize(npx);
    CUDA_TRY(cudaMemcpyAsync(fcu.data(), d_fc, 4 * npx, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  if (fc) {
    for (uint32_t u = 0; u < p.upi * nsl; ++u) {
      const Unit un = unit_info(p, u);
      const size_t sl = (size_t)un.img * width * height;
      for (uint32_t r = 0; r < un.h; ++r)
        memcpy(&fc[sl + (size_t)(un.y0 + r) * width + un.x0], &fcu[un.fc_off + (size_t)r * un.w], 4ull * un.w);
    }
  }
  return DLIC_OK;
}

dlic_status dlic_encode_batch(const dlic_model* m, const uint8_t* imgs, uint32_t n, uint32_t width,
                              uint32_t height, const dlic_opts* opts, uint8_t** out, size_t* out_len,
                              uint64_t* sizes) {
  if (!imgs || !out || !out_len || !sizes || n == 0) return fail(DLIC_E_INVALID_ARG, "null pointer or n = 0");
  dlic_status s = check_model_gpu(m);
  if (s != DLIC_OK) return s;
  Plan p;
  s = make_plan(width, height, n, opts, p, m);
  if (s != DLIC_OK) return s;
  s = check_schedulable(p);
  if (s != DLIC_OK) return s;
  cudaStream_t st = my_stream();
  Scratch sc(st);
  const size_t npx = (size_t)n * width * height * (p.bits == 12 ? 2 : 1);  // image bytes
  uint8_t *d_imgs, *d_out;
  uint64_t* d_sizes;
  CUDA_TRY(sc.alloc(&d_imgs, npx));
  const uint32_t nc = p.n_cont;  // containers (volumes hold volume_depth images each)
  CUDA_TRY(sc.alloc(&d_out, p.max_container * nc));
  CUDA_TRY(sc.alloc(&d_sizes, 8ull * nc));
  CUDA_TRY(h2d(d_imgs, imgs, npx, st));
  s = run_encode(m, p, d_imgs, d_out, p.max_container, d_sizes, st, sc, opts ? opts->meta : nullptr);
  if (s != DLIC_OK) return s;
  std::vector<uint64_t> hs(nc);
  CUDA_TRY(cudaMemcpyAsync(hs.data(), d_sizes, 8ull * nc, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  uint64_t total = 0;
  for (uint32_t i = 0; i < nc; ++i) {
    if (hs[i] > p.max_container) return fail(DLIC_E_CUDA, "container size out of range");
    total += hs[i];
  }
  // pack the containers back to back on the device, then one D2H
  uint8_t* d_pack;
  CUDA_TRY(sc.alloc(&d_pack, total));
  uint64_t off = 0;
  for (uint32_t i = 0; i < nc; ++i) {
    CUDA_TRY(cudaMemcpyAsync(d_pack + off, d_out + (size_t)i * p.max_container, hs[i], cudaMemcpyDeviceToDevice,
                             st));
    off += hs[i];
  }
  uint8_t* hb = static_cast<uint8_t*>(g_pin_out.get(total + 64));
  if (!hb) return fail(DLIC_E_OUT_OF_MEMORY, "pinned staging");
  CUDA_TRY(cudaMemcpyAsync(hb, d_pack, total, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  uint8_t* res = static_cast<uint8_t*>(malloc(total ? total : 1));
  if (!res) return fail(DLIC_E_OUT_OF_MEMORY, "malloc");
  par_memcpy(res, hb, total);
  for (uint32_t i = 0; i < nc; ++i) sizes[i] = hs[i];
  *out = res;
  *out_len = total;
  return DLIC_OK;
}

dlic_status dlic_decode_batch(const dlic_model* m, const uint8_t* bits, size_t len, const uint64_t* offsets,
                              uint32_t n, uint8_t* imgs, size_t img_capacity) {
  if (!bits || !offsets || !imgs || n == 0) return fail(DLIC_E_INVALID_ARG, "null pointer or n = 0");
  dlic_status s = check_model_gpu(m);
  if (s != DLIC_OK) return s;
  std::vector<uint64_t> lens(n);
  dlic_header h0;
  for (uint32_t i = 0; i < n; ++i) {
    const uint64_t end = i + 1 < n ? offsets[i + 1] : (uint64_t)len;
    if (offsets[i] > end || end > len) return fail(DLIC_E_INVALID_ARG, "offsets not ascending within len");
    lens[i] = end - offsets[i];
    dlic_header h;
    s = peek(bits + offsets[i], lens[i], &h, nullptr);
    if (s != DLIC_OK) return s;
    if (memcmp(h.model_sha256, m->sha, 32) != 0)
      return fail(DLIC_E_MODEL_HASH_MISMATCH, "container was coded with another model");
    if (h.numerics != NUMERICS_REV)
      return fail(DLIC_E_VERSION_MISMATCH, "container tables come from another arithmetic revision");
    if (i == 0) {
      h0 = h;
    } else if (h.width != h0.width || h.height != h0.height || h.precision != h0.precision || h.depth != h0.depth ||
               h.group_rows != h0.group_rows || h.tile_w != h0.tile_w || h.tile_h != h0.tile_h) {
      return fail(DLIC_E_SHAPE_MISMATCH, "batch containers differ in dims or options");
    }
  }
  if (h0.bits != (m->p12 ? 12u : 8u))
    return fail(DLIC_E_SHAPE_MISMATCH, "container alphabet does not match the model's output layer");
  const size_t npx = (size_t)n * h0.width * h0.height * (h0.depth ? h0.depth : 1u) * (h0.bits == 12 ? 2 : 1);  // bytes
  if (img_capacity < npx) return fail(DLIC_E_BUFFER_TOO_SMALL, "image buffer");
  dlic_opts o = opts_of(h0);
  Plan p;
  s = make_plan(h0.width, h0.height, n * (h0.depth ? h0.depth : 1u), &o, p, m);
  if (s != DLIC_OK) return s;
  if (p.spc != h0.n_streams) return fail(DLIC_E_CORRUPT_CONTAINER, "stream count does not match the header dims");
  s = check_schedulable(p);
  if (s != DLIC_OK) return s;
  cudaStream_t st = my_stream();
  Scratch sc(st);
  uint8_t *d_bits, *d_imgs;
  uint64_t* d_meta;  // [0, n) offsets, [n, 2n) lengths
  uint32_t *d_sbase, *d_slen;
  int32_t* d_status;
  CUDA_TRY(sc.alloc(&d_bits, len));
  CUDA_TRY(sc.alloc(&d_imgs, npx));
  CUDA_TRY(sc.alloc(&d_meta, 16ull * n));
  CUDA_TRY(sc.alloc(&d_sbase, 4ull * n * p.spc));
  CUDA_TRY(sc.alloc(&d_slen, 4ull * n * p.spc));
  CUDA_TRY(sc.alloc(&d_status, 4ull * n));
  CUDA_TRY(cudaMemsetAsync(d_status, 0, 4ull * n, st));
  std::vector<uint64_t> meta(2ull * n);
  for (uint32_t i = 0; i < n; ++i) {
    meta[i] = offsets[i];
    meta[n + i] = lens[i];
  }
  CUDA_TRY(cudaMemcpyAsync(d_meta, meta.data(), 16ull * n, cudaMemcpyHostToDevice, st));
  CUDA_TRY(h2d(d_bits, bits, len, st));
  CUDA_TRY(launch_dec_prep(p, d_bits, d_meta, d_meta + n, d_sbase, d_slen, d_status, st));
  const float* b1img = nullptr;
  s = meta_bias(m, p, nullptr, d_bits, d_meta, st, sc, &b1img);
  if (s != DLIC_OK) return s;
  ev_begin("decode", st);
  uint32_t* d_sync;
  s = alloc_sync(p, sc, st, &d_sync);
  if (s != DLIC_OK) return s;
  CUDA_TRY(launch_decode(p, m->dw(b1img, p.engine), d_bits, d_meta, d_sbase, d_slen, d_imgs, d_status, st, nullptr, d_sync));
  ev_end("decode", st);
  uint8_t* ho = static_cast<uint8_t*>(g_pin_out.get(npx + 4ull * n + 64));
  if (!ho) return fail(DLIC_E_OUT_OF_MEMORY, "pinned staging");
  CUDA_TRY(cudaMemcpyAsync(ho, d_status, 4ull * n, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(ho + ((4ull * n + 63) & ~63ull), d_imgs, npx, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (uint32_t i = 0; i < n; ++i) {
    int32_t stat;
    memcpy(&stat, ho + 4ull * i, 4);
    if (stat != 0) return fail((dlic_status)stat, "lane invariant / framing check failed on the device (image " +
                                                      std::to_string(i) + ")");
  }
  par_memcpy(imgs, ho + ((4ull * n + 63) & ~63ull), npx);
  return DLIC_OK;
}

dlic_status dlic_encode_batch_device(const dlic_model* m, const uint8_t* d_imgs, uint32_t n, uint32_t width,
                                     uint32_t height, const dlic_opts* opts, uint8_t* d_out, size_t out_capacity,
                                     uint64_t* d_sizes, void* cuda_stream) {
  if (!d_imgs || !d_out || !d_sizes) return fail(DLIC_E_INVALID_ARG, "null pointer");
  dlic_status s = check_model_gpu(m);
  if (s != DLIC_OK) return s;
  Plan p;
  s = make_plan(width, height, n, opts, p, m);
  if (s != DLIC_OK) return s;
  if (out_capacity < p.max_container * p.n_cont)
    return fail(DLIC_E_BUFFER_TOO_SMALL, "out_capacity < containers * max bytes");
  s = check_schedulable(p);
  if (s != DLIC_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  Scratch sc(st);
  return run_encode(m, p, d_imgs, d_out, p.max_container, d_sizes, st, sc, opts ? opts->meta : nullptr);
}

dlic_status dlic_decode_batch_device(const dlic_model* m, const uint8_t* d_bits, const uint64_t* h_offsets,
                                     const uint64_t* h_lengths, uint32_t n, const dlic_header* h_header,
                                     uint8_t* d_imgs, int32_t* d_status, void* cuda_stream) {
  if (!d_bits || !h_offsets || !h_lengths || !h_header || !d_imgs || n == 0)
    return fail(DLIC_E_INVALID_ARG, "null pointer");
  if (!d_status) return fail(DLIC_E_INVALID_ARG, "d_status is required: lane-invariant failures are reported there");
  dlic_status s = check_model_gpu(m);
  if (s != DLIC_OK) return s;
  if (memcmp(h_header->model_sha256, m->sha, 32) != 0)
    return fail(DLIC_E_MODEL_HASH_MISMATCH, "container was coded with another model");
  if (h_header->numerics != NUMERICS_REV)
    return fail(DLIC_E_VERSION_MISMATCH, "container tables come from another arithmetic revision");
  if (h_header->bits != (m->p12 ? 12u : 8u))
    return fail(DLIC_E_SHAPE_MISMATCH, "container alphabet does not match the model's output layer");
  dlic_opts o = opts_of(*h_header);
  Plan p;
  s = make_plan(h_header->width, h_header->height, n * (h_header->depth ? h_header->depth : 1u), &o, p, m);
  if (s != DLIC_OK) return s;
  s = check_schedulable(p);
  if (s != DLIC_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  Scratch sc(st);
  uint64_t* d_meta;  // [0, n) offsets, [n, 2n) lengths
  uint32_t *d_sbase, *d_slen;
  CUDA_TRY(sc.alloc(&d_meta, 16ull * n));
  CUDA_TRY(sc.alloc(&d_sbase, 4ull * n * p.spc));
  CUDA_TRY(sc.alloc(&d_slen, 4ull * n * p.spc));
  CUDA_TRY(cudaMemcpyAsync(d_meta, h_offsets, 8ull * n, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_meta + n, h_lengths, 8ull * n, cudaMemcpyHostToDevice, st));
  // k_dec_prep checks every header and stream size against its container's
  // length before k_decode reads a byte of payload (failures -> d_status[i])
  CUDA_TRY(launch_dec_prep(p, d_bits, d_meta, d_meta + n, d_sbase, d_slen, d_status, st));
  const float* b1img = nullptr;  // every container's metadata block, re-read on the device
  s = meta_bias(m, p, nullptr, d_bits, d_meta, st, sc, &b1img);
  if (s != DLIC_OK) return s;
  ev_begin("decode", st);
  uint32_t* d_sync;
  s = alloc_sync(p, sc, st, &d_sync);
  if (s != DLIC_OK) return s;
  CUDA_TRY(launch_decode(p, m->dw(b1img, p.engine), d_bits, d_meta, d_sbase, d_slen, d_imgs, d_status, st, nullptr, d_sync));
  ev_end("decode", st);
  return DLIC_OK;
}

// ---- volumes (§8(f) f2)
dlic_status dlic_encode_volume(const dlic_model* m, const uint8_t* vol, uint32_t width, uint32_t height,
                               uint32_t depth, const dlic_opts* opts, uint8_t** out, size_t* out_len) {
  if (depth == 0) return fail(DLIC_E_INVALID_ARG, "depth = 0");
  dlic_opts o = opts ? *opts : dlic_opts{DLIC_PREC_BF16, 32, 0, 0, 0, nullptr, 0};
  o.volume_depth = depth;
  uint64_t size = 0;
  return dlic_encode_batch(m, vol, depth, width, height, &o, out, out_len, &size);
}

dlic_status dlic_decode_volume(const dlic_model* m, const uint8_t* bits, size_t len, uint8_t* vol,
                               size_t vol_capacity) {
  if (!m) return fail(DLIC_E_INVALID_ARG, "null model");
  dlic_header h;
  dlic_status s = peek(bits, len, &h, nullptr);
  if (s != DLIC_OK) return s;
  if (h.depth == 0) return fail(DLIC_E_SHAPE_MISMATCH, "not a volume container (window id 1)");
  const uint64_t off = 0;
  return dlic_decode_batch(m, bits, len, &off, 1, vol, vol_capacity);
}

// ---- unit ranges (multi-GPU sharding of one image's independent tiles)
dlic_status dlic_unit_streams(uint32_t width, uint32_t height, const dlic_opts* opts, uint32_t unit_lo,
                              uint32_t unit_hi, uint32_t* first_stream, uint32_t* n_streams) {
  if (!first_stream || !n_streams) return fail(DLIC_E_INVALID_ARG, "null pointer");
  Plan p;
  dlic_status s = make_plan(width, height, 1, opts, p);
  if (s != DLIC_OK) return s;
  s = restrict_units(p, unit_lo, unit_hi);
  if (s != DLIC_OK) return s;
  *first_stream = p.s_lo;
  *n_streams = p.s_cnt;
  return DLIC_OK;
}

dlic_status dlic_encode_units(const dlic_model* m, const uint8_t* img, uint32_t width, uint32_t height,
                              size_t row_stride, const dlic_opts* opts, uint32_t unit_lo, uint32_t unit_hi,
                              uint8_t** payload, size_t* payload_len, uint32_t* stream_sizes) {
  if (!img || !payload || !payload_len || !stream_sizes) return fail(DLIC_E_INVALID_ARG, "null pointer");
  if (row_stride == 0) row_stride = width;
  if (row_stride < width) return fail(DLIC_E_SHAPE_MISMATCH, "row_stride < width");
  dlic_status s = check_model_gpu(m);
  if (s == DLIC_OK && m->p12) return fail(DLIC_E_INVALID_ARG, "unit ranges are for 8-bit images");
  if (s != DLIC_OK) return s;
  Plan p;
  s = make_plan(width, height, 1, opts, p, m);
  if (s != DLIC_OK) return s;
  s = restrict_units(p, unit_lo, unit_hi);
  if (s != DLIC_OK) return s;
  s = check_schedulable(p);
  if (s != DLIC_OK) return s;
  cudaStream_t st = my_stream();
  Scratch sc(st);
  uint8_t *d_img, *d_out;
  uint64_t* d_size;
  uint32_t* d_words = nullptr;
  CUDA_TRY(sc.alloc(&d_img, (size_t)width * height));
  CUDA_TRY(sc.alloc(&d_out, p.max_container));
  CUDA_TRY(sc.alloc(&d_size, 8));
  CUDA_TRY(cudaMemcpy2DAsync(d_img, width, img, row_stride, width, height, cudaMemcpyHostToDevice, st));
  s = run_encode(m, p, d_img, d_out, p.max_container, d_size, st, sc, opts ? opts->meta : nullptr, &d_words);
  if (s != DLIC_OK) return s;
  uint64_t n = 0;
  std::vector<uint32_t> words(p.s_cnt);
  CUDA_TRY(cudaMemcpyAsync(&n, d_size, 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(words.data(), d_words + p.s_lo, 4ull * p.s_cnt, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (n > p.max_container) return fail(DLIC_E_CUDA, "payload size out of range");
  uint8_t* res = static_cast<uint8_t*>(malloc(n ? n : 1));
  if (!res) return fail(DLIC_E_OUT_OF_MEMORY, "malloc");
  CUDA_TRY(cudaMemcpyAsync(res, d_out, n, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (uint32_t i = 0; i < p.s_cnt; ++i) stream_sizes[i] = 2u * words[i];
  *payload = res;
  *payload_len = n;
  return DLIC_OK;
}

dlic_status dlic_container_build(uint32_t width, uint32_t height, const dlic_opts* opts, const uint8_t* model_sha256,
                                 const uint32_t* stream_sizes, uint32_t n_streams, const uint8_t* payload,
                                 size_t payload_len, uint8_t** out, size_t* out_len) {
  if (!stream_sizes || !model_sha256 || !out || !out_len || (!payload && payload_len))
    return fail(DLIC_E_INVALID_ARG, "null pointer");
  Plan p;
  dlic_status s = make_plan(width, height, 1, opts, p);
  if (s != DLIC_OK) return s;
  if (n_streams != p.spc) return fail(DLIC_E_SHAPE_MISMATCH, "stream count does not match (width, height, opts)");
  if (p.n_meta && !opts->meta) return fail(DLIC_E_INVALID_ARG, "opts.n_meta > 0 but opts.meta is null");
  uint64_t tot = 0;
  for (uint32_t i = 0; i < n_streams; ++i) {
    if (stream_sizes[i] & 1u) return fail(DLIC_E_CORRUPT_CONTAINER, "odd stream size");
    tot += stream_sizes[i];
  }
  if (tot != payload_len) return fail(DLIC_E_SHAPE_MISMATCH, "payload length != sum of stream sizes");
  const size_t n = p.hdr_bytes + payload_len;
  uint8_t* o = static_cast<uint8_t*>(malloc(n));
  if (!o) return fail(DLIC_E_OUT_OF_MEMORY, "malloc");
  auto w16 = [&](size_t at, uint32_t v) { o[at] = (uint8_t)v; o[at + 1] = (uint8_t)(v >> 8); };
  auto w32 = [&](size_t at, uint32_t v) { for (int i = 0; i < 4; ++i) o[at + i] = (uint8_t)(v >> (8 * i)); };
  memcpy(o, "DLIC", 4);
  o[4] = (uint8_t)CONTAINER_VERSION;
  o[5] = (uint8_t)p.precision;
  o[6] = 1;
  o[7] = 0;
  w32(8, width);
  w32(12, height);
  w16(16, p.hdr_tw);
  w16(18, p.hdr_th);
  w16(20, p.G);
  w16(22, NUMERICS_REV);
  memcpy(o + 24, model_sha256, 32);
  w32(56, p.spi);
  for (uint32_t i = 0; i < n_streams; ++i) w32(HDR_FIXED + 4 * (size_t)i, stream_sizes[i]);
  const size_t mo = HDR_FIXED + 4 * (size_t)n_streams;  // metadata block
  w32(mo, p.n_meta);
  for (uint32_t k = 0; k < p.n_meta; ++k) {
    uint32_t u;
    memcpy(&u, &opts->meta[k], 4);
    w32(mo + 4 + 4 * k, u);
  }
  if (payload_len) memcpy(o + p.hdr_bytes, payload, payload_len);
  *out = o;
  *out_len = n;
  return DLIC_OK;
}

dlic_status dlic_decode_units(const dlic_model* m, const uint8_t* bits, size_t len, uint32_t unit_lo,
                              uint32_t unit_hi, uint8_t* img, size_t img_capacity) {
  if (!m) return fail(DLIC_E_INVALID_ARG, "null model");
  if (unit_hi <= unit_lo) return fail(DLIC_E_INVALID_ARG, "empty unit range");
  return decode_common(m, bits, len, nullptr, img, img_capacity, unit_lo, unit_hi);
}

uint32_t dlic_numerics_rev(void) { return NUMERICS_REV; }

dlic_status dlic_info(char* buf, size_t cap) {
  int dev = 0, n = 0;
  char name[256] = "none";
  int sms = 0, cc = 0;
  if (cudaGetDeviceCount(&n) == cudaSuccess && n > 0) {
    cudaGetDevice(&dev);
    cudaDeviceProp pr;
    if (cudaGetDeviceProperties(&pr, dev) == cudaSuccess) {
      snprintf(name, sizeof(name), "%s", pr.name);
      sms = pr.multiProcessorCount;
      cc = pr.major * 10 + pr.minor;
    }
  } else {
    cudaGetLastError();
  }
  char tmp[512];
  snprintf(tmp, sizeof(tmp),
           "{\"device\": \"%s\", \"sm_count\": %d, \"cc\": %d, \"arch\": \"sm_100a\", "
           "\"engines\": [\"fp32_ffma\", \"bf16_tcgen05\"], \"enc_smem\": [%zu, %zu], \"dec_smem\": [%zu, %zu]}",
           name, sms, cc, enc_smem_bytes(0), enc_smem_bytes(1), dec_smem_bytes(0, 16), dec_smem_bytes(1, 16));
  if (strlen(tmp) + 1 > cap) return fail(DLIC_E_BUFFER_TOO_SMALL, "info buffer");
  memcpy(buf, tmp, strlen(tmp) + 1);
  return DLIC_OK;
}

void dlic_set_timing(int enable) { g_timing = enable != 0; }

double dlic_last_kernel_ms(const char* name) {
  auto it = g_ev.find(name ? name : "");
  if (it == g_ev.end() || !it->second.used) return -1.0;
  if (cudaEventSynchronize(it->second.b) != cudaSuccess) return -1.0;
  float ms = -1.0f;
  if (cudaEventElapsedTime(&ms, it->second.a, it->second.b) != cudaSuccess) return -1.0;
  return ms;
}

}  // extern "C"
