/*
 * dlic.h — C-ABI of the B200-native DLIC hot path (libdlic.so).
 *
 * DLIC (arXiv 2207.05152, /root/reference/PAPER.md cited as P:<line>) codes an
 * 8-bit grayscale image losslessly: a dense network maps each pixel's causal
 * window of already-coded neighbours (Fig. 6; dummy value outside
 * the image P:59) to a 256-way PDF, which drives rANS coder instances,
 * at most one per pixel row.  Encoding evaluates every pixel at
 * once; decoding walks the wavefront step(r,c) = c + 3r (WPP).
 *
 * The paper states the problem as encode(image, weights) -> bitstream and
 * decode(bitstream, weights) -> image (Fig. 2); dlic_encode /
 * dlic_decode follow it.  Readings of everything the paper leaves open
 * (window shape, fill, quantiser, rANS constants, lane framing) are DESIGN.md
 * R1-R10.
 *
 * Conventions
 *  - Every call returns dlic_status; no exception crosses the ABI.  On error
 *    outputs are untouched (except where noted) and dlic_last_error() holds a
 *    thread-local detail string.  CUDA failures map to DLIC_E_CUDA.
 *  - Host pointers are plain CPU memory; pointers named d_* are CUDA device
 *    memory owned by the caller; cuda_stream is a cudaStream_t (NULL = the
 *    legacy default stream).  The library never takes ownership of caller
 *    memory; buffers it returns are released with dlic_free.
 *  - Images are row-major uint8, row_stride >= width bytes.
 *  - A dlic_model is immutable after load and may be shared by threads.
 *  - No CPU fallback exists: every pixel-level step runs in CUDA kernels on
 *    an sm_100a device; without one, calls return DLIC_E_CUDA.
 */
#ifndef DLIC_H
#define DLIC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DLIC_OK = 0,
  DLIC_E_INVALID_ARG = 1,      /* null pointer, zero size, unsupported option */
  DLIC_E_SHAPE_MISMATCH = 2,   /* image / tables / model dims disagree */
  DLIC_E_NONCAUSAL_WINDOW = 3, /* reserved: window id other than the causal 9x9 */
  DLIC_E_CORRUPT_MODEL = 4,    /* model blob magic/length/hash invalid */
  DLIC_E_VERSION_MISMATCH = 5, /* container version or window id unknown */
  DLIC_E_CORRUPT_CONTAINER = 6,/* bad framing, or a lane ended off its invariant */
  DLIC_E_MODEL_HASH_MISMATCH = 7, /* container coded with another model (checked first) */
  DLIC_E_STREAM_UNDERFLOW = 8, /* a lane needed a word past its stream end */
  DLIC_E_SUM_MISMATCH = 9,     /* a frequency table does not sum to 2^16 */
  DLIC_E_ZERO_FREQUENCY = 10,  /* a frequency of 0 in a table */
  DLIC_E_BUFFER_TOO_SMALL = 11,
  DLIC_E_CUDA = 12,            /* CUDA runtime / launch failure, or no sm_100 device */
  DLIC_E_OUT_OF_MEMORY = 13,
  DLIC_E_UNSUPPORTED_MODEL = 14 /* topology outside the GPU engines' (see dlic_model_load) */
} dlic_status;

/* Precision path of the density estimator (recorded in the container; both
 * sides of a bitstream must use the same path).
 *  DLIC_PREC_FP32: fp32 FFMA on CUDA cores, fixed summation order (meets the
 *                  1e-4 relative logit bar vs the fp64 oracle).
 *  DLIC_PREC_BF16: bf16 operands on tcgen05 tensor cores, fp32 accumulation in
 *                  TMEM (bpp gated to within 0.5% of fp32). */
enum { DLIC_PREC_FP32 = 0, DLIC_PREC_BF16 = 1 };

typedef struct dlic_model dlic_model; /* opaque; immutable after load */

#define DLIC_MAX_META 8

typedef struct {
  uint32_t precision;  /* DLIC_PREC_* */
  uint32_t group_rows; /* G: rows per interleaved stream (R7); 0 -> 32 */
  uint32_t tile_w;     /* independent tiles (Q16); 0,0 = untiled */
  uint32_t tile_h;
  /* metadata inputs: n_meta raw reals per image, HOST array
   * meta[i * n_meta + k] for image i of a call (single-image calls: i = 0).
   * n_meta must equal the model's metadata feature count (0 = none). */
  uint32_t n_meta;
  const float* meta;
  /* volumes (3D window R13 + overlapped 3D wavefront R14):
   * 0 = 2D images (container window id 1, the 78-tap window); D >= 1 = each
   * group of D consecutive images of a call is one volume (slices in order)
   * coded into ONE container (window id 2, streams slice-major); requires a
   * model with 87 (+ n_meta) inputs.  Metadata (n_meta reals) is then per
   * volume: meta[v * n_meta + k]. */
  uint32_t volume_depth;
} dlic_opts;

/* Container (version 2, little-endian):
 *   "DLIC", u8 version 2, u8 precision, u8 window id 1 (R1), u8 alphabet (0 =
 *   8-bit pixels, 12 = 12-bit pixels: P:184-186, R15),
 *   u32 width, u32 height, u16 tile_w, u16 tile_h (0,0 = untiled; Q16),
 *   u16 G (rows per stream, R7), u16 numerics (arithmetic revision of the
 *   tables, see dlic_numerics_rev), 32-byte SHA-256 of the model file,
 *   u32 n_streams, u32 sizes[n_streams] (bytes), u32 n_meta, f32
 *   meta[n_meta] (the image's raw metadata reals, uncompressed), then
 *   the streams tile-major, group-major within a tile.  Each stream: the
 *   group's flushed rANS states (rows ascending, hi word then lo word)
 *   followed by its renormalisation words in decoder order (front ascending,
 *   row ascending), 16-bit LE words. */
typedef struct {
  uint32_t width, height, precision, group_rows, tile_w, tile_h, n_streams, n_units;
  uint32_t numerics; /* arithmetic revision recorded by the encoder */
  uint32_t depth;    /* slices: 0 for a 2D image (window id 1), D for a volume (window id 2) */
  uint32_t n_meta;   /* metadata reals stored in the container */
  float meta[DLIC_MAX_META];
  uint8_t model_sha256[32];
  uint64_t payload_bytes, header_bytes;
  uint32_t bits;     /* alphabet: 8, or 12 (byte 7 = 12; pixels are u16, R15) */
} dlic_header;

/* ---- models --------------------------------------------------------------
 * "DLICMDL1" blob: magic, u16 layers, per layer {u32 in, u32 out,
 * u8 act, u8 pool group g (0 = none), f32 W[in][out] row-major, f32 b[out]},
 * u16 metadata feature count n, n x f32 (min, max), SHA-256 of all preceding
 * bytes.  Uploads fp32 and bf16 device copies to `cuda_device`.
 * The GPU engines run six dense layers with 128-unit hidden layers and 256
 * outputs ("P100K"), on 78 window inputs (or 87 for volumes: + the 3x3
 * box of the slice below, R13) + n <= 8 metadata inputs
 * (min-max normalised with the stored constants), with optional average
 * pooling of g = 2^k units after any hidden layer ("two optional
 * pooling layers"; the next layer then has 128 / g inputs).  Pooling is linear
 * and is folded into the next layer's weights at load (W' = P^T W: exact in
 * bf16 and fp32 because 1/g is a power of two); the metadata inputs are
 * folded into a per-image layer-1 bias by a kernel at each call.
 * Two larger networks run on a streamed-weight bf16 engine (weights exceed
 * one SM's shared memory; layers 2-6 arrive from L2 in 32 KB TMA bulk chunks):
 *   P350K = 78 -> 256 x5 -> 256 (Table I ~350K; §8(f) f1);
 *   P12   = 78 -> 256 x5 -> 4096 ("4096 output layer neurons";
 *           Table III ~1.35M): the 12-bit alphabet.  With a P12
 *           model every image buffer of the calls below holds u16 pixels
 *           (values < 4096; byte sizes and capacities double, row_stride
 *           stays in pixels) and containers carry alphabet byte 12.
 * Both are bf16 only, without metadata, volumes or unit ranges.  Other
 * topologies load (hash, dlic_peek) but encode/decode return
 * DLIC_E_UNSUPPORTED_MODEL.  Errors: DLIC_E_CORRUPT_MODEL, DLIC_E_CUDA. */
dlic_status dlic_model_load(const void* bytes, size_t len, int cuda_device, dlic_model** out);
/* Same from arrays: dims[n_layers+1]; W[l] row-major [dims[l]][dims[l+1]]
 * float32; b[l] float32[dims[l+1]].  The blob (and its hash) is built here. */
dlic_status dlic_model_from_arrays(uint32_t n_layers, const uint32_t* dims, const float* const* W,
                                   const float* const* b, int cuda_device, dlic_model** out);
void dlic_model_free(dlic_model* m);
/* SHA-256 content hash recorded in containers (host only). */
dlic_status dlic_model_sha256(const dlic_model* m, uint8_t out[32]);
/* Host-only check of a model blob (magic, length, SHA-256); no device work. */
dlic_status dlic_model_blob_check(const void* bytes, size_t len, uint8_t sha_out[32]);

/* ---- the paper's statement: encode(image, weights) -> bitstream ----------
 * Host image in, library-allocated container out (release with dlic_free).
 * Exactly one host->device copy (the image) and one device->host copy of the
 * result, on an internal stream.  opts NULL = {DLIC_PREC_BF16, G = 32,
 * untiled}. */
dlic_status dlic_encode(const dlic_model* m, const uint8_t* img, uint32_t width, uint32_t height,
                        size_t row_stride, const dlic_opts* opts, uint8_t** out, size_t* out_len);

/* decode(bitstream, weights) -> image.  Verifies the model hash and the
 * arithmetic revision BEFORE any pixel work, checks every lane's end state
 * (2^16) and cursor, and writes width*height bytes (row-major, stride =
 * width) to img.
 * Errors: DLIC_E_MODEL_HASH_MISMATCH, DLIC_E_VERSION_MISMATCH (container of
 * another version or numerics revision), DLIC_E_CORRUPT_CONTAINER,
 * DLIC_E_STREAM_UNDERFLOW, DLIC_E_BUFFER_TOO_SMALL. */
dlic_status dlic_decode(const dlic_model* m, const uint8_t* bits, size_t len, uint8_t* img,
                        size_t img_capacity);

/* Parse a container header (host only, no device work; any numerics value). */
dlic_status dlic_peek(const uint8_t* bits, size_t len, dlic_header* out);

/* Arithmetic revision of this build's density estimator + softmax/quantiser
 * (the integer tables depend on the exact instruction sequence, "as long
 * as the precision of the floating point arithmetic is the same").  Written
 * into every container; decode rejects any other value with
 * DLIC_E_VERSION_MISMATCH.  0 is reserved for the CPU oracle's arithmetic. */
uint32_t dlic_numerics_rev(void);

/* Upper bound of the container size for (width, height, opts): one image, or
 * one volume of opts->volume_depth slices. */
size_t dlic_max_container_bytes(uint32_t width, uint32_t height, const dlic_opts* opts);

void dlic_free(void* p);
const char* dlic_status_str(dlic_status s);
const char* dlic_last_error(void);

/* ---- host batch: the same calls over n independent images ----------------
 * (units are whole images, R7/Q16; each container is byte-identical to what
 * dlic_encode produces for that image alone).  One host->device copy of all
 * images and one device->host copy of all containers per call.
 * encode: imgs = n*height*width bytes (image i at imgs + i*width*height,
 * row-major); *out = library-allocated buffer (dlic_free) holding the
 * containers back to back (n, or n / opts->volume_depth for volumes), *out_len
 * its total size, sizes[i] (caller array, one per container) the size of
 * container i.
 * decode: container i at bits + offsets[i] (offsets ascending, all containers
 * of the same width/height/options and model); writes n*width*height bytes to
 * imgs.  Each header is checked on the host (hash before any pixel work), each
 * container's lane invariants on the device; the first failing image's status
 * is returned. */
dlic_status dlic_encode_batch(const dlic_model* m, const uint8_t* imgs, uint32_t n, uint32_t width,
                              uint32_t height, const dlic_opts* opts, uint8_t** out, size_t* out_len,
                              uint64_t* sizes);
dlic_status dlic_decode_batch(const dlic_model* m, const uint8_t* bits, size_t len, const uint64_t* offsets,
                              uint32_t n, uint8_t* imgs, size_t img_capacity);

/* ---- device-resident batch variants (caller owns memory and stream) -------
 * n images of width x height, packed (image i at d_imgs + i*width*height).
 * Encode writes container i at d_out + i*dlic_max_container_bytes(...) and its
 * byte size to d_sizes[i] (uint64).  out_capacity must be >= n * max bytes.
 * Asynchronous on cuda_stream except for small internal scratch allocations
 * (stream-ordered).  Errors are reported for the launch; framing and
 * lane-invariant failures of decode are reported through d_status[i] (0 = ok,
 * else a dlic_status), which is required. */
dlic_status dlic_encode_batch_device(const dlic_model* m, const uint8_t* d_imgs, uint32_t n,
                                     uint32_t width, uint32_t height, const dlic_opts* opts,
                                     uint8_t* d_out, size_t out_capacity, uint64_t* d_sizes,
                                     void* cuda_stream);
/* Decode n containers that all share (width, height, opts) — i.e. produced by
 * dlic_encode_batch_device — container i at d_bits + h_offsets[i], exactly
 * h_lengths[i] bytes long (HOST arrays).  The headers are re-read on the
 * device and every stream size is checked against h_lengths[i] before any
 * payload byte is read (a truncated or corrupt size table cannot make the
 * decoder read outside its container); h_header is the parsed header of
 * container 0 (dlic_peek on a host copy), used for planning.  d_status (n
 * int32, device) is required: framing errors and lane-invariant failures of
 * image i land in d_status[i] (callers zero it first).
 * Errors (returned): DLIC_E_INVALID_ARG (incl. d_status NULL),
 * DLIC_E_MODEL_HASH_MISMATCH, DLIC_E_VERSION_MISMATCH, DLIC_E_CUDA. */
dlic_status dlic_decode_batch_device(const dlic_model* m, const uint8_t* d_bits,
                                     const uint64_t* h_offsets, const uint64_t* h_lengths,
                                     uint32_t n, const dlic_header* h_header, uint8_t* d_imgs,
                                     int32_t* d_status, void* cuda_stream);

/* ---- volumes (§8(f) f2): the paper's MRI coder ----------------
 * vol = depth slices of width x height (slice z at vol + z*height*row_stride...
 * contiguous, row_stride = width).  One container per volume (window id 2).
 * Decode runs every slice's wavefront at once, each slice delayed behind the
 * one below by the 3D window's reach (the 3D wavefront). */
dlic_status dlic_encode_volume(const dlic_model* m, const uint8_t* vol, uint32_t width, uint32_t height,
                               uint32_t depth, const dlic_opts* opts, uint8_t** out, size_t* out_len);
dlic_status dlic_decode_volume(const dlic_model* m, const uint8_t* bits, size_t len, uint8_t* vol,
                               size_t vol_capacity);

/* ---- unit ranges: one image's independent tiles split across GPUs ---------
 * (north_star: "independent image tiles with their own streams are
 * partitioned across the GPUs"; units = tiles of Q16 in row-major order,
 * untiled = one unit).  A rank codes units [unit_lo, unit_hi) of the image;
 * the only exchange is the per-stream sizes (NCCL all_gather), from which any
 * rank frames the container with dlic_container_build.
 *
 * dlic_unit_streams: the streams [first, first + n) of those units (host only).
 * dlic_encode_units: host image in (the whole image; only the range's units are
 *   coded); *payload = library-allocated concatenation of the range's streams
 *   in container order (dlic_free), stream_sizes (caller array of n_streams of
 *   dlic_unit_streams) their byte sizes.  Bytes are identical to the
 *   corresponding streams of dlic_encode's container.
 * dlic_container_build: host-only framing of a complete container from all
 *   n_streams sizes and the concatenated payload (*out: dlic_free).
 * dlic_decode_units: decodes only units [unit_lo, unit_hi) of a container
 *   into img (width*height bytes); the other pixels of img are left untouched. */
dlic_status dlic_unit_streams(uint32_t width, uint32_t height, const dlic_opts* opts, uint32_t unit_lo,
                              uint32_t unit_hi, uint32_t* first_stream, uint32_t* n_streams);
dlic_status dlic_encode_units(const dlic_model* m, const uint8_t* img, uint32_t width, uint32_t height,
                              size_t row_stride, const dlic_opts* opts, uint32_t unit_lo, uint32_t unit_hi,
                              uint8_t** payload, size_t* payload_len, uint32_t* stream_sizes);
dlic_status dlic_container_build(uint32_t width, uint32_t height, const dlic_opts* opts,
                                 const uint8_t* model_sha256, const uint32_t* stream_sizes, uint32_t n_streams,
                                 const uint8_t* payload, size_t payload_len, uint8_t** out, size_t* out_len);
dlic_status dlic_decode_units(const dlic_model* m, const uint8_t* bits, size_t len, uint32_t unit_lo,
                              uint32_t unit_hi, uint8_t* img, size_t img_capacity);

/* ---- parity / debug taps ---------------------------------------------------
 * rANS only, fed integer tables (north_star: "the same quantised frequency
 * tables and bitstream bit-exactly as the oracle when the oracle is fed the
 * same integer tables").  fc[r*width+c] = f_s | (c_s << 16) of the TRUE symbol
 * of pixel (r,c) (host array).  Produces the container exactly as dlic_encode
 * would (precision field = opts->precision, model hash = model_sha256 or zeros). */
dlic_status dlic_rans_encode_tables(const uint32_t* fc, uint32_t width, uint32_t height,
                                    const dlic_opts* opts, const uint8_t* model_sha256,
                                    uint8_t** out, size_t* out_len);
/* Decode a container given every pixel's full frequency table
 * freq_tables[(r*width+c)*256 + s] (host, uint16, each table sums to 2^16).
 * Writes the image to img (width*height bytes). */
dlic_status dlic_rans_decode_tables(const uint8_t* bits, size_t len, const uint16_t* freq_tables,
                                    uint8_t* img);
/* Run the encoder's density-estimator kernel on every pixel of a host image
 * (tile-aware per opts) and export, per pixel in raster order, any of
 * (bf16: the production kernel k_enc_pp itself, with its debug exports
 * compiled in; fp32: k_enc_mlp<fp32>):
 * logits[256] (fp32), probs[256] (fp32 softmax as used by the quantiser),
 * freqs[256] (uint16 integer table), fc (f_s | c_s<<16 of the true symbol).
 * NULL outputs are skipped. */
dlic_status dlic_debug_mlp(const dlic_model* m, const uint8_t* img, uint32_t width, uint32_t height,
                           const dlic_opts* opts, float* logits, float* probs, uint16_t* freqs,
                           uint32_t* fc);

/* Library / device info: writes a short JSON string (device name, SM count,
 * kernel variants) into buf.  Returns DLIC_E_BUFFER_TOO_SMALL if cap is short. */
dlic_status dlic_info(char* buf, size_t cap);

/* Per-kernel timing of the last call on this thread (milliseconds, CUDA
 * events on the launching stream): names "mlp", "rans_enc", "compact",
 * "decode".  Returns -1 when not measured.  Enabled by dlic_set_timing(1). */
void dlic_set_timing(int enable);
double dlic_last_kernel_ms(const char* name);

#ifdef __cplusplus
}
#endif
#endif /* DLIC_H */
