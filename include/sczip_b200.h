/*
 * sczip_b200.h -- C ABI of libsczip_b200.so, the sm_100a implementation of
 * the sczip feature-compression hot path (quantise -> reshape search ->
 * modified CSR -> frequency table -> rANS, and back).
 *
 * The reference (/root/reference/pkg/src/sczip) is a Python package with no
 * FFI; the boundary it exposes is its Python API.  Each entry point below
 * replaces one reference function and keeps its argument meaning and error
 * class (status codes map 1:1 onto errors.py:4-45):
 *
 *   scz_compress        container.compress         container.py:73-106
 *   scz_decompress      container.decompress       container.py:109-121
 *   scz_encode_batch    compress over a device batch (SPEC.md:394 batch mode)
 *   scz_encode_batch_ptrs  compress over a heterogeneous device batch
 *   scz_decode_batch    decompress over a device batch
 *   scz_quantize        tensor.params_for+quantize tensor.py:125-140
 *   scz_quantize_params tensor.quantize            tensor.py:130-140
 *   scz_dequantize      tensor.dequantize          tensor.py:143-156
 *   scz_csr_encode      sparse.csr_encode+concat   sparse.py:63-69,98-101
 *   scz_csr_decode      sparse.split+csr_decode    sparse.py:72-95,104-111
 *   scz_build_counts    rans.build_counts          rans.py:76-85
 *   scz_normalize       rans.normalize_frequencies rans.py:88-131
 *   scz_rans_encode     rans.encode (v1) / FORMAT.md v2 lanes  rans.py:155-180
 *   scz_rans_decode     rans.decode (v1) / v2      rans.py:183-213
 *   scz_search          optimizer.search / exhaustive_search   optimizer.py:109-166
 *
 * Conventions: plain pointers and sizes, no torch types.  Functions without
 * a `_batch` suffix take HOST buffers and are synchronous; `_batch`
 * functions take DEVICE pointers and are stream-ordered on the context's
 * stream (scz_ctx_stream).  A context is used by one host thread at a time;
 * separate contexts may run concurrently.  Every call returns an SCZ_*
 * status; scz_last_error() gives the message of the last failure.
 */
#ifndef SCZIP_B200_H
#define SCZIP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum scz_status {
    SCZ_OK = 0,
    SCZ_INVALID_INPUT = 1,        /* errors.InvalidInput */
    SCZ_NON_DIVISIBLE = 2,        /* errors.NonDivisible */
    SCZ_CORRUPT_STREAM = 3,       /* errors.CorruptStream */
    SCZ_INVALID_CONTAINER = 4,    /* errors.InvalidContainer */
    SCZ_UNSUPPORTED_VERSION = 5,  /* errors.UnsupportedVersion */
    SCZ_ALPHABET_OVERFLOW = 6,    /* errors.AlphabetOverflow */
    SCZ_NORMALIZE_ERROR = 7,      /* errors.NormalizeError */
    SCZ_PRECISION_TOO_SMALL = 8,  /* errors.PrecisionTooSmall */
    SCZ_UNCODABLE_SYMBOL = 9,     /* errors.UncodableSymbol */
    SCZ_CUDA_ERROR = 100,         /* launch / runtime failure */
    SCZ_NO_DEVICE = 101,          /* no sm_100 device visible */
    SCZ_OUT_OF_MEMORY = 102,
    SCZ_UNSUPPORTED = 103         /* outside this build's limits (e.g. T >= 2^31) */
};

/* One compressed tensor: the header fields of container.py:32-46 plus the
 * FORMAT.md v2 block layout and the locations of its variable-length parts
 * inside a batch's buffers. */
typedef struct scz_info {
    int32_t status;        /* SCZ_* for this tensor */
    uint8_t version;       /* 1 = reference wire format, 2 = interleaved lanes */
    uint8_t q_bits;        /* Q in [2, 8] */
    uint8_t precision;     /* rANS table precision n */
    uint8_t sym_bytes;     /* width of col/row symbols on device (1, 2 or 4) */
    uint64_t total;        /* T = prod(dims) */
    uint32_t n_rows;       /* N */
    uint32_t n_cols;       /* K = T / N */
    uint64_t nnz;          /* original-nonzero count */
    double scale;          /* QuantParams.scale (float64) */
    int64_t zero_point;    /* QuantParams.zero_point */
    uint32_t alphabet;     /* A = max(D) + 1 */
    uint32_t lanes;        /* v2: interleaved lanes per block (W) */
    uint32_t block_syms;   /* v2: symbols per block (multiple of W) */
    uint32_t n_blocks;     /* v2: blocks; 1 for v1 */
    uint64_t payload_len;  /* rANS payload bytes */
    uint64_t payload_off;  /* byte offset of the payload in the batch payload buffer */
    uint64_t freqs_off;    /* element offset of the u32 freq table in the batch table */
    uint64_t blocks_off;   /* element offset of the u32 block lengths (v2) */
    uint32_t search_flags; /* SCZ_SEARCH_* */
    uint32_t n_evaluated;  /* candidates the early-stopped scan evaluated */
} scz_info;

enum {
    SCZ_SEARCH_NEAR_TIE = 1u,      /* a decision compared costs within 1e-12: host re-decides */
    SCZ_SEARCH_EARLY_STOPPED = 2u, /* SearchReport.early_stopped */
    SCZ_SEARCH_USED = 4u           /* N came from Algorithm 1 (n_rows was None) */
};

/* Device-resident outputs of scz_encode_batch, owned by the context until
 * its next encode call.  Tensor i's payload is d_payload[info.payload_off
 * .. + payload_len), its table d_freqs[info.freqs_off .. + alphabet) and its
 * v2 block lengths d_block_bytes[info.blocks_off .. + n_blocks).  v1 payloads
 * are packed back to back; v2 payloads sit at a fixed per-tensor stride (the
 * encoder packs each tensor's blocks in place), so payload_total spans the
 * strided region and the host path copies them with one pitched copy. */
typedef struct scz_batch {
    uint32_t batch;
    scz_info* d_info;
    uint32_t* d_freqs;
    uint32_t* d_block_bytes;
    uint8_t* d_payload;
    uint64_t payload_total;   /* valid after scz_batch_sync */
    uint64_t freqs_total;
    uint64_t blocks_total;
} scz_batch;

typedef struct scz_ctx scz_ctx;

int scz_ctx_create(int device, scz_ctx** out);
void scz_ctx_destroy(scz_ctx* ctx);
const char* scz_last_error(const scz_ctx* ctx);
void* scz_ctx_stream(scz_ctx* ctx); /* cudaStream_t the batch calls are ordered on */
int scz_abi_version(void);
/* Number of kernel launches this context issued since creation. */
uint64_t scz_launch_count(const scz_ctx* ctx);

/* ---- container.py: whole pipeline, host buffers ------------------------ */
/* compress: n_rows < 0 selects N with Algorithm 1 (optimizer.search);
 * format 1 = reference wire format (single rANS stream), 2 = FORMAT.md v2.
 * On success *info is filled and freqs/block_bytes/payload point at
 * context-owned host memory valid until the next call on ctx. */
int scz_compress(scz_ctx* ctx, const float* x, uint64_t total, int q_bits,
                 int64_t n_rows, int precision, int format, uint32_t lanes,
                 uint32_t block_syms, scz_info* info, const uint32_t** freqs,
                 const uint32_t** block_bytes, const uint8_t** payload);
/* decompress: info fields as parsed from the header (version, q_bits,
 * precision, total, n_rows, n_cols, nnz, scale, zero_point, alphabet,
 * lanes, block_syms, n_blocks, payload_len); out receives T float32. */
int scz_decompress(scz_ctx* ctx, const scz_info* info, const uint32_t* freqs,
                   const uint32_t* block_bytes, const uint8_t* payload, float* out);

/* ---- device batch (stream-ordered) ------------------------------------- */
/* Encode `batch` tensors of `total` float32 each, contiguous at d_x. */
int scz_encode_batch(scz_ctx* ctx, const float* d_x, uint64_t total, uint32_t batch,
                     int q_bits, int64_t n_rows, int precision, int format,
                     uint32_t lanes, uint32_t block_syms, scz_batch* out);
/* Heterogeneous batch: tensor i is numel[i] float32 at the
 * DEVICE address d_x[i] (d_x and numel are host arrays).  Tensors of equal
 * size are encoded together (gathered into one [B][T] array first unless they
 * already are one) and every group's output is appended to one
 * context-owned result: out describes all `batch` tensors in the caller's
 * order, and scz_batch_sync / scz_decode_batch(_async) consume it like any
 * batch (tensor i decodes to d_out + numel[0] + ... + numel[i-1]).  Returns
 * after the device work (the staging tables are reused by the next call). */
int scz_encode_batch_ptrs(scz_ctx* ctx, const float* const* d_x, const uint64_t* numel, uint32_t batch,
                          int q_bits, int64_t n_rows, int precision, int format, uint32_t lanes,
                          uint32_t block_syms, scz_batch* out);
/* Wait for the batch, copy its infos to h_info[batch] and set payload_total. */
int scz_batch_sync(scz_ctx* ctx, scz_batch* b, scz_info* h_info);
/* Decode `batch` tensors described by h_info (host copy; its offsets index
 * the device buffers) into d_out (tensor i at d_out + sum of earlier totals).
 * Per-tensor status goes to h_status after completion (synchronous). */
int scz_decode_batch(scz_ctx* ctx, const scz_info* h_info, uint32_t batch,
                     const uint32_t* d_freqs, const uint32_t* d_block_bytes,
                     const uint8_t* d_payload, float* d_out, int32_t* h_status);
/* Asynchronous form of scz_decode_batch: statuses stay on device until
 * scz_decode_status (used by the bench to keep the timed region device-only). */
int scz_decode_batch_async(scz_ctx* ctx, const scz_info* h_info, uint32_t batch,
                           const uint32_t* d_freqs, const uint32_t* d_block_bytes,
                           const uint8_t* d_payload, float* d_out);
int scz_decode_status(scz_ctx* ctx, uint32_t batch, int32_t* h_status);
/* Decode, without any host round trip, the batch that the last
 * scz_encode_batch of this context produced (its headers stay on the device;
 * launch geometry is bounded by that call's plan) into d_out (tensor i at
 * d_out + i * total).  Same checks as the host-header path, done on the
 * device; statuses via scz_decode_status.  The bench's device-resident
 * round trip: encode + decode queue back to back with no synchronisation. */
int scz_decode_batch_device(scz_ctx* ctx, float* d_out);

/* ---- batch over HOST buffers (the e2e path) ---------------------------- */
/* compress `batch` tensors of `total` float32 (contiguous at h_x; pinned
 * memory gives full PCIe rate).  Outputs point at context-owned pinned host
 * memory valid until the next call: infos[batch] (offsets index the three
 * buffers), the packed payload, freqs and v2 block lengths; sizes[3] gets
 * their element counts (payload bytes, freqs, blocks). */
int scz_compress_batch(scz_ctx* ctx, const float* h_x, uint64_t total, uint32_t batch,
                       int q_bits, int64_t n_rows, int precision, int format, uint32_t lanes,
                       uint32_t block_syms, const scz_info** infos, const uint8_t** payload,
                       const uint32_t** freqs, const uint32_t** block_bytes, uint64_t* sizes);
/* decompress `batch` containers laid out as scz_compress_batch returns them
 * into h_out (tensor i after the totals of tensors < i); h_status[batch]. */
int scz_decompress_batch(scz_ctx* ctx, const scz_info* h_info, uint32_t batch,
                         const uint32_t* h_freqs, uint64_t freqs_count,
                         const uint32_t* h_blocks, uint64_t blocks_count,
                         const uint8_t* h_payload, uint64_t payload_bytes, float* h_out,
                         int32_t* h_status);

/* ---- instrumentation ---------------------------------------------------- */
/* Device time (CUDA events) of the last host-buffer call on ctx
 * (scz_compress, scz_decompress, scz_compress_batch, scz_decompress_batch):
 * from its first host->device copy to its last device->host copy.  Replaces
 * the wall clock of bench._time_ms (bench.py:88-98) for enc_ms / dec_ms. */
int scz_last_call_ms(scz_ctx* ctx, float* ms);
/* Per-kernel CUDA-event timing on the context stream (off by default). */
int scz_ctx_set_timing(scz_ctx* ctx, int enable);
/* "name total_ms launches\n" lines accumulated since the last read. */
int scz_ctx_read_timing(scz_ctx* ctx, char* buf, uint64_t cap);

/* ---- stage entry points used by the parity suite (host buffers) -------- */
/* tensor.params_for + tensor.quantize: symbols (u32) and zero mask (u8). */
int scz_quantize(scz_ctx* ctx, const float* x, uint64_t n, int q_bits, float* minmax,
                 double* scale, int64_t* zero_point, uint32_t* q, uint8_t* mask);
/* tensor.dequantize (masked positions -> +0.0). */
int scz_dequantize(scz_ctx* ctx, const uint32_t* q, const uint8_t* mask, uint64_t n,
                   int q_bits, double scale, int64_t zero_point, float* out);
/* sparse.csr_encode + concat: D = v ++ c ++ r (u32, capacity 2n + n_rows). */
int scz_csr_encode(scz_ctx* ctx, const uint32_t* q, const uint8_t* mask, uint64_t n_rows,
                   uint64_t n_cols, uint32_t* d, uint64_t* nnz);
/* sparse.split + csr_decode. */
int scz_csr_decode(scz_ctx* ctx, const uint32_t* d, uint64_t nnz, uint64_t n_rows,
                   uint64_t n_cols, uint32_t* q, uint8_t* mask);
int scz_build_counts(scz_ctx* ctx, const uint32_t* d, uint64_t n, uint64_t alphabet,
                     int64_t* counts);
int scz_normalize(scz_ctx* ctx, const int64_t* counts, uint64_t alphabet, int precision,
                  uint32_t* freqs);
/* lanes == 0: v1 single stream; else FORMAT.md v2 (block_bytes[n_blocks]).
 * out capacity: 4*max(lanes,1)*n_blocks + 2*n bytes. */
int scz_rans_encode(scz_ctx* ctx, const uint32_t* d, uint64_t n, const uint32_t* freqs,
                    uint64_t alphabet, int precision, uint32_t lanes, uint32_t block_syms,
                    uint8_t* out, uint64_t* out_len, uint32_t* block_bytes);
int scz_rans_decode(scz_ctx* ctx, const uint8_t* data, uint64_t len, const uint32_t* freqs,
                    uint64_t alphabet, int precision, uint32_t lanes, uint32_t block_syms,
                    uint64_t n_blocks, const uint32_t* block_bytes, uint64_t count,
                    uint32_t* out);
/* tensor.quantize with caller-given parameters (QuantParams scale, zero_point). */
int scz_quantize_params(scz_ctx* ctx, const float* x, uint64_t n, int q_bits, double scale,
                        int64_t zero_point, uint32_t* q, uint8_t* mask);
/* Algorithm 1 over a float tensor (optimizer.search / exhaustive_search /
 * cost): every candidate is priced in one device pass.  rows == NULL prices
 * the feasible candidates of optimizer.candidate_rows; otherwise the
 * n_rows_list given row counts (optimizer.cost).  Writes n_cand rows of
 * cand[6] = {N, K, nnz, stream_len, entropy (double bits), cost (double
 * bits)} and, if counts is non-null, each candidate's histogram of D
 * (counts_stride u32 entries per row, zero-padded).  *chosen is the index of
 * the early-stopped choice, *chosen_exhaustive the exhaustive optimum; flags
 * as scz_info.search_flags. */
int scz_search(scz_ctx* ctx, const float* x, uint64_t n, int q_bits, const uint64_t* rows,
               uint32_t n_rows_list, uint32_t max_cand, uint32_t* n_cand, uint64_t* cand,
               uint32_t* counts, uint32_t counts_stride, uint32_t* chosen,
               uint32_t* chosen_exhaustive, uint32_t* flags);

#ifdef __cplusplus
}
#endif
#endif /* SCZIP_B200_H */
