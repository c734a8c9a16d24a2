// decode.cu -- CSR decode + dequantisation (K8) and the small
// stage kernels used by the parity entry points.
//
//   k_row_sums   per 4096-row chunk: sum of row counts, r <= K check
//   k_row_scan   per tensor: chunk offsets, sum(r) == nnz check
//   k_rows_out   per chunk: row offsets (block scan), col checks
//                (col < K, strictly increasing: sparse.py:74-89), and the
//                dense row written once: LUT[v] at listed columns, +0.0
//                elsewhere (tensor.py:154-155), or (q, mask) for the stage API.
#include "common.cuh"

namespace scz {

constexpr int ROW_CHUNK = 4096;
constexpr int ROW_THREADS = 256;

struct RowParams {
    const scz_info* info;   // [B]
    const void* dsym;       // [B][dsym_stride] decoded D
    uint64_t dsym_stride;
    uint32_t* chunk_sum;    // [B][nchunk_cap]
    uint32_t nchunk_cap;
    int32_t* status;        // [B]
    float* out;             // [B] tensors at out_off[b]
    const uint64_t* out_off;
    uint32_t* q_out;        // stage API: symbols
    uint8_t* mask_out;      // stage API: zero mask
};

template <typename S>
__global__ void __launch_bounds__(ROW_THREADS) k_row_sums(RowParams p) {
    const uint32_t b = blockIdx.y, chunk = blockIdx.x;
    const scz_info& in = p.info[b];
    if (p.status[b] != SCZ_OK || in.sym_bytes != sizeof(S)) return;
    const uint64_t N = in.n_rows, r0 = (uint64_t)chunk * ROW_CHUNK;
    if (r0 >= N) return;
    const S* r = reinterpret_cast<const S*>(p.dsym) + (uint64_t)b * p.dsym_stride + 2 * in.nnz;
    uint32_t sum = 0, bad = 0;
    const uint64_t r1 = min(N, r0 + ROW_CHUNK);
    for (uint64_t i = r0 + threadIdx.x; i < r1; i += ROW_THREADS) {
        uint32_t v = r[i];
        bad |= v > in.n_cols;
        sum += v;
    }
    sum = warp_sum(sum);
    bad = __reduce_or_sync(0xffffffffu, bad);
    __shared__ uint32_t s_sum[ROW_THREADS / 32], s_bad[ROW_THREADS / 32];
    if ((threadIdx.x & 31) == 0) {
        s_sum[threadIdx.x >> 5] = sum;
        s_bad[threadIdx.x >> 5] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < ROW_THREADS / 32; ++w) {
            sum += s_sum[w];
            bad |= s_bad[w];
        }
        p.chunk_sum[(uint64_t)b * p.nchunk_cap + chunk] = sum;
        if (bad) p.status[b] = SCZ_CORRUPT_STREAM;  // sparse.py:88-89
    }
}

__global__ void __launch_bounds__(256) k_row_scan(RowParams p) {
    const uint32_t b = blockIdx.x;
    const scz_info& in = p.info[b];
    if (p.status[b] != SCZ_OK) return;
    __shared__ uint32_t s_scan[33];
    const uint32_t nch = (uint32_t)((in.n_rows + ROW_CHUNK - 1) / ROW_CHUNK);
    uint32_t* cs = p.chunk_sum + (uint64_t)b * p.nchunk_cap;
    unsigned long long carry = 0;
    for (uint32_t base = 0; base < nch; base += 256) {
        uint32_t i = base + threadIdx.x;
        uint32_t v = i < nch ? cs[i] : 0;
        uint32_t tot;
        uint32_t ex = block_exclusive_scan<256>(v, s_scan, &tot);
        if (i < nch) cs[i] = (uint32_t)(carry + ex);
        carry += tot;
    }
    if (threadIdx.x == 0 && carry != in.nnz) p.status[b] = SCZ_CORRUPT_STREAM;  // sparse.py:84-87
}

template <typename S, bool STAGE>
__global__ void __launch_bounds__(ROW_THREADS) k_rows_out(RowParams p) {
    const uint32_t b = blockIdx.y, chunk = blockIdx.x;
    const scz_info& in = p.info[b];
    if (p.status[b] != SCZ_OK || in.sym_bytes != sizeof(S)) return;
    const uint64_t N = in.n_rows, r0 = (uint64_t)chunk * ROW_CHUNK;
    if (r0 >= N) return;
    const uint32_t K = in.n_cols;
    const uint64_t nnz = in.nnz;
    const S* d = reinterpret_cast<const S*>(p.dsym) + (uint64_t)b * p.dsym_stride;
    const S* vals = d;
    const S* cols = d + nnz;
    const S* rc = d + 2 * nnz;
    __shared__ uint32_t s_off[ROW_CHUNK];
    __shared__ uint32_t s_scan[33];
    __shared__ float s_lut[256];
    __shared__ int s_bad;
    const uint32_t nrow = (uint32_t)((N - r0) < (uint64_t)ROW_CHUNK ? (N - r0) : (uint64_t)ROW_CHUNK);
    // dequantisation LUT: float32(float64(q - z) * scale) (tensor.py:154)
    const uint32_t nq = in.q_bits <= 8 ? (1u << in.q_bits) : 256u;  // header q_bits is unchecked here
    if (!STAGE)
        for (uint32_t i = threadIdx.x; i < nq; i += ROW_THREADS)
            s_lut[i] = __double2float_rn(__dmul_rn(__dsub_rn((double)i, (double)in.zero_point), in.scale));
    if (threadIdx.x == 0) s_bad = 0;
    // per-chunk row offsets: each thread scans 16 consecutive rows
    constexpr int PER = ROW_CHUNK / ROW_THREADS;
    uint32_t loc[PER], sum = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        uint32_t i = threadIdx.x * PER + j;
        loc[j] = i < nrow ? (uint32_t)rc[r0 + i] : 0;
        sum += loc[j];
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan<ROW_THREADS>(sum, s_scan, &tot);
    const uint32_t cbase = p.chunk_sum[(uint64_t)b * p.nchunk_cap + chunk];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        s_off[threadIdx.x * PER + j] = cbase + ex;
        ex += loc[j];
    }
    __syncthreads();
    bool bad = false;
    float* orow_base = STAGE ? nullptr : p.out + p.out_off[b];
    for (uint32_t li = threadIdx.x; li < nrow; li += ROW_THREADS) {
        const uint64_t i = r0 + li;
        const uint32_t off = s_off[li];
        const uint32_t r = (uint32_t)rc[i];
        uint32_t prev = 0xffffffffu;
        uint32_t j = 0;
        uint32_t nc = r ? (uint32_t)cols[off] : 0xffffffffu;
        if (STAGE) {
            uint32_t* qo = p.q_out + i * K;
            uint8_t* mo = p.mask_out + i * K;
            for (uint32_t col = 0; col < K; ++col) {
                if (j < r && nc == col) {
                    qo[col] = (uint32_t)vals[off + j];
                    mo[col] = 0;
                    prev = nc;
                    ++j;
                    nc = j < r ? (uint32_t)cols[off + j] : 0xffffffffu;
                    if (j < r && (nc <= prev || nc >= K)) bad = true;
                } else {
                    qo[col] = 0;
                    mo[col] = 1;
                }
            }
        } else {
            float* orow = orow_base + i * K;
            for (uint32_t col = 0; col < K; ++col) {
                float o = 0.0f;
                if (j < r && nc == col) {
                    const uint32_t v = (uint32_t)vals[off + j];
                    o = v < nq ? s_lut[v]
                               : __double2float_rn(__dmul_rn(
                                     __dsub_rn((double)v, (double)in.zero_point), in.scale));
                    prev = nc;
                    ++j;
                    nc = j < r ? (uint32_t)cols[off + j] : 0xffffffffu;
                    if (j < r && (nc <= prev || nc >= K)) bad = true;
                }
                orow[col] = o;
            }
        }
        if (j != r) bad = true;  // a column >= K or out of order was never matched
    }
    if (bad) s_bad = 1;
    __syncthreads();
    if (threadIdx.x == 0 && s_bad) p.status[b] = SCZ_CORRUPT_STREAM;
}

#define SCZ_INST_ROWS(S)                                        \
    template __global__ void k_row_sums<S>(RowParams);          \
    template __global__ void k_rows_out<S, false>(RowParams);   \
    template __global__ void k_rows_out<S, true>(RowParams);
SCZ_INST_ROWS(uint8_t)
SCZ_INST_ROWS(uint16_t)
SCZ_INST_ROWS(uint32_t)

// ------------------------------------------------------ stage-API helpers
// zero mask (u8) -> bitmap + per-tile nnz (tile_stats.z), for csr_encode.
__global__ void __launch_bounds__(TILE_THREADS) k_mask_bitmap(const uint8_t* mask, uint64_t n,
                                                              uint32_t* bitmap, uint32_t* tile_nnz) {
    const uint32_t tile = blockIdx.x;
    const uint64_t w = (uint64_t)tile * TILE_WORDS + threadIdx.x;
    uint32_t word = 0;
    for (int j = 0; j < 32; ++j) {
        uint64_t idx = w * 32 + j;
        if (idx < n && !mask[idx]) word |= 1u << j;
    }
    bitmap[w] = word;
    uint32_t c = warp_sum((uint32_t)__popc(word));
    __shared__ uint32_t s[TILE_THREADS / 32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < TILE_THREADS / 32; ++i) c += s[i];
        tile_nnz[tile] = c;
    }
}

// exclusive scan of per-tile counts (single CTA); total -> *nnz
__global__ void __launch_bounds__(256) k_tile_scan(uint32_t* cnt, uint32_t n, uint64_t* nnz) {
    __shared__ uint32_t s_scan[33];
    unsigned long long carry = 0;
    for (uint32_t base = 0; base < n; base += 256) {
        uint32_t i = base + threadIdx.x;
        uint32_t v = i < n ? cnt[i] : 0;
        uint32_t tot;
        uint32_t ex = block_exclusive_scan<256>(v, s_scan, &tot);
        if (i < n) cnt[i] = (uint32_t)(carry + ex);
        carry += tot;
    }
    if (threadIdx.x == 0) *nnz = carry;
}

// values at original-nonzero positions, rank order (sparse.py:65-67)
__global__ void __launch_bounds__(TILE_THREADS) k_compact_u32(const uint32_t* q, const uint32_t* bitmap,
                                                              const uint32_t* tile_off, uint32_t* d) {
    const uint32_t tile = blockIdx.x;
    __shared__ uint32_t s_scan[33];
    const uint64_t w = (uint64_t)tile * TILE_WORDS + threadIdx.x;
    uint32_t word = bitmap[w], tot;
    uint32_t rank = tile_off[tile] + block_exclusive_scan<TILE_THREADS>(__popc(word), s_scan, &tot);
    while (word) {
        int bit = __ffs(word) - 1;
        word &= word - 1;
        d[rank++] = q[w * 32 + bit];
    }
}

__global__ void k_unpack_mask(const uint32_t* bitmap, uint64_t n, uint8_t* mask) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) mask[i] = ((bitmap[i >> 5] >> (i & 31)) & 1u) ? 0 : 1;
}

__global__ void k_dequant_flat(const uint32_t* q, const uint8_t* mask, uint64_t n, double scale,
                               int64_t z, float* out) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n)
        out[i] = mask[i] ? 0.0f
                         : __double2float_rn(__dmul_rn(__dsub_rn((double)q[i], (double)z), scale));
}

// bincount with AlphabetOverflow flag (rans.py:76-85)
__global__ void k_hist_u32(const uint32_t* d, uint64_t n, uint32_t A, uint32_t* counts,
                           int32_t* overflow) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        uint32_t v = d[i];
        if (v >= A) *overflow = 1;
        else atomicAdd(counts + v, 1u);
    }
}

}  // namespace scz
