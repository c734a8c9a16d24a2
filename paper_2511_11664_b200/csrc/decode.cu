// decode.cu -- CSR decode + dequantisation (K8) and the small
// stage kernels used by the parity entry points.
//
// Rows are processed in chunks of R(K) = min(1024, 4096 / K) rows so a chunk's
// dense output (R*K fp32) fits 16 KB of shared memory; its column and value
// segments are staged there too with coalesced loads before the scatter.
// One pass: each chunk sums its row counts (r <= K check, sparse.py:88-89),
// publishes the sum and finds its nonzero offset by decoupled look-back over
// the previous chunks of the tensor (the last chunk checks sum(r) == nnz,
// sparse.py:84-87); then
//   k_rows_out   per chunk: row offsets (block scan), column checks (col < K,
//                strictly increasing: sparse.py:90-97); the dense rows are
//                assembled in shared memory -- +0.0 everywhere, LUT[v] at the
//                listed columns (tensor.py:154-155) -- and written back with
//                coalesced 16-byte stores; or (q, mask) for the stage API.
#include "common.cuh"

namespace scz {

constexpr int ROW_CHUNK = 1024;     // max rows per chunk
constexpr int OUT_ELEMS = 4096;     // dense fp32 elements staged per chunk
constexpr int ROW_THREADS = 256;
constexpr int SMALL8_THREADS = 256;  // k_rows_small8: SMALL_ROWS / 8 rows per thread

__host__ __device__ inline uint32_t rows_per_chunk(uint32_t K) {
    const uint32_t r = K ? (uint32_t)OUT_ELEMS / K : (uint32_t)ROW_CHUNK;
    return r < 1 ? 1u : (r > (uint32_t)ROW_CHUNK ? (uint32_t)ROW_CHUNK : r);
}

// Rows per chunk of the decode pipeline's row kernels: u8 symbols with
// K in {1, 2, 4} go to k_rows_small8 (SMALL_ROWS), everything else (and the
// stage API) to the kernels chunked by rows_per_chunk.
constexpr uint32_t SMALL_ROWS = SMALL_ROWS_DEC;  // chunk sums from the v2 decoder
__host__ __device__ inline uint32_t dec_chunk_rows(uint32_t K, uint32_t sym_bytes, bool stage) {
    return (!stage && sym_bytes == 1 && (K == 1 || K == 2 || K == 4)) ? SMALL_ROWS : rows_per_chunk(K);
}

// float32((float64(v) - z) * scale) (tensor.py:154).  The 256-entry LUT covers
// every u8 symbol; wider symbols >= 256 (only in hand-made streams) take an
// out-of-line fp64 path so it is never if-converted into the hot loop.
__device__ __noinline__ float dequant_slow(uint32_t v, double z, double scale) {
    return __double2float_rn(__dmul_rn(__dsub_rn((double)v, z), scale));
}
template <typename S>
__device__ __forceinline__ float dequant(uint32_t v, const float* lut, double z, double scale) {
    if constexpr (sizeof(S) == 1) return lut[v];
    else return v < 256u ? lut[v] : dequant_slow(v, z, scale);
}

struct RowParams {
    const scz_info* info;   // [B]
    const void* dsym;       // decoded D: tensor b's row at byte b * dsym_stride
    uint64_t dsym_stride;   // bytes (Lmax x the widest symbol class of the batch)
    unsigned long long* chunk_state;  // [B][nchunk_cap] look-back words, zeroed per launch
    uint32_t nchunk_cap;
    int32_t* status;        // [B]
    float* out;             // [B] tensors at out_off[b]
    const uint64_t* out_off;
    uint32_t* q_out;        // stage API: symbols
    uint8_t* mask_out;      // stage API: zero mask
    const float* dq_lut;    // [B][256] from k_dec_prepare (k_rows_small8)
};

// A chunk of a tensor already marked bad (possibly by another chunk of this
// very launch) still publishes, so later chunks never wait on it forever.
__device__ bool chunk_dead(const RowParams& p, uint32_t b, uint32_t chunk) {
    __shared__ int s_dead;  // one read for the CTA: status may change under us
    if (threadIdx.x == 0) s_dead = *(const volatile int32_t*)(p.status + b) != SCZ_OK;
    __syncthreads();
    if (s_dead && threadIdx.x < 32) chunk_prefix(p.chunk_state + (uint64_t)b * p.nchunk_cap, chunk, 0);
    return s_dead != 0;
}

// Chunk offset of the block (all threads): publishes `tot`, returns the
// exclusive prefix; flags s_bad when the chunk's nonzeros overrun nnz or the
// last chunk's inclusive sum differs from nnz (sparse.py:84-87).
__device__ uint32_t block_chunk_base(const RowParams& p, uint32_t b, uint32_t chunk, uint32_t tot, uint64_t nnz,
                                     bool last, int* s_bad) {
    __shared__ uint32_t s_base;
    if (threadIdx.x < 32) {
        const uint32_t e = chunk_prefix(p.chunk_state + (uint64_t)b * p.nchunk_cap, chunk, tot);
        if (threadIdx.x == 0) {
            s_base = e;
            if ((uint64_t)e + tot > nnz || (last && (uint64_t)e + tot != nnz)) *s_bad = 1;
        }
    }
    __syncthreads();
    return s_base;
}

template <typename S, bool STAGE>
__global__ void __launch_bounds__(ROW_THREADS) k_rows_out(RowParams p) {
    pdl_wait();
    const uint32_t b = blockIdx.y, chunk = blockIdx.x;
    const scz_info& in = p.info[b];
    if (in.sym_bytes != sizeof(S)) return;
    const uint32_t K = in.n_cols;
    if (!STAGE && sizeof(S) <= 2 && K <= (uint32_t)OUT_ELEMS) return;  // k_rows_fast's case
    const uint32_t R = rows_per_chunk(K);
    const uint64_t N = in.n_rows, r0 = (uint64_t)chunk * R;
    if (r0 >= N) return;
    if (chunk_dead(p, b, chunk)) return;
    const uint64_t nnz = in.nnz;
    const S* d = reinterpret_cast<const S*>(reinterpret_cast<const uint8_t*>(p.dsym) + (uint64_t)b * p.dsym_stride);
    const S* vals = d;
    const S* cols = d + nnz;
    const S* rc = d + 2 * nnz;
    __shared__ uint32_t s_off[ROW_CHUNK];
    __shared__ __align__(16) float s_out[OUT_ELEMS];
    __shared__ uint32_t s_scan[33];
    __shared__ float s_lut[256];
    __shared__ int s_bad;
    constexpr bool STAGE_CV = !STAGE && sizeof(S) <= 2;
    __shared__ S s_cs[STAGE_CV ? OUT_ELEMS : 1], s_vs[STAGE_CV ? OUT_ELEMS : 1];
    const uint32_t nrow = (uint32_t)((N - r0) < (uint64_t)R ? (N - r0) : (uint64_t)R);
    // dequantisation LUT: float32(float64(q - z) * scale) (tensor.py:154)
    if (!STAGE) build_dequant_lut(s_lut, (double)in.zero_point, in.scale);
    if (threadIdx.x == 0) s_bad = 0;
    // per-chunk row offsets: each thread scans ROW_CHUNK / 256 consecutive rows
    constexpr int PER = ROW_CHUNK / ROW_THREADS;
    uint32_t loc[PER], sum = 0;
    bool rbad = false;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t i = threadIdx.x * PER + j;
        const uint32_t v = i < nrow ? (uint32_t)rc[r0 + i] : 0;
        rbad |= v > K;  // sparse.py:88-89
        loc[j] = min(v, K + 1);
        sum += loc[j];
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan<ROW_THREADS>(sum, s_scan, &tot);
    if (rbad) s_bad = 1;
    const uint32_t cbase = block_chunk_base(p, b, chunk, tot, nnz, r0 + nrow == N, &s_bad);
    if (s_bad) {
        if (threadIdx.x == 0) p.status[b] = SCZ_CORRUPT_STREAM;
        return;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        s_off[threadIdx.x * PER + j] = cbase + ex;
        ex += loc[j];
    }
    const uint32_t n_el = nrow * K;  // <= OUT_ELEMS unless K > OUT_ELEMS (then nrow == 1)
    const bool staged = !STAGE && n_el <= (uint32_t)OUT_ELEMS;
    if (staged)
        for (uint32_t i = threadIdx.x; i < n_el; i += ROW_THREADS) s_out[i] = 0.0f;
    // the chunk's nonzeros are [cbase, cbase + tot): stage their columns and values
    const bool cv_staged = STAGE_CV && staged && tot <= (uint32_t)OUT_ELEMS;
    if constexpr (STAGE_CV) {
        if (cv_staged)
            for (uint32_t i = threadIdx.x; i < tot; i += ROW_THREADS) {
                s_cs[i] = cols[cbase + i];
                s_vs[i] = vals[cbase + i];
            }
    }
    __syncthreads();
    bool bad = false;
    float* ochunk = STAGE ? nullptr : p.out + p.out_off[b] + r0 * K;
    for (uint32_t li = threadIdx.x; li < nrow; li += ROW_THREADS) {
        const uint64_t i = r0 + li;
        const uint32_t off = s_off[li];
        const uint32_t r = (uint32_t)rc[i];
        if (STAGE) {
            uint32_t* qo = p.q_out + i * K;
            uint8_t* mo = p.mask_out + i * K;
            for (uint32_t col = 0; col < K; ++col) {
                qo[col] = 0;
                mo[col] = 1;
            }
        } else if (!staged) {
            for (uint32_t col = 0; col < K; ++col) ochunk[(uint64_t)li * K + col] = 0.0f;
        }
        uint32_t prev = 0;
        for (uint32_t j = 0; j < r; ++j) {
            const uint32_t c = cv_staged ? (uint32_t)s_cs[off - cbase + j] : (uint32_t)cols[off + j];
            if (c >= K || (j > 0 && c <= prev)) {  // sparse.py:90-97
                bad = true;
                break;
            }
            prev = c;
            const uint32_t v = cv_staged ? (uint32_t)s_vs[off - cbase + j] : (uint32_t)vals[off + j];
            if (STAGE) {
                p.q_out[i * K + c] = v;
                p.mask_out[i * K + c] = 0;
            } else {
                const float o = dequant<S>(v, s_lut, (double)in.zero_point, in.scale);
                if (staged) s_out[li * K + c] = o;
                else ochunk[(uint64_t)li * K + c] = o;
            }
        }
    }
    if (bad) s_bad = 1;
    __syncthreads();
    if (threadIdx.x == 0 && s_bad) p.status[b] = SCZ_CORRUPT_STREAM;
    if (staged && !s_bad) {
        // coalesced write-back of the chunk's dense rows
        const uintptr_t addr = reinterpret_cast<uintptr_t>(ochunk);
        if ((addr & 15) == 0) {
            const uint32_t n4 = n_el / 4;
            for (uint32_t i = threadIdx.x; i < n4; i += ROW_THREADS)
                reinterpret_cast<float4*>(ochunk)[i] = reinterpret_cast<const float4*>(s_out)[i];
            for (uint32_t i = 4 * n4 + threadIdx.x; i < n_el; i += ROW_THREADS) ochunk[i] = s_out[i];
        } else {
            for (uint32_t i = threadIdx.x; i < n_el; i += ROW_THREADS) ochunk[i] = s_out[i];
        }
    }
}

// Fast path of k_rows_out for u8/u16 symbols and K <= OUT_ELEMS (the search
// path and every BASELINE config): the chunk's columns and values are staged
// with coalesced loads, rows are scattered into a zeroed shared tile, and the
// tile is written back with 16-byte stores.  Static shared arrays only.
template <typename S>
__global__ void __launch_bounds__(ROW_THREADS) k_rows_fast(RowParams p) {
    pdl_wait();
    const uint32_t b = blockIdx.y, chunk = blockIdx.x;
    const scz_info& in = p.info[b];
    if (in.sym_bytes != sizeof(S)) return;
    const uint32_t K = in.n_cols;
    if (K > (uint32_t)OUT_ELEMS) return;       // k_rows_out handles these
    if (K == 1 || K == 2 || K == 4) return;    // k_rows_small handles these
    const uint32_t R = rows_per_chunk(K);
    const uint64_t N = in.n_rows, r0 = (uint64_t)chunk * R;
    if (r0 >= N) return;
    if (chunk_dead(p, b, chunk)) return;
    const uint64_t nnz = in.nnz;
    const S* d = reinterpret_cast<const S*>(reinterpret_cast<const uint8_t*>(p.dsym) + (uint64_t)b * p.dsym_stride);
    __shared__ uint32_t s_off[ROW_CHUNK];
    __shared__ __align__(16) float s_out[OUT_ELEMS];
    __shared__ S s_c[OUT_ELEMS], s_v[OUT_ELEMS];
    __shared__ uint32_t s_scan[33];
    __shared__ float s_lut[256];
    __shared__ int s_bad;
    const uint32_t nrow = (uint32_t)((N - r0) < (uint64_t)R ? (N - r0) : (uint64_t)R);
    build_dequant_lut(s_lut, (double)in.zero_point, in.scale);
    if (threadIdx.x == 0) s_bad = 0;
    constexpr int PER = ROW_CHUNK / ROW_THREADS;
    uint32_t loc[PER], sum = 0;
    const S* rc = d + 2 * nnz + r0;
    bool rbad = false;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t i = threadIdx.x * PER + j;
        const uint32_t v = i < nrow ? (uint32_t)rc[i] : 0u;
        rbad |= v > K;  // sparse.py:88-89
        loc[j] = min(v, K + 1);
        sum += loc[j];
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan<ROW_THREADS>(sum, s_scan, &tot);
    if (rbad) s_bad = 1;
    const uint32_t cbase = block_chunk_base(p, b, chunk, tot, nnz, r0 + nrow == N, &s_bad);
    if (s_bad) {  // tot <= nrow * K holds from here on
        if (threadIdx.x == 0) p.status[b] = SCZ_CORRUPT_STREAM;
        return;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        s_off[threadIdx.x * PER + j] = ex;  // chunk-local offset
        ex += loc[j];
    }
    const uint32_t n_el = nrow * K;
    for (uint32_t i = threadIdx.x; i < OUT_ELEMS / 4; i += ROW_THREADS)
        reinterpret_cast<float4*>(s_out)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    const S* gc = d + nnz + cbase;
    const S* gv = d + cbase;
    for (uint32_t i = threadIdx.x; i < tot; i += ROW_THREADS) {  // tot <= nrow * K (checked above)
        s_c[i] = gc[i];
        s_v[i] = gv[i];
    }
    __syncthreads();
    bool bad = false;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t li = threadIdx.x * PER + j;  // this thread's rows (their counts are in loc[])
        if (li >= nrow) break;
        const uint32_t off = s_off[li], r = loc[j];
        uint32_t prev = 0;
        for (uint32_t e = 0; e < r; ++e) {
            const uint32_t c = s_c[off + e];
            bad |= (c >= K) | ((e > 0) & (c <= prev));  // sparse.py:90-97
            prev = c;
            const uint32_t v = s_v[off + e];
            const float o = dequant<S>(v, s_lut, (double)in.zero_point, in.scale);
            if (c < K) s_out[li * K + c] = o;
        }
    }
    if (bad) s_bad = 1;
    __syncthreads();
    if (s_bad) {
        if (threadIdx.x == 0) p.status[b] = SCZ_CORRUPT_STREAM;
        return;
    }
    float* ochunk = p.out + p.out_off[b] + r0 * K;
    if ((reinterpret_cast<uintptr_t>(ochunk) & 15) == 0) {
        const uint32_t n4 = n_el / 4;
        for (uint32_t i = threadIdx.x; i < n4; i += ROW_THREADS)
            reinterpret_cast<float4*>(ochunk)[i] = reinterpret_cast<const float4*>(s_out)[i];
        for (uint32_t i = 4 * n4 + threadIdx.x; i < n_el; i += ROW_THREADS) ochunk[i] = s_out[i];
    } else {
        for (uint32_t i = threadIdx.x; i < n_el; i += ROW_THREADS) ochunk[i] = s_out[i];
    }
}
template __global__ void k_rows_fast<uint8_t>(RowParams);
template __global__ void k_rows_fast<uint16_t>(RowParams);

// K in {1, 2, 4} (every BASELINE shape picks one of these): a row is one
// 4/8/16-byte vector assembled in registers from <= K independent,
// predicated loads; consecutive threads own consecutive rows, so every store
// instruction of a warp is one contiguous, coalesced span.
template <typename S, int KK>
__global__ void __launch_bounds__(ROW_THREADS) k_rows_small(RowParams p) {
    pdl_wait();
    const uint32_t b = blockIdx.y, chunk = blockIdx.x;
    const scz_info& in = p.info[b];
    if (in.sym_bytes != sizeof(S) || in.n_cols != (uint32_t)KK) return;
    if (sizeof(S) == 1) return;                  // k_rows_small8 handles u8
    constexpr uint32_t R = (uint32_t)ROW_CHUNK;  // == rows_per_chunk(KK) for KK <= 4
    const uint64_t N = in.n_rows, r0 = (uint64_t)chunk * R;
    if (r0 >= N) return;
    if (chunk_dead(p, b, chunk)) return;
    const uint64_t nnz = in.nnz;
    const S* d = reinterpret_cast<const S*>(reinterpret_cast<const uint8_t*>(p.dsym) + (uint64_t)b * p.dsym_stride);
    __shared__ uint32_t s_off[ROW_CHUNK];
    __shared__ uint8_t s_r[ROW_CHUNK];
    __shared__ uint32_t s_scan[33];
    __shared__ float s_lut[256];
    __shared__ int s_bad;
    const uint32_t nrow = (uint32_t)((N - r0) < (uint64_t)R ? (N - r0) : (uint64_t)R);
    build_dequant_lut(s_lut, (double)in.zero_point, in.scale);
    if (threadIdx.x == 0) s_bad = 0;
    constexpr int PER = ROW_CHUNK / ROW_THREADS;
    uint32_t loc[PER], sum = 0;
    const S* rc = d + 2 * nnz + r0;
    bool rbad = false;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t i = threadIdx.x * PER + j;
        const uint32_t v = i < nrow ? (uint32_t)rc[i] : 0u;
        rbad |= v > (uint32_t)KK;  // sparse.py:88-89
        loc[j] = min(v, (uint32_t)KK + 1);
        sum += loc[j];
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan<ROW_THREADS>(sum, s_scan, &tot);
    if (rbad) s_bad = 1;
    ex += block_chunk_base(p, b, chunk, tot, nnz, r0 + nrow == N, &s_bad);
    if (s_bad) {
        if (threadIdx.x == 0) p.status[b] = SCZ_CORRUPT_STREAM;
        return;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        s_off[threadIdx.x * PER + j] = ex;
        s_r[threadIdx.x * PER + j] = (uint8_t)loc[j];
        ex += loc[j];
    }
    __syncthreads();
    const S* cols = d + nnz;
    float* orow0 = p.out + p.out_off[b] + r0 * KK;
    // rows are KK floats: one alignment test for the whole chunk (uniform)
    const bool vec_ok = (reinterpret_cast<uintptr_t>(orow0) & (KK * 4 - 1)) == 0;
    bool bad = false;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t li = j * ROW_THREADS + threadIdx.x;
        if (li >= nrow) break;
        const uint32_t off = s_off[li], r = s_r[li];
        // branch-free: clamped unconditional loads, then a column-presence mask
        uint32_t c[KK];
        float a[KK];
        uint32_t mask = 0;
#pragma unroll
        for (int e = 0; e < KK; ++e) {
            const bool live = (uint32_t)e < r;
            const uint32_t idx = off + (live ? (uint32_t)e : 0u);  // off <= nnz: in-bounds
            c[e] = (uint32_t)cols[idx];
            a[e] = dequant<S>((uint32_t)d[idx], s_lut, (double)in.zero_point, in.scale);
            const bool order_bad = e > 0 && c[e] <= c[e > 0 ? e - 1 : 0];
            bad |= live & ((c[e] >= (uint32_t)KK) | order_bad);  // sparse.py:90-97
            mask |= live ? (1u << (c[e] & (KK - 1))) : 0u;
        }
        float o[KK];
#pragma unroll
        for (int col = 0; col < KK; ++col) {
            const uint32_t before = __popc(mask & ((1u << col) - 1u));  // entries left of col
            float val = a[0];
#pragma unroll
            for (int e = 1; e < KK; ++e) val = before == (uint32_t)e ? a[e] : val;
            o[col] = (mask >> col) & 1u ? val : 0.0f;
        }
        float* orow = orow0 + (uint64_t)li * KK;
        if constexpr (KK == 4) {
            if (vec_ok) __stcs(reinterpret_cast<float4*>(orow), make_float4(o[0], o[1], o[2], o[3]));
            else { orow[0] = o[0]; orow[1] = o[1]; orow[2] = o[2]; orow[3] = o[3]; }
        } else if constexpr (KK == 2) {
            if (vec_ok) __stcs(reinterpret_cast<float2*>(orow), make_float2(o[0], o[1]));
            else { orow[0] = o[0]; orow[1] = o[1]; }
        } else {
            __stcs(orow, o[0]);
        }
    }
    if (bad) s_bad = 1;
    __syncthreads();
    if (threadIdx.x == 0 && s_bad) p.status[b] = SCZ_CORRUPT_STREAM;
}
// Copy n bytes starting at an arbitrary global address into shared memory
// with aligned 16-byte loads: byte i lands at dst[sh + i], sh = src & 15
// (returned).  dst must hold n + 31 bytes; the over-read of up to 15 bytes
// either side stays inside the caller's allocation.
// The copies are cp.async (every 16-byte piece in flight at once, none
// blocking the thread); the caller commits, waits and synchronises.
__device__ __forceinline__ uint32_t stage_window(uint8_t* dst, const uint8_t* src, uint32_t n) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src) & ~(uintptr_t)15;
    const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(src) - a);
    const uint32_t n16 = (sh + n + 15) >> 4;
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x)
        cp_async16(dst + 16 * i, reinterpret_cast<const uint4*>(a) + i);
    return sh;
}

// The 16-byte aligned span holding n bytes at src, for one bulk copy: byte i
// lands at dst[sh + i] (same contract as stage_window).
struct Win {
    const uint8_t* a;
    uint32_t sh, bytes;
};
__device__ __forceinline__ Win window_of(const uint8_t* src, uint32_t n) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src) & ~(uintptr_t)15;
    const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(src) - a);
    return Win{reinterpret_cast<const uint8_t*>(a), sh, ((sh + n + 15) >> 4) << 4};
}

// 4 consecutive bytes at byte offset o of a shared array (any alignment).
__device__ __forceinline__ uint32_t smem_word_at(const uint8_t* s, uint32_t o) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(s) + (o >> 2);
    return __funnelshift_r(w[0], w[1], (o & 3) * 8);
}

// u8 symbols, K in {1, 2, 4} (the decode pipeline's hot case: every BASELINE
// shape picks one of these).  A chunk is SMALL_ROWS rows.  Its row counts,
// and after the chunk's nonzero offset is known its column and value
// segments, are staged into shared memory with aligned 16-byte loads; a row
// then reads its <= 4 columns and values as one funnel-shifted word each, so
// a row costs a handful of instructions.  Consecutive threads own
// consecutive rows: every store instruction of a warp is one contiguous,
// coalesced span of 32 rows.  Checks as sparse.py:84-97.
// K = 4 row table: entry [r][idx], idx = the low two bits of the row's four
// column bytes packed (c0 | c1 << 2 | c2 << 4 | c3 << 6), only the first r
// fields meaningful.  Entry = PRMT selector (16 bits: nibble j = rank of
// column j among the row's columns, 4 = absent) | mask << 16 (present
// columns) | valid << 20 (the r columns strictly increase, sparse.py:90-97).
// Initialised once per device by k_init_row_lut (scz_ctx_create).
__device__ __align__(16) uint32_t g_row_lut4[5 * 256];

__global__ void k_init_row_lut() {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 5 * 256) return;
    const uint32_t r = i >> 8, idx = i & 255;
    uint32_t mask = 0, valid = 1, prev = 0;
    for (uint32_t e = 0; e < r; ++e) {
        const uint32_t c = (idx >> (2 * e)) & 3u;
        if (e > 0 && c <= prev) valid = 0;
        mask |= 1u << c;
        prev = c;
    }
    uint32_t sel = 0, k = 0;
    for (uint32_t j = 0; j < 4; ++j) {
        const bool here = (mask >> j) & 1u;
        sel |= (here ? k : 4u) << (4 * j);
        k += here;
    }
    g_row_lut4[i] = sel | (mask << 16) | (valid << 20);
}

// SUMS: v2 tensors (decoder chunk sums); else v1 (look-back).  VEC: every
// output row is KK * 4-byte aligned (host-checked), so rows leave with one
// vector store and no alignment test.
template <int KK, bool SUMS, bool VEC = false>
__global__ void __launch_bounds__(SMALL8_THREADS, SUMS ? 6 : 1) k_rows_small8(RowParams p) {
    static_assert(KK == 1 || KK == 2 || KK == 4, "row width");
    constexpr uint32_t R = SMALL_ROWS;
    constexpr uint32_t PER = R / SMALL8_THREADS;
    constexpr uint32_t MAXE = R * KK;  // nonzeros of a valid chunk
    __shared__ __align__(16) uint8_t s_r[R + 32];
    __shared__ __align__(16) uint8_t s_c[MAXE + 32];
    __shared__ __align__(16) uint8_t s_v[MAXE + 32];
    __shared__ __align__(16) uint32_t s_or[R];  // row: nonzero offset in the chunk | count << 16
    __shared__ uint32_t s_scan[33];
    __shared__ __align__(1024) float s_lut[256];  // bin address = base | 4 * symbol
    __shared__ int s_bad;
    // per column-presence mask: the sorted column packing and the PRMT
    // selector that moves the k-th value byte to its column (4 = zero byte)
    __shared__ uint32_t s_pk[1 << KK], s_sel[1 << KK];
    __shared__ __align__(16) uint32_t s_lut4[KK == 4 ? 5 * 256 : 4];
    if (threadIdx.x < (1u << KK)) {  // no dependency on the decoder: before the wait
        uint32_t pk = 0, sel = 0, k = 0;
        for (uint32_t j = 0; j < 4; ++j) {
            const bool here = j < (uint32_t)KK && ((threadIdx.x >> j) & 1u);
            if (here) pk |= j << (8 * k);
            sel |= (here ? k : 4u) << (4 * j);
            k += here;
        }
        s_pk[threadIdx.x] = pk;
        s_sel[threadIdx.x] = sel;
    }
    // SUMS: [0] r window + both tables, [1] c and v windows (bulk copies)
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ uint32_t s_cb[3];  // SUMS: chunk's nonzero offset, count, ok (warp 0)
    if (threadIdx.x == 0) {
        s_bad = 0;
        if (SUMS) {
            mbar_init(&s_bar[0], 1);
            mbar_init(&s_bar[1], 1);
        }
    }
    pdl_wait();
    const uint32_t b = blockIdx.y, chunk = blockIdx.x;
    const scz_info& in = p.info[b];
    const uint64_t out_off = p.out_off[b];
    if (in.sym_bytes != 1 || in.n_cols != (uint32_t)KK) return;
    const uint64_t N = in.n_rows, r0 = (uint64_t)chunk * R;
    if (r0 >= N) return;
    if ((in.version == 2) != SUMS) return;  // the other variant's tensor
    const uint64_t nnz = in.nnz;
    const uint32_t nrow = (uint32_t)((N - r0) < (uint64_t)R ? (N - r0) : (uint64_t)R);
    const uint8_t* d = reinterpret_cast<const uint8_t*>(p.dsym) + (uint64_t)b * p.dsym_stride;
    uint32_t cbase = 0, own = 0, rsh, csh = 0, vsh = 0;
    if constexpr (SUMS) {
        // v2 tensors: the decoder summed every chunk's row counts.  Warp 0
        // alone puts the r window and both tables in flight (one bulk copy
        // each, before the prefix is known), reduces the earlier chunks'
        // counts to the chunk's nonzero offset, checks it and starts the c
        // and v windows; the other warps learn the result at one barrier.
        // Two memory round trips, as before, without a 256-thread copy loop.
        rsh = window_of(d + 2 * nnz + r0, nrow).sh;
        if (threadIdx.x < 32) {
            const uint32_t lane = threadIdx.x;
            if (lane == 0) {
                const Win wr = window_of(d + 2 * nnz + r0, nrow);
                mbar_expect_tx(&s_bar[0], wr.bytes + 1024u + (KK == 4 ? 5u * 256u * 4u : 0u));
                bulk_g2s(s_r, wr.a, wr.bytes, &s_bar[0]);
                bulk_g2s(s_lut, p.dq_lut + (uint64_t)b * 256, 1024u, &s_bar[0]);
                if constexpr (KK == 4) bulk_g2s(s_lut4, g_row_lut4, 5u * 256u * 4u, &s_bar[0]);
            }
            const int32_t st0 = *(const volatile int32_t*)(p.status + b);
            const unsigned long long* cs = p.chunk_state + (uint64_t)b * p.nchunk_cap;
            const unsigned long long mine = cs[chunk];
            unsigned long long acc = 0;
            for (uint32_t j0 = 0; j0 < chunk; j0 += 128) {  // four loads in flight per lane
                unsigned long long v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t j = j0 + 32 * k + lane;
                    v[k] = j < chunk ? cs[j] : 0ull;
                }
                acc += (v[0] + v[1]) + (v[2] + v[3]);
            }
            acc = warp_sum(acc);
            if (lane == 0) {
                const uint32_t cb = (uint32_t)min(acc, 0xFFFFFFFFull);
                const uint32_t ow = (uint32_t)min(mine, 0xFFFFFFFFull);
                const bool ok = st0 == SCZ_OK && ow <= nrow * KK && (uint64_t)cb + ow <= nnz;
                if (st0 == SCZ_OK && !ok) p.status[b] = SCZ_CORRUPT_STREAM;
                if (ok) {
                    const Win wc = window_of(d + nnz + cb, ow), wv = window_of(d + cb, ow);
                    mbar_expect_tx(&s_bar[1], wc.bytes + wv.bytes);
                    if (wc.bytes) bulk_g2s(s_c, wc.a, wc.bytes, &s_bar[1]);
                    if (wv.bytes) bulk_g2s(s_v, wv.a, wv.bytes, &s_bar[1]);
                }
                s_cb[0] = cb;
                s_cb[1] = ow;
                s_cb[2] = ok;
            }
        }
        __syncthreads();
        if (!s_cb[2]) {  // uniform; no copy may land after the CTA is gone
            if (threadIdx.x == 0) mbar_wait(&s_bar[0], 0);
            return;
        }
        cbase = s_cb[0];
        own = s_cb[1];
        csh = window_of(d + nnz + cbase, own).sh;
        vsh = window_of(d + cbase, own).sh;
        mbar_wait(&s_bar[0], 0);
    } else {
        if (chunk_dead(p, b, chunk)) return;
        if constexpr (KK == 4)
            for (uint32_t i = threadIdx.x; i < 5 * 256 / 4; i += SMALL8_THREADS)
                cp_async16(reinterpret_cast<uint4*>(s_lut4) + i, reinterpret_cast<const uint4*>(g_row_lut4) + i);
        rsh = stage_window(s_r, d + 2 * nnz + r0, nrow);
        if (threadIdx.x < 64)  // the tensor's dequantisation table (k_dec_prepare)
            cp_async16(reinterpret_cast<uint4*>(s_lut) + threadIdx.x,
                       reinterpret_cast<const uint4*>(p.dq_lut + (uint64_t)b * 256) + threadIdx.x);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
    }
    // thread t owns rows [8t, 8t + 8) of the chunk for the scan: their count
    // bytes as two words (bytes past nrow masked off), checked, summed and
    // prefix-summed four at a time (SWAR; counts <= K keep every byte sum
    // below 256), then written as (offset | r << 16) entries, two 16-byte
    // stores per thread
    static_assert(PER == 8, "two count words per thread");
    const uint32_t a_r = (uint32_t)__cvta_generic_to_shared(s_r) + rsh;
    const uint32_t nt = nrow > 8 * threadIdx.x ? min(nrow - 8 * threadIdx.x, 8u) : 0u;
    auto word_at = [](uint32_t a) {  // 4 bytes at any shared byte address
        const uint32_t w = a & ~3u;
        return __funnelshift_r(lds_u32(w), lds_u32(w + 4), (a & 3) * 8);
    };
    const uint32_t w0 = word_at(a_r + 8 * threadIdx.x) & __funnelshift_lc(0xFFFFFFFFu, 0u, 8 * min(nt, 4u));
    const uint32_t w1 = word_at(a_r + 8 * threadIdx.x + 4) & __funnelshift_lc(0xFFFFFFFFu, 0u, 8 * (nt > 4 ? nt - 4 : 0u));
    // a byte > K sets its top bit here (bytes >= 128 already have it)
    constexpr uint32_t KB = (0x7Fu - (uint32_t)KK) * 0x01010101u;
    const bool rbad = (((w0 + KB) | w0 | (w1 + KB) | w1) & 0x80808080u) != 0;  // sparse.py:88-89
    const uint32_t s0 = __dp4a(w0, 0x01010101u, 0u);
    const uint32_t sum = __dp4a(w1, 0x01010101u, s0);
    uint32_t tot;
    uint32_t ex = block_exclusive_scan<SMALL8_THREADS>(sum, s_scan, &tot);
    if (rbad) s_bad = 1;
    if (SUMS) {
        if (threadIdx.x == 0 && (tot != own || (r0 + nrow == N && (uint64_t)cbase + tot != nnz)))  // sparse.py:84-87
            s_bad = 1;
        __syncthreads();
    } else {
        cbase = block_chunk_base(p, b, chunk, tot, nnz, r0 + nrow == N, &s_bad);
    }
    if (s_bad) {  // from here on tot <= nrow * KK and cbase + tot <= nnz
        // no copy may land after the CTA is gone
        if (SUMS) mbar_wait(&s_bar[1], 0);
        else cp_async_wait<0>();
        if (threadIdx.x == 0) p.status[b] = SCZ_CORRUPT_STREAM;
        return;
    }
    {
        // byte k of w * 0x01010100 = sum of bytes < k; byte 0 is 0, which
        // PRMT also uses as the zero filler: entry = [pfx_k, 0, r_k, 0] + ex
        const uint32_t p0 = w0 * 0x01010100u, p1 = w1 * 0x01010100u;
        const uint32_t e1 = ex + s0;
        uint4* dst = reinterpret_cast<uint4*>(s_or) + 2 * threadIdx.x;
        dst[0] = make_uint4(__byte_perm(p0, w0, 0x0400) + ex, __byte_perm(p0, w0, 0x0501) + ex,
                            __byte_perm(p0, w0, 0x0602) + ex, __byte_perm(p0, w0, 0x0703) + ex);
        dst[1] = make_uint4(__byte_perm(p1, w1, 0x0400) + e1, __byte_perm(p1, w1, 0x0501) + e1,
                            __byte_perm(p1, w1, 0x0602) + e1, __byte_perm(p1, w1, 0x0703) + e1);
    }
    if (!SUMS) {  // look-back path: the windows are known only now
        csh = stage_window(s_c, d + nnz + cbase, tot);
        vsh = stage_window(s_v, d + cbase, tot);
        cp_async_commit();
        cp_async_wait<0>();
    } else {
        mbar_wait(&s_bar[1], 0);
    }
    __syncthreads();
    float* orow0 = p.out + out_off + r0 * KK;
    const bool vec_ok = VEC || (reinterpret_cast<uintptr_t>(orow0) & (KK * 4 - 1)) == 0;
    bool bad = false;
    // explicit 32-bit shared addresses (see lds_u32)
    const uint32_t a_or = (uint32_t)__cvta_generic_to_shared(s_or);
    const uint32_t a_c = (uint32_t)__cvta_generic_to_shared(s_c) + csh;
    const uint32_t a_v = (uint32_t)__cvta_generic_to_shared(s_v) + vsh;
    const uint32_t a_pk = (uint32_t)__cvta_generic_to_shared(s_pk);
    const uint32_t a_sel = (uint32_t)__cvta_generic_to_shared(s_sel);
    const uint32_t a_lut4 = (uint32_t)__cvta_generic_to_shared(s_lut4);
    const uint32_t a_lut = (uint32_t)__cvta_generic_to_shared(s_lut);
#pragma unroll 2
    for (uint32_t j = 0; j < PER; ++j) {
        const uint32_t li = j * SMALL8_THREADS + threadIdx.x;
        if (li >= nrow) break;
        const uint32_t e = lds_u32(a_or + 4 * li);  // offset | r << 16
        const uint32_t off = e & 0xFFFFu, r = e >> 16;
        const uint32_t cw = word_at(a_c + off);  // bytes past r are ignored
        const uint32_t vw = word_at(a_v + off);
        uint32_t mask, vs;
        const uint32_t live = __funnelshift_lc(0xFFFFFFFFu, 0u, 8 * r);  // low r bytes
        if constexpr (KK == 4) {
            // one table entry per row: the two low bits of the four column
            // bytes gathered by a multiply, (r, idx) -> selector, mask, valid;
            // a live column byte >= 4 is caught separately
            const uint32_t idx = ((cw & 0x03030303u) * 0x01041040u) >> 24;
            const uint32_t ent = lds_u32(a_lut4 + 4 * (r * 256 + idx));
            mask = (ent >> 16) & 0xFu;
            bad |= !((ent >> 20) & 1u) | ((cw & live & 0xFCFCFCFCu) != 0);  // sparse.py:90-97
            vs = __byte_perm(vw, 0u, ent & 0xFFFFu);
        } else {
            // column-presence mask of the row; a row is valid (sparse.py:90-97:
            // columns < K, strictly increasing) iff its live column bytes equal
            // the sorted packing of its mask and the mask has r bits
            mask = 0;
#pragma unroll
            for (int e = 0; e < KK; ++e) mask |= (uint32_t)((uint32_t)e < r) << ((cw >> (8 * e)) & (KK - 1));
            bad |= ((cw & live) != lds_u32(a_pk + 4 * mask)) | ((uint32_t)__popc(mask) != r);
            // value byte of every present column in column order (PRMT), 0 elsewhere
            vs = __byte_perm(vw, 0u, lds_u32(a_sel + 4 * mask));
        }
        float o[KK];
#pragma unroll
        for (int col = 0; col < KK; ++col) {
            const uint32_t sh = col == 0 ? (vs << 2) : (vs >> (8 * col - 2));
            const float val = __uint_as_float(lds_u32(a_lut | (sh & 0x3FCu)));
            o[col] = (mask >> col) & 1u ? val : 0.0f;
        }
        float* orow = orow0 + (uint64_t)li * KK;
        if constexpr (KK == 4) {
            if (vec_ok) __stcs(reinterpret_cast<float4*>(orow), make_float4(o[0], o[1], o[2], o[3]));
            else { orow[0] = o[0]; orow[1] = o[1]; orow[2] = o[2]; orow[3] = o[3]; }
        } else if constexpr (KK == 2) {
            if (vec_ok) __stcs(reinterpret_cast<float2*>(orow), make_float2(o[0], o[1]));
            else { orow[0] = o[0]; orow[1] = o[1]; }
        } else {
            __stcs(orow, o[0]);
        }
    }
    if (bad) s_bad = 1;
    __syncthreads();
    if (threadIdx.x == 0 && s_bad) p.status[b] = SCZ_CORRUPT_STREAM;
}
template __global__ void k_rows_small8<1, true>(RowParams);
template __global__ void k_rows_small8<2, true>(RowParams);
template __global__ void k_rows_small8<4, true>(RowParams);
template __global__ void k_rows_small8<1, true, true>(RowParams);
template __global__ void k_rows_small8<2, true, true>(RowParams);
template __global__ void k_rows_small8<4, true, true>(RowParams);
template __global__ void k_rows_small8<1, false>(RowParams);
template __global__ void k_rows_small8<2, false>(RowParams);
template __global__ void k_rows_small8<4, false>(RowParams);

#define SCZ_INST_SMALL(S)                                      \
    template __global__ void k_rows_small<S, 1>(RowParams);    \
    template __global__ void k_rows_small<S, 2>(RowParams);    \
    template __global__ void k_rows_small<S, 4>(RowParams);
SCZ_INST_SMALL(uint8_t)
SCZ_INST_SMALL(uint16_t)

#define SCZ_INST_ROWS(S)                                        \
    template __global__ void k_rows_out<S, false>(RowParams);   \
    template __global__ void k_rows_out<S, true>(RowParams);
SCZ_INST_ROWS(uint8_t)
SCZ_INST_ROWS(uint16_t)
SCZ_INST_ROWS(uint32_t)

// ------------------------------------------------------ stage-API helpers
// zero mask (u8) -> bitmap + per-tile nnz, for csr_encode.
__global__ void __launch_bounds__(TILE_THREADS) k_mask_bitmap(const uint8_t* mask, uint64_t n,
                                                              uint32_t* bitmap, uint32_t* tile_nnz) {
    pdl_wait();
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
    pdl_wait();
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
    pdl_wait();
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
    pdl_wait();
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) mask[i] = ((bitmap[i >> 5] >> (i & 31)) & 1u) ? 0 : 1;
}

__global__ void k_dequant_flat(const uint32_t* q, const uint8_t* mask, uint64_t n, double scale,
                               int64_t z, float* out) {
    pdl_wait();
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n)
        out[i] = mask[i] ? 0.0f
                         : __double2float_rn(__dmul_rn(__dsub_rn((double)q[i], (double)z), scale));
}

// bincount with AlphabetOverflow flag (rans.py:76-85)
__global__ void k_hist_u32(const uint32_t* d, uint64_t n, uint32_t A, uint32_t* counts,
                           int32_t* overflow) {
    pdl_wait();
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        uint32_t v = d[i];
        if (v >= A) *overflow = 1;
        else atomicAdd(counts + v, 1u);
    }
}

}  // namespace scz
