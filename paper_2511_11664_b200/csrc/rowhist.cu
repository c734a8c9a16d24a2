// rowhist.cu -- row-count histograms of every reshape candidate (Algorithm 1
// pricing, optimizer.py:87-96: the r segment of D for each N).
//
// For candidate K the rows are the K-bit fields of the zero bitmap; r_i is
// their popcount and the search needs hist(r).  Three regimes:
//   K in {2, 4, 8}  rows are aligned sub-word fields: SWAR field popcounts,
//                   per-value field counts with popc / __vcmpeq4, register
//                   counters (no shared-memory traffic per row);
//   K < 64          funnel-shift extraction, per-lane private u16 counters in
//                   shared memory (no atomics, no bank conflicts);
//   K >= 64         few rows: shared-memory atomics aggregated by match_any.
// Value 0 is never counted per row: it is N - sum(others), so bitmap padding
// beyond T never matters.
//
// The grid also carries one fold CTA per candidate: the column histogram of
// candidate K (nonzeros per p mod K) is H_P folded onto K columns (K | P),
// stored after the candidate's K + 1 row bins, so k_select never touches H_P.
#include "common.cuh"

namespace scz {

constexpr int RH_THREADS = 256;
constexpr int RH_PRIV_BINS = 64;  // K + 1 <= 64 uses lane-private counters
constexpr size_t RH_PRIV_SMEM = (size_t)(RH_THREADS / 32) * RH_PRIV_BINS * 32 * sizeof(uint16_t);

struct RowHist2Params {
    const uint32_t* bitmap;
    uint32_t words_pad;
    uint32_t n_words;                  // ceil(T / 32)
    uint32_t n_cand;
    uint32_t cand_k[MAX_CAND];
    uint32_t cand_rows[MAX_CAND];
    uint32_t chunk_start[MAX_CAND + 1];
    uint32_t units_per_chunk[MAX_CAND];  // words (SWAR) or rows (other regimes)
    uint32_t rhist_off[MAX_CAND];
    uint32_t* rhist;                   // [B][rhist_stride]: per candidate K + 1 row bins, K column bins
    uint32_t rhist_stride;
    const uint32_t* hp;                // [B][hp_stride] nonzeros per (p mod P)
    uint32_t hp_stride, period;
    uint32_t n_fold;                   // CTAs [0, n_fold): column fold of candidate blockIdx.x (first in the
                                       // grid: they are the longest CTAs and start right away)
    const TensorState* state;          // pending_only: skip tensors whose search already stopped
    int pending_only;
    uint32_t n_tensors;                // pending_only: tensor b = blockIdx.y, + gridDim.y, ...
};

__device__ void fold_columns(const RowHist2Params& p, uint32_t b, uint32_t c) {
    const uint32_t K = p.cand_k[c], P = p.period;
    if (K <= 1) return;
    const uint32_t* hp = p.hp + (uint64_t)b * p.hp_stride;
    uint32_t* ch = p.rhist + (uint64_t)b * p.rhist_stride + p.rhist_off[c] + K + 1;
    auto fold = [&](uint32_t j, uint32_t stride) -> uint32_t {
        uint32_t a[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // independent load chains
        for (; j + 7 * stride < P; j += 8 * stride) {
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] += __ldg(hp + j + u * stride);
        }
        for (; j < P; j += stride) a[0] += __ldg(hp + j);
        return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    };
    if (K <= RH_THREADS) {
        extern __shared__ uint32_t s_dyn[];
        for (uint32_t i = threadIdx.x; i < K; i += RH_THREADS) s_dyn[i] = 0;
        __syncthreads();
        const uint32_t L = K * (RH_THREADS / K);
        if (threadIdx.x < L) {
            const uint32_t acc = fold(threadIdx.x, L);
            if (acc) atomicAdd(&s_dyn[threadIdx.x % K], acc);
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < K; i += RH_THREADS) ch[i] = s_dyn[i];
    } else {
        for (uint32_t col = threadIdx.x; col < K; col += RH_THREADS) ch[col] = fold(col, K);
    }
}

template <int K>
__device__ __forceinline__ void swar_counts(uint32_t w, uint32_t* c) {
    uint32_t x = w - ((w >> 1) & 0x55555555u);  // 2-bit field counts
    if constexpr (K == 2) {
        c[2] += __popc(x & 0xAAAAAAAAu);
        c[1] += __popc(x & 0x55555555u);
        return;
    }
    x = (x & 0x33333333u) + ((x >> 2) & 0x33333333u);  // 4-bit field counts (0..4)
    if constexpr (K == 4) {
#pragma unroll
        for (uint32_t v = 1; v <= 4; ++v) {
            const uint32_t y = x ^ (v * 0x11111111u);
            const uint32_t nz = (y | (y >> 1) | (y >> 2)) & 0x11111111u;
            c[v] += 8 - __popc(nz);
        }
        return;
    }
    x = (x + (x >> 4)) & 0x0F0F0F0Fu;  // byte counts (0..8)
#pragma unroll
    for (uint32_t v = 1; v <= 8; ++v) c[v] += __popc(__vcmpeq4(x, v * 0x01010101u)) >> 3;
}

template <int K>
__device__ void rowhist_swar(const uint32_t* bm, uint32_t w0, uint32_t w1, uint32_t* gh) {
    uint32_t c[K + 1];
#pragma unroll
    for (int v = 0; v <= K; ++v) c[v] = 0;
    // four loads in flight per thread (the bitmap is L2-resident: latency-bound)
    uint32_t w = w0 + threadIdx.x;
    for (; w + 3 * RH_THREADS < w1; w += 4 * RH_THREADS) {
        uint32_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(bm + w + u * RH_THREADS);
#pragma unroll
        for (int u = 0; u < 4; ++u) swar_counts<K>(v[u], c);
    }
    for (; w < w1; w += RH_THREADS) swar_counts<K>(__ldg(bm + w), c);
    __shared__ uint32_t s_c[9];
    if (threadIdx.x <= K) s_c[threadIdx.x] = 0;
    __syncthreads();
#pragma unroll
    for (int v = 1; v <= K; ++v) {
        const uint32_t t = warp_sum(c[v]);
        if ((threadIdx.x & 31) == 0 && t) atomicAdd(&s_c[v], t);
    }
    __syncthreads();
    if (threadIdx.x >= 1 && threadIdx.x <= K && s_c[threadIdx.x]) atomicAdd(gh + threadIdx.x, s_c[threadIdx.x]);
}

__device__ __forceinline__ void rowhist2_tensor(const RowHist2Params& p, uint32_t b) {
    if (blockIdx.x < p.n_fold) {
        fold_columns(p, b, blockIdx.x);
        return;
    }
    const uint32_t chunk = blockIdx.x - p.n_fold;
    uint32_t c = 0;
    while (c + 1 < p.n_cand && p.chunk_start[c + 1] <= chunk) ++c;
    const uint32_t K = p.cand_k[c], N = p.cand_rows[c];
    const uint32_t* bm = p.bitmap + (uint64_t)b * p.words_pad;
    uint32_t* gh = p.rhist + (uint64_t)b * p.rhist_stride + p.rhist_off[c];
    const uint32_t u0 = (chunk - p.chunk_start[c]) * p.units_per_chunk[c];
    if (K == 2 || K == 4 || K == 8) {
        const uint32_t w1 = min(p.n_words, u0 + p.units_per_chunk[c]);
        if (K == 2) rowhist_swar<2>(bm, u0, w1, gh);
        else if (K == 4) rowhist_swar<4>(bm, u0, w1, gh);
        else rowhist_swar<8>(bm, u0, w1, gh);
        return;
    }
    const uint32_t r1 = min(N, u0 + p.units_per_chunk[c]);
    if (K + 1 <= RH_PRIV_BINS) {
        // lane-private u16 counters: s_h[warp][bin][lane] (dynamic smem)
        extern __shared__ uint32_t s_dyn[];
        auto s_h = reinterpret_cast<uint16_t(*)[RH_PRIV_BINS][32]>(s_dyn);
        const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (uint32_t v = 0; v <= K; ++v) s_h[warp][v][lane] = 0;
        const uint32_t kmask = K >= 32 ? 0xffffffffu : ((1u << K) - 1u);
        uint32_t r = u0 + threadIdx.x;
        if (K <= 32) {  // four rows (eight loads) in flight per thread
            for (; r + 3 * RH_THREADS < r1; r += 4 * RH_THREADS) {
                uint32_t lo[4], hi[4], sh[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t start = (r + u * RH_THREADS) * K;  // < 2^32: T < 2^31
                    sh[u] = start & 31;
                    lo[u] = __ldg(bm + (start >> 5));
                    hi[u] = __ldg(bm + (start >> 5) + 1);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) s_h[warp][__popc(__funnelshift_r(lo[u], hi[u], sh[u]) & kmask)][lane] += 1;
            }
        }
        for (; r < r1; r += RH_THREADS) {
            const uint64_t start = (uint64_t)r * K;
            const uint32_t w = (uint32_t)(start >> 5), s = (uint32_t)(start & 31);
            uint32_t v;
            if (K <= 32) {
                const uint32_t lo = __ldg(bm + w), hi = __ldg(bm + w + 1);
                v = __popc(__funnelshift_r(lo, hi, s) & kmask);
            } else {
                const uint32_t lo = __ldg(bm + w), mid = __ldg(bm + w + 1), hi = __ldg(bm + w + 2);
                const uint32_t first = __funnelshift_r(lo, mid, s);
                const uint32_t second = __funnelshift_r(mid, hi, s) & ((1u << (K - 32)) - 1u);
                v = __popc(first) + __popc(second);
            }
            s_h[warp][v][lane] += 1;
        }
        __syncthreads();
        // warp `warp` reduces bins warp, warp + 8, ...: lane l sums the 8 warp
        // copies of its column, then a warp sum (no serial per-bin loops)
        for (uint32_t v = 1 + warp; v <= K; v += RH_THREADS / 32) {
            uint32_t t = 0;
#pragma unroll
            for (int wv = 0; wv < RH_THREADS / 32; ++wv) t += s_h[wv][v][lane];
            t = warp_sum(t);
            if (lane == 0 && t) atomicAdd(gh + v, t);
        }
        return;
    }
    // large K: few rows, aggregated shared-memory atomics
    extern __shared__ uint32_t s_big[];  // same dynamic buffer as s_h
    const bool use_smem = K + 1 <= 4096;
    if (use_smem)
        for (uint32_t i = threadIdx.x; i <= K; i += RH_THREADS) s_big[i] = 0;
    __syncthreads();
    for (uint32_t r = u0 + threadIdx.x; r < u0 + ((r1 - u0 + 31) & ~31u); r += RH_THREADS) {
        const bool live = r < r1;
        uint32_t v = 0xffffffffu;
        if (live) {
            const uint64_t start = (uint64_t)r * K, end = start + K;
            const uint64_t w0 = start >> 5, wl = (end - 1) >> 5;
            const uint32_t s = (uint32_t)(start & 31), e = (uint32_t)(end & 31);
            uint32_t cnt = __popc(__ldg(bm + w0) >> s);
            for (uint64_t w = w0 + 1; w < wl; ++w) cnt += __popc(__ldg(bm + w));
            const uint32_t last = __ldg(bm + wl);
            cnt += __popc(e ? (last & ((1u << e) - 1u)) : last);
            v = cnt;
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, v);
        if (live && v && (threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) {
            if (use_smem) atomicAdd(&s_big[v], (uint32_t)__popc(peers));
            else atomicAdd(gh + v, (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    if (use_smem)
        for (uint32_t i = 1 + threadIdx.x; i <= K; i += RH_THREADS)
            if (s_big[i]) atomicAdd(gh + i, s_big[i]);
}

// First pass: one tensor per blockIdx.y.  Lazy second pass (pending tensors
// only, usually none): a short grid striding over the batch, so a batch
// whose scans all stopped costs a wave of CTAs that exit, not B x chunks.
__global__ void __launch_bounds__(RH_THREADS) k_rowhist2(const __grid_constant__ RowHist2Params p) {
    pdl_wait();
    if (!p.pending_only) {
        rowhist2_tensor(p, blockIdx.y);
        return;
    }
    for (uint32_t b = blockIdx.y; b < p.n_tensors; b += gridDim.y) {
        if (!p.state[b].sel_pending) continue;  // uniform per CTA
        rowhist2_tensor(p, b);
        __syncthreads();  // shared scratch reused by the next tensor
    }
}

}  // namespace scz
