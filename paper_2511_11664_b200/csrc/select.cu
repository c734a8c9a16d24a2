// select.cu -- reshape search decision (Algorithm 1) and frequency tables.
//
//   k_select  grid (groups, B).  For every feasible candidate N (descending,
//             optimizer.py:72-75) it assembles the histogram of D = v ++ c ++ r
//             from the value histogram, the column histogram and the
//             row-count histogram (k_rowhist2), prices it as l_D * H (optimizer.py:87-96,
//             rans.py:216-223 with numpy's pairwise summation order), replays
//             the early-stopped scan (optimizer.py:129-138), then normalises
//             the chosen histogram (rans.py:88-131) and builds the encoder
//             table (freq, cum, exact reciprocal).
//   k_normalize_only  stage entry point for rans.normalize_frequencies.
#include "common.cuh"

namespace scz {

constexpr int SEL_THREADS = 256;

struct SelectParams {
    uint32_t n_cand;
    uint32_t cand_k[MAX_CAND];
    uint32_t cand_n[MAX_CAND];
    uint32_t rhist_off[MAX_CAND];
    const uint32_t* rhist;      // per candidate: K + 1 row bins, then K column bins
    uint32_t rhist_stride;
    const uint32_t* vhist;      // [B][256]
    int q_bits;
    int precision;
    int searching;              // 1: Algorithm 1; 0: single explicit candidate
    uint64_t total;
    TensorState* state;
    uint32_t* counts;           // scratch [B][acap]
    double* terms;              // scratch [B][acap]
    uint32_t acap;
    uint32_t* freqs;            // out [B][acap]
    uint32_t* cum;              // out [B][acap + 1]
    EncTab* enctab;             // out [B][acap]
    double* cand_out;           // optional out [B][MAX_CAND][2] (entropy, cost)
    uint32_t* dump;             // optional out [B][n_cand][acap] histogram of D per candidate
    // candidate pricing split over `groups` CTAs per tensor (small batches):
    // each publishes its costs, the last to arrive decides and normalises
    uint32_t groups;
    uint32_t* ticket;           // [B], zeroed before the launch
    double* gcost;              // [B][MAX_CAND][2] (entropy, cost)
    uint32_t* gacnt;            // [B][MAX_CAND] alphabet per candidate
    // SCZ_SELECT_PROBE=1: %globaltimer stamps per CTA (debug timeline)
    unsigned long long* probe;
    // Lazy search (pass 1 / 2; 0 = everything in one pass): pass 1 prices
    // candidates [0, c_end) and decides if the early-stopped scan stops among
    // them, else flags sel_pending; pass 2 (pending tensors only) prices
    // [c_begin, c_end) and replays the scan over all of them.  Every priced
    // (entropy, cost, alphabet) is kept in gcost / gacnt between the passes.
    uint32_t c_begin, c_end;
    int pass;
};
__device__ __forceinline__ unsigned long long sel_timer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SEL_PROBE(i)                                                                           \
    do {                                                                                       \
        if (p.probe && threadIdx.x == 0) p.probe[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + (i)] = sel_timer(); \
    } while (0)

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src
// pairwise_sum) of a[0..n): blocks of <= 128 with 8 accumulators, halves
// rounded down to a multiple of 8 above that.  One thread; the recursion is
// replayed with an explicit stack (depth <= 25 for n < 2^31), so no device
// call stack is needed.
__device__ __forceinline__ double pairwise_leaf(const double* a, uint32_t n) {
    if (n < 8) {
        double r = 0.0;
        for (uint32_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    uint32_t i;
    for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

__device__ __noinline__ double pairwise_sum(const double* a, uint32_t n) {
    uint32_t offs[26], lens[26];
    double lefts[26];
    uint32_t right = 0;  // bit d: the node at depth d is a right child
    int d = 0;
    offs[0] = 0;
    lens[0] = n;
    for (;;) {
        while (lens[d] > 128) {  // descend to the leftmost leaf
            uint32_t n2 = lens[d] / 2;
            n2 -= n2 % 8;
            offs[d + 1] = offs[d];
            lens[d + 1] = n2;
            right &= ~(1u << (d + 1));
            ++d;
        }
        double ret = pairwise_leaf(a + offs[d], lens[d]);
        for (;;) {  // ascend past finished right children
            if (d == 0) return ret;
            if ((right >> d) & 1u) {
                ret = __dadd_rn(lefts[d - 1], ret);
                --d;
            } else {  // left child done: visit its right sibling
                lefts[d - 1] = ret;
                offs[d] = offs[d - 1] + lens[d];
                lens[d] = lens[d - 1] - lens[d];
                right |= 1u << d;
                break;
            }
        }
    }
}

struct BlockScratch {
    uint32_t scan[33];
    uint32_t hist[256];
    unsigned long long red64[SEL_THREADS / 32];
    uint32_t red32[SEL_THREADS / 32];
    uint64_t bcast64[4];
    double costs[MAX_CAND];
    double ents[MAX_CAND];
    uint32_t alph[MAX_CAND];
    uint32_t acnt[MAX_CAND];        // alphabet of every priced candidate (warp path)
    unsigned long long keys[1024];  // remainder keys for the small-alphabet ranking
};

__device__ unsigned long long block_sum64(unsigned long long v, BlockScratch& s) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s.red64[warp] = v;
    __syncthreads();
    unsigned long long t = 0;
    for (int w = 0; w < SEL_THREADS / 32; ++w) t += s.red64[w];
    __syncthreads();
    return t;
}

__device__ uint32_t block_max32(uint32_t v, BlockScratch& s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s.red32[warp] = v;
    __syncthreads();
    uint32_t t = 0;
    for (int w = 0; w < SEL_THREADS / 32; ++w) t = max(t, s.red32[w]);
    __syncthreads();
    return t;
}

// rans.py:88-131 normalize_frequencies over counts[0..A) by one CTA.
// Returns an SCZ_* status (same for all threads).
// Code size matters here: k_select runs most of its code once per tensor, so
// instruction-cache misses, not arithmetic, set its latency.  The bulky
// helpers are out of line.
__device__ __noinline__ double plog2p(double pp) { return __dmul_rn(pp, log2(pp)); }

// Large alphabets (A > 1024): add 1 to the `k` largest remainders (ties to
// the lower index, np.lexsort) by an 8-pass radix select over the remainder
// bits.  Out of line: the common small-alphabet path stays contiguous code.
__device__ __noinline__ void deficit_radix(const double* rem, uint32_t A, unsigned long long k, uint32_t* freqs,
                                           BlockScratch& s) {
    unsigned long long prefix = 0, pmask = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += SEL_THREADS) s.hist[i] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < A; i += SEL_THREADS) {
            unsigned long long key = (unsigned long long)__double_as_longlong(rem[i]);
            if ((key & pmask) == prefix) atomicAdd(&s.hist[(key >> shift) & 255], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long acc = 0;
            int d = 255;
            for (; d > 0; --d) {
                if (acc + s.hist[d] >= k) break;
                acc += s.hist[d];
            }
            s.bcast64[0] = prefix | ((unsigned long long)d << shift);
            s.bcast64[1] = k - acc;
        }
        __syncthreads();
        prefix = s.bcast64[0];
        k = s.bcast64[1];
        pmask |= 0xFFull << shift;
        __syncthreads();
    }
    // take every key > prefix, and the first k keys == prefix by index
    uint32_t carry = 0;
    for (uint32_t base = 0; base < A; base += SEL_THREADS) {
        uint32_t i = base + threadIdx.x;
        unsigned long long key =
            i < A ? (unsigned long long)__double_as_longlong(rem[i]) : 0ull;
        uint32_t eq = (i < A && key == prefix) ? 1u : 0u;
        uint32_t tot;
        uint32_t ex = block_exclusive_scan<SEL_THREADS>(eq, s.scan, &tot);
        if (i < A) {
            if (key > prefix || (eq && carry + ex < k)) freqs[i] += 1;
        }
        carry += tot;
    }
}

__device__ __noinline__ int block_normalize(const uint32_t* counts, uint32_t A, int precision,
                               uint32_t* freqs, double* rem, uint32_t* cum, BlockScratch& s) {
    unsigned long long total = 0, npresent = 0;
    for (uint32_t i = threadIdx.x; i < A; i += SEL_THREADS) {
        total += counts[i];
        npresent += counts[i] > 0;
    }
    total = block_sum64(total, s);
    npresent = block_sum64(npresent, s);
    if (total == 0) return SCZ_NORMALIZE_ERROR;
    if (precision < 1 || precision > 16) return SCZ_INVALID_INPUT;
    const unsigned long long target = 1ull << precision;
    if (npresent > target) return SCZ_PRECISION_TOO_SMALL;
    const double ratio = __ddiv_rn((double)target, (double)total);
    unsigned long long sumf = 0;
    for (uint32_t i = threadIdx.x; i < A; i += SEL_THREADS) {
        double ideal = __dmul_rn((double)counts[i], ratio);
        double f = floor(ideal);
        freqs[i] = (uint32_t)f;
        rem[i] = __dsub_rn(ideal, f);
        sumf += (unsigned long long)f;
    }
    sumf = block_sum64(sumf, s);
    long long deficit = (long long)target - (long long)sumf;
    if (deficit > 0) {
        // np.lexsort((arange, -rem))[:deficit]: radix-select the deficit-th
        // largest remainder (non-negative doubles order as their bits), then
        // take ties in index order.
        unsigned long long k = (unsigned long long)deficit;
        if (k >= A) {
            for (uint32_t i = threadIdx.x; i < A; i += SEL_THREADS) freqs[i] += 1;
        } else if (A <= 1024) {
            // small alphabets: rank every symbol against all others in one pass
            // (keys padded with zeros to a multiple of 8: a zero pad never
            // outranks a real key, since pads sit at indices >= A)
            const uint32_t A8 = (A + 7) & ~7u;
            for (uint32_t i = threadIdx.x; i < A8; i += SEL_THREADS)
                s.keys[i] = i < A ? (unsigned long long)__double_as_longlong(rem[i]) : 0ull;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < A; i += SEL_THREADS) {
                const unsigned long long ki = s.keys[i];
                uint32_t r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (uint32_t j = 0; j < A8; j += 8) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const unsigned long long kj = s.keys[j + u];
                        r[u] += (kj > ki) | ((kj == ki) & (j + u < i));
                    }
                }
                const uint32_t rank = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
                if (rank < k) freqs[i] += 1;
            }
        } else {
            deficit_radix(rem, A, k, freqs, s);
        }
    }
    __syncthreads();
    unsigned long long sum2 = 0;
    for (uint32_t i = threadIdx.x; i < A; i += SEL_THREADS) {
        if (counts[i] > 0 && freqs[i] == 0) freqs[i] = 1;
        sum2 += freqs[i];
    }
    sum2 = block_sum64(sum2, s);
    long long surplus = (long long)sum2 - (long long)target;
    while (surplus > 0) {
        // argmax, first index on ties (np.argmax)
        unsigned long long best = 0;
        for (uint32_t i = threadIdx.x; i < A; i += SEL_THREADS) {
            unsigned long long key = ((unsigned long long)freqs[i] << 32) | (0xffffffffu - i);
            best = key > best ? key : best;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
            best = y > best ? y : best;
        }
        if ((threadIdx.x & 31) == 0) s.red64[threadIdx.x >> 5] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long bb = 0;
            for (int w = 0; w < SEL_THREADS / 32; ++w) bb = s.red64[w] > bb ? s.red64[w] : bb;
            s.bcast64[2] = bb;
        }
        __syncthreads();
        unsigned long long bb = s.bcast64[2];
        __syncthreads();
        uint32_t idx = 0xffffffffu - (uint32_t)(bb & 0xffffffffu);
        long long room = (long long)(bb >> 32) - 1;
        long long cut = room < surplus ? room : surplus;
        if (cut <= 0) return SCZ_PRECISION_TOO_SMALL;
        if (threadIdx.x == 0) freqs[idx] -= (uint32_t)cut;
        surplus -= cut;
        __syncthreads();
    }
    // cdf (rans.py:130)
    if (cum) {
        uint32_t carry = 0;
        for (uint32_t base = 0; base < A; base += SEL_THREADS) {
            uint32_t i = base + threadIdx.x;
            uint32_t v = i < A ? freqs[i] : 0;
            uint32_t tot;
            uint32_t ex = block_exclusive_scan<SEL_THREADS>(v, s.scan, &tot);
            if (i < A) cum[i] = carry + ex;
            carry += tot;
        }
        if (threadIdx.x == 0) cum[A] = carry;
    }
    __syncthreads();
    return SCZ_OK;
}

// Histogram of D for candidate c into counts[0..acap); returns alphabet.
__device__ __noinline__ uint32_t assemble_counts(const SelectParams& p, uint32_t b, uint32_t c,
                                    uint32_t* counts, BlockScratch& s) {
    const TensorState& st = p.state[b];
    const uint32_t K = p.cand_k[c], N = p.cand_n[c];
    const uint64_t nnz = st.nnz;
    const uint32_t nv = 1u << p.q_bits;
    const uint32_t ubound = max(nv, K + 1);
    const uint32_t* vh = p.vhist + (uint64_t)b * 256;
    const uint32_t* rh = p.rhist + (uint64_t)b * p.rhist_stride + p.rhist_off[c];
    // rows with r = 0: N minus the rows counted in bins 1..K (k_rowhist2 skips 0)
    unsigned long long rsum = 0;
    if (K > 1)
        for (uint32_t i = 1 + threadIdx.x; i <= K; i += SEL_THREADS) rsum += rh[i];
    rsum = block_sum64(rsum, s);
    for (uint32_t i = threadIdx.x; i < ubound; i += SEL_THREADS) {
        uint32_t v = (i < nv) ? vh[i] : 0;
        if (K == 1) {
            if (i == 0) v += (uint32_t)(N - nnz) + (uint32_t)nnz;  // c = 0 for all, r = 0 rows
            if (i == 1) v += (uint32_t)nnz;                      // r = 1 rows
        } else if (i == 0) {
            v += N - (uint32_t)rsum;
        } else if (i <= K) {
            v += rh[i];
        }
        counts[i] = v;
    }
    __syncthreads();
    if (K > 1) {  // column histogram (folded by k_rowhist2 after the row bins)
        for (uint32_t col = threadIdx.x; col < K; col += SEL_THREADS) counts[col] += rh[K + 1 + col];
    }
    __syncthreads();
    uint32_t last = 0;
    for (uint32_t i = threadIdx.x; i < ubound; i += SEL_THREADS)
        if (counts[i]) last = i + 1;
    return block_max32(last, s);
}

// -(p log2 p).sum() over the positive counts, in numpy's order (rans.py:219-223).
__device__ __noinline__ double block_entropy(const uint32_t* counts, uint32_t A, double total, double* terms,
                                BlockScratch& s) {
    uint32_t carry = 0;
    for (uint32_t base = 0; base < A; base += SEL_THREADS) {
        uint32_t i = base + threadIdx.x;
        uint32_t c = i < A ? counts[i] : 0;
        uint32_t tot;
        uint32_t ex = block_exclusive_scan<SEL_THREADS>(c > 0 ? 1u : 0u, s.scan, &tot);
        if (c > 0) {
            double pp = __ddiv_rn((double)c, total);
            terms[carry + ex] = plog2p(pp);
        }
        carry += tot;
    }
    __syncthreads();
    __shared__ double s_h;
    if (threadIdx.x == 0) s_h = -pairwise_sum(terms, carry);
    __syncthreads();
    return s_h;
}

// Candidate pricing with one warp per candidate (search path, A <= 1024):
// dynamic smem = [vhist][row + column histograms if they fit]
//                [per warp: terms f64[acap], counts u32[acap]],
// the histograms staged with one batch of cp.async copies.
constexpr uint32_t SEL_WARP_ACAP = 1024;
constexpr uint32_t SEL_RH_SMEM_MAX = 16384;  // histogram words staged in smem (64 KB)

__host__ __device__ inline size_t select_smem_bytes(uint32_t acap, uint32_t rh_stride) {
    if (acap > SEL_WARP_ACAP) return 0;
    size_t s = (size_t)(SEL_THREADS / 32) * acap * (4 + 8) + 256 * 4;
    if (rh_stride <= SEL_RH_SMEM_MAX) s += ((size_t)rh_stride * 4 + 15) & ~(size_t)15;
    return (s + 15) & ~(size_t)15;
}

// Returns the start of the per-warp scratch (reused by the final normalise).
__device__ uint8_t* warp_parallel_costs(const SelectParams& p, uint32_t b, uint32_t g, BlockScratch& s) {
    extern __shared__ __align__(16) uint8_t sel_dyn[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const TensorState& st = p.state[b];
    const uint64_t nnz = st.nnz;
    const uint32_t* grh = p.rhist + (uint64_t)b * p.rhist_stride;
    const uint32_t* gvh = p.vhist + (uint64_t)b * 256;
    const bool rh_smem = p.rhist_stride <= SEL_RH_SMEM_MAX;
    uint8_t* dyn = sel_dyn;
    uint32_t* s_vh = reinterpret_cast<uint32_t*>(dyn);
    if (threadIdx.x < 64) cp_async16(s_vh + 4 * threadIdx.x, gvh + 4 * threadIdx.x);
    dyn += 256 * 4;
    uint32_t* s_rh = reinterpret_cast<uint32_t*>(dyn);
    if (rh_smem) {
        for (uint32_t i = threadIdx.x; i < p.rhist_stride; i += SEL_THREADS) cp_async4(s_rh + i, grh + i);
        dyn += ((size_t)p.rhist_stride * 4 + 15) & ~(size_t)15;
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    SEL_PROBE(1);
    const uint32_t* rhb = rh_smem ? s_rh : grh;
    double* terms = reinterpret_cast<double*>(dyn) + (size_t)warp * p.acap;
    uint32_t* cb = reinterpret_cast<uint32_t*>(dyn + (size_t)(SEL_THREADS / 32) * p.acap * 8) +
                   (size_t)warp * p.acap;
    const uint32_t nv = 1u << p.q_bits;
    const uint32_t* vh = s_vh;
    constexpr uint32_t NW = SEL_THREADS / 32;
    const bool keep = p.groups > 1 || p.pass != 0;  // costs go to gcost for another CTA / pass
    for (uint32_t c = p.c_begin + g * NW + warp; c < p.c_end; c += NW * p.groups) {
        const uint32_t K = p.cand_k[c], N = p.cand_n[c];
        const uint32_t ub = max(nv, K + 1);
        const uint32_t* rh = rhb + p.rhist_off[c];
        uint32_t rsum = 0;  // rows with r >= 1 (bin 0 is N - rsum)
        if (K > 1)
            for (uint32_t i = 1 + lane; i <= K; i += 32) rsum += rh[i];
        rsum = warp_sum(rsum);
        for (uint32_t i = lane; i < ub; i += 32) {
            uint32_t v = (i < nv) ? vh[i] : 0;
            if (K == 1) {
                if (i == 0) v += N;             // nnz column-0 entries + (N - nnz) empty rows
                if (i == 1) v += (uint32_t)nnz;  // full rows
            } else if (i == 0) {
                v += N - rsum;
            } else if (i <= K) {
                v += rh[i];
            }
            cb[i] = v;
        }
        __syncwarp();
        if (K > 1)  // column histogram (folded by k_rowhist2 after the row bins)
            for (uint32_t col = lane; col < K; col += 32) cb[col] += rh[K + 1 + col];
        __syncwarp();
        uint32_t last = 0;
        for (uint32_t i = lane; i < ub; i += 32)
            if (cb[i]) last = i + 1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
        const uint32_t A = last;
        if (p.dump) {  // kept for the chosen candidate's table (and scz_search)
            uint32_t* dd = p.dump + ((uint64_t)b * p.n_cand + c) * p.acap;
            for (uint32_t i = lane; i < p.acap; i += 32) dd[i] = i < A ? cb[i] : 0;
        }
        if (lane == 0) {
            s.acnt[c] = A;
            if (keep) p.gacnt[(uint64_t)b * MAX_CAND + c] = A;
        }
        // entropy over the positive counts in index order (rans.py:219-223)
        const uint64_t len = 2 * nnz + N;
        const double total = (double)len;
        // one division + logarithm per lane per 32 symbols; kept compact
        // (not unrolled, log2 out of line): at small batches this kernel runs
        // once per tensor and instruction-cache misses, not arithmetic, set
        // its latency
        uint32_t m = 0;
#pragma unroll 1
        for (uint32_t i0 = 0; i0 < A; i0 += 32) {
            const uint32_t i = i0 + lane;
            const uint32_t cnt = i < A ? cb[i] : 0;
            const uint32_t bal = __ballot_sync(0xffffffffu, cnt > 0);
            const uint32_t pos = m + __popc(bal & lanemask_lt());
            m += __popc(bal);
            if (cnt > 0) terms[pos] = plog2p(__ddiv_rn((double)cnt, total));
        }
        __syncwarp();
        if (lane == 0) {
            const double h = -pairwise_sum(terms, m);
            s.ents[c] = h;
            s.costs[c] = __dmul_rn((double)len, h);
            if (keep) {
                double* gc = p.gcost + ((uint64_t)b * MAX_CAND + c) * 2;
                gc[0] = h;
                gc[1] = s.costs[c];
            }
        }
        __syncwarp();
    }
    __syncthreads();
    SEL_PROBE(2);
    return dyn;
}

// Multi-CTA pricing: true in the CTA that arrives last for tensor b, which
// then holds every candidate's (entropy, cost, alphabet) in `s`.
__device__ bool gather_costs(const SelectParams& p, uint32_t b, BlockScratch& s) {
    if (p.groups > 1) {
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            s.alph[3] = atomicAdd(p.ticket + b, 1u) == p.groups - 1;
            if (s.alph[3]) p.ticket[b] = 0;  // re-armed for the next pass
        }
        __syncthreads();
        if (!s.alph[3]) return false;
        __threadfence();
    }
    // from gcost: this pass's candidates when several CTAs priced them, and
    // in pass 2 the first pass's candidates
    const uint32_t lo = p.pass == 2 ? 0 : p.c_begin;
    const uint32_t hi = p.groups > 1 ? p.c_end : (p.pass == 2 ? p.c_begin : 0);
    for (uint32_t c = lo + threadIdx.x; c < hi; c += SEL_THREADS) {
        const volatile double* gc = p.gcost + ((uint64_t)b * MAX_CAND + c) * 2;
        s.ents[c] = gc[0];
        s.costs[c] = gc[1];
        s.acnt[c] = *(const volatile uint32_t*)(p.gacnt + (uint64_t)b * MAX_CAND + c);
    }
    __syncthreads();
    return true;
}

__global__ void __launch_bounds__(SEL_THREADS) k_select(const __grid_constant__ SelectParams p) {
    pdl_wait();
    const uint32_t b = blockIdx.y, g = blockIdx.x;
    SEL_PROBE(0);
    TensorState& st = p.state[b];
    if (st.status != SCZ_OK) return;
    if (p.pass == 2 && !st.sel_pending) return;  // decided by the first pass
    __shared__ BlockScratch s;
    uint32_t* counts = p.counts + (uint64_t)b * p.acap;
    double* terms = p.terms + (uint64_t)b * p.acap;
    const uint64_t nnz = st.nnz;

    uint32_t chosen = 0, flags = 0, evaluated = 0;
    uint8_t* work = nullptr;  // shared scratch for the final normalise (warp path)
    if (p.searching) {
        if (p.acap <= SEL_WARP_ACAP) {
            work = warp_parallel_costs(p, b, g, s);
            if (!gather_costs(p, b, s)) return;
            SEL_PROBE(3);
        } else for (uint32_t c = 0; c < p.n_cand; ++c) {
            uint32_t A = assemble_counts(p, b, c, counts, s);
            if (p.dump) {
                uint32_t* dd = p.dump + ((uint64_t)b * p.n_cand + c) * p.acap;
                for (uint32_t i = threadIdx.x; i < p.acap; i += SEL_THREADS) dd[i] = i < A ? counts[i] : 0;
            }
            uint64_t len = 2 * nnz + p.cand_n[c];
            double h = block_entropy(counts, A, (double)len, terms, s);
            if (threadIdx.x == 0) {
                s.ents[c] = h;
                s.costs[c] = __dmul_rn((double)len, h);
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            // optimizer.py:116-138 replay; flag decisions that a 1e-12
            // relative perturbation of either cost could flip.
            double best = INFINITY, prev = INFINITY;
            bool stopped = false;
            auto near = [](double a, double bb) {
                if (isinf(a) || isinf(bb)) return false;
                if (a == 0.0 && bb == 0.0) return false;
                return fabs(a - bb) <= 1e-12 * fmax(fabs(a), fabs(bb));
            };
            for (uint32_t c = 0; c < p.c_end; ++c) {
                double v = s.costs[c];
                ++evaluated;
                if (near(v, best) || near(v, prev)) flags |= SCZ_SEARCH_NEAR_TIE;
                if (v < best) {
                    best = v;
                    chosen = c;
                }
                if (v > prev) {
                    stopped = true;
                    break;
                }
                prev = v;
            }
            if (stopped) flags |= SCZ_SEARCH_EARLY_STOPPED;
            flags |= SCZ_SEARCH_USED;
            // first pass that did not stop among its candidates: price the rest
            s.alph[4] = (p.pass == 1 && !stopped && p.c_end < p.n_cand) ? 1u : 0u;
            if (p.pass == 1) st.sel_pending = s.alph[4];
            if (p.cand_out) {
                double* co = p.cand_out + (uint64_t)b * MAX_CAND * 2;
                for (uint32_t c = 0; c < p.n_cand; ++c) {
                    co[2 * c] = s.ents[c];
                    co[2 * c + 1] = s.costs[c];
                }
            }
            s.alph[0] = chosen;
            s.alph[1] = flags;
            s.alph[2] = evaluated;
        }
        __syncthreads();
        chosen = s.alph[0];
        flags = s.alph[1];
        evaluated = s.alph[2];
        const bool pending = s.alph[4] != 0;
        __syncthreads();
        if (pending) return;  // pass 2 decides
    }
    // chosen candidate: histogram -> normalised table -> encoder table
    uint32_t A;
    const uint32_t* ccounts = counts;
    if (p.searching && p.acap <= SEL_WARP_ACAP && p.dump) {  // already assembled by its warp
        A = s.acnt[chosen];
        ccounts = p.dump + ((uint64_t)b * p.n_cand + chosen) * p.acap;
    } else {
        A = assemble_counts(p, b, chosen, counts, s);
    }
    uint32_t* gfreqs = p.freqs + (uint64_t)b * p.acap;
    uint32_t* gcum = p.cum + (uint64_t)b * (p.acap + 1);
    uint32_t* freqs = gfreqs;
    uint32_t* cum = gcum;
    double* rem = terms;
    if (work) {  // normalise in shared memory (per-warp scratch >= 20 bytes per symbol)
        rem = reinterpret_cast<double*>(work);
        uint32_t* scnt = reinterpret_cast<uint32_t*>(rem + p.acap);
        freqs = scnt + p.acap;
        cum = freqs + p.acap;
        for (uint32_t i = threadIdx.x; i < A; i += SEL_THREADS) scnt[i] = ccounts[i];
        __syncthreads();
        ccounts = scnt;
    }
    SEL_PROBE(4);
    int status = block_normalize(ccounts, A, p.precision, freqs, rem, cum, s);
    SEL_PROBE(5);
    EncTab* et = p.enctab + (uint64_t)b * p.acap;
    if (status == SCZ_OK)
        for (uint32_t i = threadIdx.x; i < A; i += SEL_THREADS) {
            make_enc_tab(freqs[i], cum[i], &et[i]);
            if (work) {
                gfreqs[i] = freqs[i];
                gcum[i] = cum[i];
            }
        }
    if (work && status == SCZ_OK && threadIdx.x == 0) gcum[A] = cum[A];
    if (threadIdx.x == 0) {
        st.status = status;
        st.cand_index = chosen;
        st.n_rows = p.cand_n[chosen];
        st.n_cols = p.cand_k[chosen];
        st.alphabet = A;
        st.stream_len = 2 * nnz + p.cand_n[chosen];
        const uint32_t K = p.cand_k[chosen];
        st.sym_bytes = K <= 255 ? 1u : (K <= 65535 ? 2u : 4u);
        st.search_flags = flags;
        st.n_evaluated = evaluated;
        SEL_PROBE(6);
    }
}

// Stage entry point: normalize_frequencies of an arbitrary count vector.
__global__ void __launch_bounds__(SEL_THREADS) k_normalize_only(const uint32_t* counts, uint32_t A,
                                                               int precision, uint32_t* freqs,
                                                               double* rem, int32_t* status) {
    pdl_wait();
    __shared__ BlockScratch s;
    int st = block_normalize(counts, A, precision, freqs, rem, nullptr, s);
    if (threadIdx.x == 0) *status = st;
}

}  // namespace scz
