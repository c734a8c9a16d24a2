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

constexpr int SEL_THREADS = 256;        // batches: one CTA (or a few) per tensor
constexpr int SEL_THREADS_WIDE = 1024;  // small batches: the whole decision of a tensor on one SM

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
    uint32_t nb;                // candidate slots per round of the cost pass (select_smem_bytes)
};
__device__ __forceinline__ unsigned long long sel_timer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SEL_PROBE(i)                                                                           \
    do {                                                                                       \
        if (p.probe && p.pass != 2 && threadIdx.x == 0)                                        \
            p.probe[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + (i)] = sel_timer();            \
    } while (0)
// inside helpers: a raw slot pointer (nullptr: off)
#define SEL_PROBE_AT(prb, i)                                \
    do {                                                    \
        if ((prb) && threadIdx.x == 0) (prb)[(i)] = sel_timer(); \
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

template <int NT>
struct BlockScratch {
    uint32_t scan[33];
    uint32_t hist[256];
    unsigned long long red64[NT / 32];
    uint32_t red32[NT / 32];
    uint32_t mk[32];                // cost pass: positive counts per candidate slot
    uint32_t moff[33];              // and their prefix (flat term index)
    double leafsum[NT / 32][8];     // pairwise-sum leaves per warp
    uint64_t bcast64[4];
    double costs[MAX_CAND];
    double ents[MAX_CAND];
    uint32_t alph[MAX_CAND];
    uint32_t acnt[MAX_CAND];        // alphabet of every priced candidate (warp path)
    unsigned long long keys[1024];  // remainder keys for the small-alphabet ranking
};

template <int NT>
__device__ unsigned long long block_sum64(unsigned long long v, BlockScratch<NT>& s) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s.red64[warp] = v;
    __syncthreads();
    // every warp folds the per-warp sums with shuffles (one load per lane,
    // not NT / 32 dependent loads per thread)
    unsigned long long t = lane < NT / 32 ? s.red64[lane] : 0ull;
    t = warp_sum(t);
    __syncthreads();
    return t;
}

template <int NT>
__device__ uint32_t block_max32(uint32_t v, BlockScratch<NT>& s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s.red32[warp] = v;
    __syncthreads();
    uint32_t t = lane < NT / 32 ? s.red32[lane] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = max(t, __shfl_xor_sync(0xffffffffu, t, o));
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
template <int NT>
__device__ __noinline__ void deficit_radix(const double* rem, uint32_t A, unsigned long long k, uint32_t* freqs,
                                           BlockScratch<NT>& s) {
    unsigned long long prefix = 0, pmask = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += NT) s.hist[i] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < A; i += NT) {
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
    for (uint32_t base = 0; base < A; base += NT) {
        uint32_t i = base + threadIdx.x;
        unsigned long long key =
            i < A ? (unsigned long long)__double_as_longlong(rem[i]) : 0ull;
        uint32_t eq = (i < A && key == prefix) ? 1u : 0u;
        uint32_t tot;
        uint32_t ex = block_exclusive_scan<NT>(eq, s.scan, &tot);
        if (i < A) {
            if (key > prefix || (eq && carry + ex < k)) freqs[i] += 1;
        }
        carry += tot;
    }
}

template <int NT>
__device__ __noinline__ int block_normalize(const uint32_t* counts, uint32_t A, int precision,
                               uint32_t* freqs, double* rem, uint32_t* cum, BlockScratch<NT>& s,
                               unsigned long long* prb = nullptr) {
    unsigned long long total = 0, npresent = 0;
    for (uint32_t i = threadIdx.x; i < A; i += NT) {
        total += counts[i];
        npresent += counts[i] > 0;
    }
    if (A < (1u << 12)) {  // one reduction: counts < 2^32, so total < 2^44 and npresent < 2^12
        const unsigned long long both = block_sum64((total << 20) | npresent, s);
        total = both >> 20;
        npresent = both & ((1ull << 20) - 1);
    } else {
        total = block_sum64(total, s);
        npresent = block_sum64(npresent, s);
    }
    if (total == 0) return SCZ_NORMALIZE_ERROR;
    if (precision < 1 || precision > 16) return SCZ_INVALID_INPUT;
    const unsigned long long target = 1ull << precision;
    if (npresent > target) return SCZ_PRECISION_TOO_SMALL;
    SEL_PROBE_AT(prb, 7);
    const double ratio = __ddiv_rn((double)target, (double)total);
    unsigned long long sumf = 0;
    for (uint32_t i = threadIdx.x; i < A; i += NT) {
        double ideal = __dmul_rn((double)counts[i], ratio);
        double f = floor(ideal);
        freqs[i] = (uint32_t)f;
        rem[i] = __dsub_rn(ideal, f);
        sumf += (unsigned long long)f;
    }
    sumf = block_sum64(sumf, s);
    SEL_PROBE_AT(prb, 8);
    long long deficit = (long long)target - (long long)sumf;
    if (deficit > 0) {
        // np.lexsort((arange, -rem))[:deficit]: radix-select the deficit-th
        // largest remainder (non-negative doubles order as their bits), then
        // take ties in index order.
        unsigned long long k = (unsigned long long)deficit;
        if (k >= A) {
            for (uint32_t i = threadIdx.x; i < A; i += NT) freqs[i] += 1;
        } else if (A <= 1024) {
            // small alphabets: rank every symbol against all others in one pass.
            // P threads per symbol (the largest power of two <= 8 with
            // A * P <= NT; neighbouring lanes) split the others by j mod P,
            // then add their partial ranks with shuffles.  Keys are padded
            // with zeros to a multiple of 8P: a zero pad never outranks a
            // real key, since pads sit at indices >= A.
            uint32_t P = 1;
            while (P < 8 && A * (2 * P) <= (uint32_t)NT) P *= 2;
            const uint32_t AP = (A + 8 * P - 1) & ~(8 * P - 1);
            for (uint32_t i = threadIdx.x; i < AP; i += NT)
                s.keys[i] = i < A ? (unsigned long long)__double_as_longlong(rem[i]) : 0ull;
            __syncthreads();
            // P > 1: one pass, every lane of a warp that holds a symbol takes
            // part in the shuffles (A * P <= NT, rounded up to whole warps)
            const uint32_t span = P > 1 ? ((A * P + 31) & ~31u) : A;
            for (uint32_t t = threadIdx.x; t < span; t += NT) {
                const uint32_t i = t / P, q = t % P;
                const bool live = i < A;
                const unsigned long long ki = s.keys[live ? i : 0];
                uint32_t r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                // lanes of one symbol read 8-byte keys j = q (mod P): distinct banks
                for (uint32_t j = q; j < AP; j += 8 * P) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t jj = j + u * P;
                        const unsigned long long kj = s.keys[jj];
                        r[u] += (kj > ki) | ((kj == ki) & (jj < i));
                    }
                }
                uint32_t rank = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
                for (uint32_t o = 1; o < P; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
                if (live && q == 0 && rank < k) freqs[i] += 1;
            }
        } else {
            deficit_radix(rem, A, k, freqs, s);
        }
    }
    __syncthreads();
    SEL_PROBE_AT(prb, 9);
    unsigned long long sum2 = 0;
    for (uint32_t i = threadIdx.x; i < A; i += NT) {
        if (counts[i] > 0 && freqs[i] == 0) freqs[i] = 1;
        sum2 += freqs[i];
    }
    sum2 = block_sum64(sum2, s);
    long long surplus = (long long)sum2 - (long long)target;
    SEL_PROBE_AT(prb, 10);
    while (surplus > 0) {
        // argmax, first index on ties (np.argmax)
        unsigned long long best = 0;
        for (uint32_t i = threadIdx.x; i < A; i += NT) {
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
            for (int w = 0; w < NT / 32; ++w) bb = s.red64[w] > bb ? s.red64[w] : bb;
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
    SEL_PROBE_AT(prb, 11);
    // cdf (rans.py:130)
    if (cum) {
        uint32_t carry = 0;
        for (uint32_t base = 0; base < A; base += NT) {
            uint32_t i = base + threadIdx.x;
            uint32_t v = i < A ? freqs[i] : 0;
            uint32_t tot;
            uint32_t ex = block_exclusive_scan<NT>(v, s.scan, &tot);
            if (i < A) cum[i] = carry + ex;
            carry += tot;
        }
        if (threadIdx.x == 0) cum[A] = carry;
    }
    __syncthreads();
    return SCZ_OK;
}

// Histogram of D for candidate c into counts[0..acap); returns alphabet.
template <int NT>
__device__ __noinline__ uint32_t assemble_counts(const SelectParams& p, uint32_t b, uint32_t c,
                                    uint32_t* counts, BlockScratch<NT>& s) {
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
        for (uint32_t i = 1 + threadIdx.x; i <= K; i += NT) rsum += rh[i];
    rsum = block_sum64(rsum, s);
    for (uint32_t i = threadIdx.x; i < ubound; i += NT) {
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
        for (uint32_t col = threadIdx.x; col < K; col += NT) counts[col] += rh[K + 1 + col];
    }
    __syncthreads();
    uint32_t last = 0;
    for (uint32_t i = threadIdx.x; i < ubound; i += NT)
        if (counts[i]) last = i + 1;
    return block_max32(last, s);
}

// -(p log2 p).sum() over the positive counts, in numpy's order (rans.py:219-223).
template <int NT>
__device__ __noinline__ double block_entropy(const uint32_t* counts, uint32_t A, double total, double* terms,
                                BlockScratch<NT>& s) {
    uint32_t carry = 0;
    for (uint32_t base = 0; base < A; base += NT) {
        uint32_t i = base + threadIdx.x;
        uint32_t c = i < A ? counts[i] : 0;
        uint32_t tot;
        uint32_t ex = block_exclusive_scan<NT>(c > 0 ? 1u : 0u, s.scan, &tot);
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

// Candidate pricing (search path, A <= 1024), all threads of the CTA on one
// batch of `nb` candidate slots at a time:
//   1. warp k assembles candidate k's histogram of D, its alphabet and its
//      positive counts in index order (ballot compaction);
//   2. every thread computes p log2 p terms over the flattened (slot, term)
//      index -- the fp64 division and logarithm dominate, so they are spread
//      over the whole CTA instead of one warp per candidate;
//   3. warp k sums candidate k's terms in numpy's pairwise order: the eight
//      accumulator chains of every <= 128-term leaf in parallel lanes, the
//      leaf's fixed combination tree by shuffles, then the recursion over the
//      leaves by lane 0 (pairwise_tree).
// dynamic smem = [vhist][row + column histograms if they fit]
//                [per slot: counts u32[acap], positive counts u32[acap], terms f64[acap]],
// the histograms staged with one batch of cp.async copies.
constexpr uint32_t SEL_WARP_ACAP = 1024;
constexpr uint32_t SEL_RH_SMEM_MAX = 16384;  // histogram words staged in smem (64 KB)

__host__ __device__ inline size_t select_smem_bytes(uint32_t acap, uint32_t rh_stride, uint32_t nb) {
    if (acap > SEL_WARP_ACAP) return 0;
    size_t s = (size_t)nb * acap * (4 + 4 + 8) + 256 * 4;
    if (rh_stride <= SEL_RH_SMEM_MAX) s += ((size_t)rh_stride * 4 + 15) & ~(size_t)15;
    return (s + 15) & ~(size_t)15;
}

// Leaves (offset, length) of numpy's pairwise recursion over n terms, in
// order (n <= 1024 gives at most 8 leaves of <= 128).
__device__ __forceinline__ uint32_t pw_leaves(uint32_t n, uint32_t* off, uint32_t* len) {
    uint32_t so[8], sl[8];
    int sp = 0;
    uint32_t cnt = 0;
    so[0] = 0;
    sl[0] = n;
    sp = 1;
    while (sp > 0) {
        --sp;
        const uint32_t o = so[sp], l = sl[sp];
        if (l > 128) {
            uint32_t n2 = l / 2;
            n2 -= n2 % 8;
            so[sp] = o + n2;  // right pushed first, left visited first
            sl[sp] = l - n2;
            ++sp;
            so[sp] = o;
            sl[sp] = n2;
            ++sp;
        } else {
            off[cnt] = o;
            len[cnt] = l;
            ++cnt;
        }
    }
    return cnt;
}

// numpy's recursion over n terms with the leaf sums given (in leaf order).
__device__ double pairwise_tree(uint32_t n, const double* leafsum) {
    uint32_t lens[26];
    double lefts[26];
    uint32_t right = 0, li = 0;
    int d = 0;
    lens[0] = n;
    for (;;) {
        while (lens[d] > 128) {
            uint32_t n2 = lens[d] / 2;
            n2 -= n2 % 8;
            lens[d + 1] = n2;
            right &= ~(1u << (d + 1));
            ++d;
        }
        double ret = leafsum[li++];
        for (;;) {
            if (d == 0) return ret;
            if ((right >> d) & 1u) {
                ret = __dadd_rn(lefts[d - 1], ret);
                --d;
            } else {
                lefts[d - 1] = ret;
                lens[d] = lens[d - 1] - lens[d];
                right |= 1u << d;
                break;
            }
        }
    }
}

// Pairwise sum of a[0..n) (n <= 1024) by one warp; the result in every lane.
template <int NT>
__device__ double pairwise_warp(const double* a, uint32_t n, uint32_t lane, BlockScratch<NT>& s) {
    uint32_t off[8], len[8];
    const uint32_t nl = pw_leaves(n, off, len);
    double* ls = s.leafsum[threadIdx.x >> 5];
#pragma unroll
    for (uint32_t r = 0; r < 2; ++r) {  // chains (leaf, j) = lane + 32 r
        const uint32_t L = 4 * r + (lane >> 3), j = lane & 7;
        double v = 0.0;
        const bool have = L < nl;
        const uint32_t o = have ? off[L] : 0, l = have ? len[L] : 0;
        if (have && l >= 8) {
            v = a[o + j];
            const uint32_t end = l - l % 8;
            for (uint32_t i = 8 + j; i < end; i += 8) v = __dadd_rn(v, a[o + i]);
        }
        // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)) within 8 lanes
        v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, 1));
        v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, 2));
        v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, 4));
        if (have && j == 0) {
            double res;
            if (l < 8) {
                res = 0.0;
                for (uint32_t i = 0; i < l; ++i) res = __dadd_rn(res, a[o + i]);
            } else {
                res = v;
                for (uint32_t i = l - l % 8; i < l; ++i) res = __dadd_rn(res, a[o + i]);
            }
            ls[L] = res;
        }
    }
    __syncwarp();
    double t = 0.0;
    if (lane == 0) t = n ? pairwise_tree(n, ls) : 0.0;
    t = __shfl_sync(0xffffffffu, t, 0);
    __syncwarp();
    return t;
}

// Returns the start of the slot scratch (reused by the final normalise).
template <int NT>
__device__ uint8_t* flat_costs(const SelectParams& p, uint32_t b, uint32_t g, BlockScratch<NT>& s) {
    extern __shared__ __align__(16) uint8_t sel_dyn[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr uint32_t NW = NT / 32;
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
        for (uint32_t i = threadIdx.x; i < p.rhist_stride; i += NT) cp_async4(s_rh + i, grh + i);
        dyn += ((size_t)p.rhist_stride * 4 + 15) & ~(size_t)15;
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    SEL_PROBE(1);
    const uint32_t* rhb = rh_smem ? s_rh : grh;
    const uint32_t acap = p.acap, nb = p.nb;
    uint32_t* cbase = reinterpret_cast<uint32_t*>(dyn);
    uint32_t* ccbase = cbase + (size_t)nb * acap;
    double* tbase = reinterpret_cast<double*>(ccbase + (size_t)nb * acap);
    const uint32_t nv = 1u << p.q_bits;
    const bool keep = p.groups > 1 || p.pass != 0;  // costs go to gcost for another CTA / pass
    const uint32_t first = p.c_begin + g;
    const uint32_t mine = first < p.c_end ? (p.c_end - first + p.groups - 1) / p.groups : 0;
    for (uint32_t r0 = 0; r0 < mine; r0 += nb) {
        const uint32_t nr = min(nb, mine - r0);
        // 1. histogram, alphabet and positive counts of slot k's candidate
        for (uint32_t k = warp; k < nr; k += NW) {
            const uint32_t c = first + p.groups * (r0 + k);
            const uint32_t K = p.cand_k[c], N = p.cand_n[c];
            const uint32_t ub = max(nv, K + 1);
            const uint32_t* rh = rhb + p.rhist_off[c];
            uint32_t* cb = cbase + (size_t)k * acap;
            uint32_t* cc = ccbase + (size_t)k * acap;
            uint32_t rsum = 0;  // rows with r >= 1 (bin 0 is N - rsum)
            if (K > 1)
                for (uint32_t i = 1 + lane; i <= K; i += 32) rsum += rh[i];
            rsum = warp_sum(rsum);
            for (uint32_t i = lane; i < ub; i += 32) {
                uint32_t v = (i < nv) ? s_vh[i] : 0;
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
            uint32_t last = 0, m = 0;
            for (uint32_t i0 = 0; i0 < ub; i0 += 32) {
                const uint32_t i = i0 + lane;
                const uint32_t cnt = i < ub ? cb[i] : 0;
                const uint32_t bal = __ballot_sync(0xffffffffu, cnt > 0);
                if (cnt > 0) {
                    cc[m + __popc(bal & lanemask_lt())] = cnt;
                    last = i + 1;
                }
                m += __popc(bal);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
            const uint32_t A = last;
            if (p.dump) {  // kept for the chosen candidate's table (and scz_search)
                uint32_t* dd = p.dump + ((uint64_t)b * p.n_cand + c) * acap;
                for (uint32_t i = lane; i < acap; i += 32) dd[i] = i < A ? cb[i] : 0;
            }
            if (lane == 0) {
                s.acnt[c] = A;
                s.mk[k] = m;
                if (keep) p.gacnt[(uint64_t)b * MAX_CAND + c] = A;
            }
        }
        __syncthreads();
        SEL_PROBE(12);
        if (threadIdx.x == 0) {
            uint32_t acc = 0;
            for (uint32_t k = 0; k < nr; ++k) {
                s.moff[k] = acc;
                acc += s.mk[k];
            }
            s.moff[nr] = acc;
        }
        __syncthreads();
        // 2. p log2 p over every (slot, term) (rans.py:219-223)
        const uint32_t M = s.moff[nr];
        for (uint32_t f = threadIdx.x; f < M; f += NT) {
            uint32_t k = 0;
            while (s.moff[k + 1] <= f) ++k;
            const uint32_t c = first + p.groups * (r0 + k);
            const double total = (double)(2 * nnz + p.cand_n[c]);
            const uint32_t j = f - s.moff[k];
            tbase[(size_t)k * acap + j] = plog2p(__ddiv_rn((double)ccbase[(size_t)k * acap + j], total));
        }
        __syncthreads();
        SEL_PROBE(13);
        // 3. entropy and cost of slot k's candidate (optimizer.py:87-96)
        for (uint32_t k = warp; k < nr; k += NW) {
            const uint32_t c = first + p.groups * (r0 + k);
            const double h = -pairwise_warp<NT>(tbase + (size_t)k * acap, s.mk[k], lane, s);
            if (lane == 0) {
                const uint64_t len = 2 * nnz + p.cand_n[c];
                s.ents[c] = h;
                s.costs[c] = __dmul_rn((double)len, h);
                if (keep) {
                    double* gc = p.gcost + ((uint64_t)b * MAX_CAND + c) * 2;
                    gc[0] = h;
                    gc[1] = s.costs[c];
                }
            }
        }
        __syncthreads();
    }
    SEL_PROBE(2);
    return dyn;
}

// Multi-CTA pricing: true in the CTA that arrives last for tensor b, which
// then holds every candidate's (entropy, cost, alphabet) in `s`.
template <int NT>
__device__ bool gather_costs(const SelectParams& p, uint32_t b, BlockScratch<NT>& s) {
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
    for (uint32_t c = lo + threadIdx.x; c < hi; c += NT) {
        const volatile double* gc = p.gcost + ((uint64_t)b * MAX_CAND + c) * 2;
        s.ents[c] = gc[0];
        s.costs[c] = gc[1];
        s.acnt[c] = *(const volatile uint32_t*)(p.gacnt + (uint64_t)b * MAX_CAND + c);
    }
    __syncthreads();
    return true;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_select(const __grid_constant__ SelectParams p) {
    pdl_wait();
    const uint32_t b = blockIdx.y, g = blockIdx.x;
    SEL_PROBE(0);
    TensorState& st = p.state[b];
    if (st.status != SCZ_OK) return;
    if (p.pass == 2 && !st.sel_pending) return;  // decided by the first pass
    __shared__ BlockScratch<NT> s;
    uint32_t* counts = p.counts + (uint64_t)b * p.acap;
    double* terms = p.terms + (uint64_t)b * p.acap;
    const uint64_t nnz = st.nnz;

    uint32_t chosen = 0, flags = 0, evaluated = 0;
    uint8_t* work = nullptr;  // shared scratch for the final normalise (warp path)
    if (p.searching) {
        if (p.acap <= SEL_WARP_ACAP) {
            work = flat_costs<NT>(p, b, g, s);
            if (!gather_costs(p, b, s)) return;
            SEL_PROBE(3);
        } else for (uint32_t c = 0; c < p.n_cand; ++c) {
            uint32_t A = assemble_counts(p, b, c, counts, s);
            if (p.dump) {
                uint32_t* dd = p.dump + ((uint64_t)b * p.n_cand + c) * p.acap;
                for (uint32_t i = threadIdx.x; i < p.acap; i += NT) dd[i] = i < A ? counts[i] : 0;
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
        for (uint32_t i = threadIdx.x; i < A; i += NT) scnt[i] = ccounts[i];
        __syncthreads();
        ccounts = scnt;
    }
    SEL_PROBE(4);
    int status = block_normalize(ccounts, A, p.precision, freqs, rem, cum, s,
                                 p.probe && p.pass != 2 ? p.probe + (blockIdx.y * gridDim.x + blockIdx.x) * 16 : nullptr);
    SEL_PROBE(5);
    EncTab* et = p.enctab + (uint64_t)b * p.acap;
    if (status == SCZ_OK)
        for (uint32_t i = threadIdx.x; i < A; i += NT) {
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

template __global__ void k_select<SEL_THREADS>(const __grid_constant__ SelectParams);
template __global__ void k_select<SEL_THREADS_WIDE>(const __grid_constant__ SelectParams);

// Stage entry point: normalize_frequencies of an arbitrary count vector.
__global__ void __launch_bounds__(SEL_THREADS) k_normalize_only(const uint32_t* counts, uint32_t A,
                                                               int precision, uint32_t* freqs,
                                                               double* rem, int32_t* status) {
    pdl_wait();
    __shared__ BlockScratch<SEL_THREADS> s;
    int st = block_normalize(counts, A, precision, freqs, rem, nullptr, s);
    if (threadIdx.x == 0) *status = st;
}

}  // namespace scz
