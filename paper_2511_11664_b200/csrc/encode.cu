// encode.cu -- compress-side kernels (K1, K2, K3, K6-prep).
//
//   k_stats      K1+K2  min/max, non-finite flag, zero bitmap, per-tile nnz;
//                       the last CTA of each tensor reduces the tiles, scans
//                       tile nnz and runs compute_params in fp64.
//   k_quantize   K3     guard-band fp32 quantiser with exact fp64 fix-up,
//                       rank-compaction of original-nonzero values into v8,
//                       and the value histogram.
//   k_colhist           column histogram modulo P = lcm(32, every candidate K)
//                       from the bitmap (one pass prices every candidate).
//   k_rowhist           per-candidate histogram of row nonzero counts.
//   k_materialize       col indices and row counts for the chosen K (c, r).
#include "common.cuh"

namespace scz {

// Per-tensor scratch regions zeroed by k_stats for the kernels after it
// (replaces memset launches on the latency path): region r of tensor b is
// ptr[r][b * words[r], (b + 1) * words[r]), split over the tensor's tiles.
struct ZeroSpec {
    uint32_t* ptr[5];
    uint32_t words[5];
    uint32_t per[5];  // words per tile CTA: ceil(words / n_tiles)
};

struct StatsParams {
    const float* x;
    uint64_t total;       // T
    uint32_t n_tiles;
    uint32_t words_pad;   // bitmap words per tensor (n_tiles * TILE_WORDS)
    int q_bits;
    uint32_t* bitmap;     // [B][words_pad]
    float4* tile_stats;   // [B][n_tiles] {min, max, nnz(bits), nonfinite(bits)}
    uint32_t* tile_off;   // [B][n_tiles] exclusive nnz prefix
    TensorState* state;   // [B]
    ZeroSpec zero;        // optional (pipeline launches)
};

// Load 4 consecutive elements starting at idx (idx % 4 == 0); out-of-range
// lanes read as 0 and are flagged invalid.
__device__ __forceinline__ float4 load4(const float* xb, uint64_t idx, uint64_t total,
                                        bool aligned, uint32_t* valid) {
    if (aligned && idx + 3 < total) {
        *valid = 0xF;
        return __ldg(reinterpret_cast<const float4*>(xb + idx));
    }
    float v[4];
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (idx + j < total) {
            v[j] = xb[idx + j];
            m |= 1u << j;
        } else {
            v[j] = 0.0f;
        }
    }
    *valid = m;
    return make_float4(v[0], v[1], v[2], v[3]);
}

// tensor.py:101-122 compute_params in fp64 with explicitly rounded ops.
__device__ void device_compute_params(float fmin, float fmax, int q_bits, double* scale,
                                      int64_t* z) {
    double x_min = (double)fmin, x_max = (double)fmax;
    int64_t q_max = (1 << q_bits) - 1;
    double lo = (0.0 < x_min) ? 0.0 : x_min;
    double hi = (0.0 > x_max) ? 0.0 : x_max;
    double s;
    int64_t zz;
    if (hi == lo) {
        s = 1.0;
        zz = 0;
    } else {
        s = __ddiv_rn(__dsub_rn(hi, lo), (double)q_max);
        double t = __ddiv_rn(-lo, s);
        double a = floor(__dadd_rn(fabs(t), 0.5));
        zz = (int64_t)copysign(a, t);
    }
    if (zz < 0) zz = 0;
    if (zz > q_max) zz = q_max;
    *scale = s;
    *z = zz;
}

#ifndef SCZ_STATS_MINB
#define SCZ_STATS_MINB 5
#endif
#ifndef SCZ_QUANT_MINB
#define SCZ_QUANT_MINB 5
#endif
#ifndef SCZ_MAT_MINB
#define SCZ_MAT_MINB 7
#endif
__global__ void __launch_bounds__(TILE_THREADS, SCZ_STATS_MINB) k_stats(StatsParams p) {
    pdl_wait();
    const uint32_t tile = blockIdx.x, b = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float* xb = p.x + (uint64_t)b * p.total;
    const bool aligned = ((reinterpret_cast<uintptr_t>(xb) & 15) == 0);
    const uint64_t tile_base = (uint64_t)tile * TILE;
    uint32_t* bm = p.bitmap + (uint64_t)b * p.words_pad + (uint64_t)tile * TILE_WORDS;

    float mn = INFINITY, mx = -INFINITY;
    uint32_t nnz = 0, bad = 0;
    // all eight 16-byte loads in flight before any use (memory-level parallelism)
    float4 vv[8];
    uint32_t vvalid[8];
#pragma unroll
    for (int it = 0; it < 8; ++it)
        vv[it] = load4(xb, tile_base + warp * 1024 + it * 128 + lane * 4, p.total, aligned, &vvalid[it]);
    // scratch zeroing for the later kernels, while the loads are in flight
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        if (!p.zero.ptr[r]) continue;
        const uint32_t w = p.zero.words[r], per = p.zero.per[r];
        uint32_t* z = p.zero.ptr[r] + (uint64_t)b * w;
        const uint32_t i1 = min(w, (tile + 1) * per);
        for (uint32_t i = tile * per + threadIdx.x; i < i1; i += TILE_THREADS) z[i] = 0u;
    }
    if (aligned && tile_base + TILE <= p.total) {
        // full tile (all but a tensor's last): no per-element validity; a
        // non-finite element turns acc = sum of e * 0 into NaN (one FMA per
        // element instead of a compare and a select)
        float acc = 0.0f;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            const float4 v = vv[it];
            mn = fminf(mn, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
            mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
            acc = __fmaf_rn(v.x, 0.0f, acc);
            acc = __fmaf_rn(v.y, 0.0f, acc);
            acc = __fmaf_rn(v.z, 0.0f, acc);
            acc = __fmaf_rn(v.w, 0.0f, acc);
            const uint32_t nib = (uint32_t)(v.x != 0.0f) | ((uint32_t)(v.y != 0.0f) << 1) |
                                 ((uint32_t)(v.z != 0.0f) << 2) | ((uint32_t)(v.w != 0.0f) << 3);
            nnz += __popc(nib);
            uint32_t w = nib << (4 * (lane & 7));
            w |= __shfl_xor_sync(0xffffffffu, w, 1);
            w |= __shfl_xor_sync(0xffffffffu, w, 2);
            w |= __shfl_xor_sync(0xffffffffu, w, 4);
            if ((lane & 7) == 0) bm[warp * 32 + it * 4 + (lane >> 3)] = w;
        }
        bad = acc != acc;
    } else {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            const uint32_t valid = vvalid[it];
            const float4 v = vv[it];
            float e[4] = {v.x, v.y, v.z, v.w};
            uint32_t nib = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (valid >> j & 1) {
                    if (!isfinite(e[j])) bad = 1;
                    mn = fminf(mn, e[j]);
                    mx = fmaxf(mx, e[j]);
                    nib |= (uint32_t)(e[j] != 0.0f) << j;
                }
            }
            nnz += __popc(nib);
            uint32_t w = nib << (4 * (lane & 7));
            w |= __shfl_xor_sync(0xffffffffu, w, 1);
            w |= __shfl_xor_sync(0xffffffffu, w, 2);
            w |= __shfl_xor_sync(0xffffffffu, w, 4);
            if ((lane & 7) == 0) bm[warp * 32 + it * 4 + (lane >> 3)] = w;
        }
    }
    // block reduce
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    __shared__ float s_mn[8], s_mx[8];
    __shared__ uint32_t s_nnz[8], s_bad[8];
    __shared__ uint32_t s_last;
    if (lane == 0) {
        s_mn[warp] = mn;
        s_mx[warp] = mx;
        s_nnz[warp] = nnz;
        s_bad[warp] = bad;
    }
    __syncthreads();
    // warp 0 alone publishes the tile, takes the ticket and, in the tensor's
    // last CTA, reduces all tiles: the other warps retire right away
    if (warp != 0) return;
    mn = lane < 8 ? s_mn[lane] : INFINITY;
    mx = lane < 8 ? s_mx[lane] : -INFINITY;
    nnz = lane < 8 ? s_nnz[lane] : 0u;
    bad = lane < 8 ? s_bad[lane] : 0u;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    uint32_t last = 0;
    if (lane == 0) {
        p.tile_stats[(uint64_t)b * p.n_tiles + tile] =
            make_float4(mn, mx, __uint_as_float(nnz), __uint_as_float(bad));
        __threadfence();
        last = atomicAdd(&p.state[b].tiles_done, 1u) == p.n_tiles - 1;
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return;
    __threadfence();

    // ---- last CTA of tensor b (warp 0): reduce tiles, scan nnz, params ----
    const float4* ts = p.tile_stats + (uint64_t)b * p.n_tiles;
    uint32_t* toff = p.tile_off + (uint64_t)b * p.n_tiles;
    float gmn = INFINITY, gmx = -INFINITY;
    uint32_t gbad = 0, carry = 0;
    for (uint32_t base = 0; base < p.n_tiles; base += 32) {
        const uint32_t i = base + lane;
        uint32_t c = 0;
        if (i < p.n_tiles) {
            const float4 t4 = __ldcg(ts + i);
            gmn = fminf(gmn, t4.x);
            gmx = fmaxf(gmx, t4.y);
            c = __float_as_uint(t4.z);
            gbad |= __float_as_uint(t4.w);
        }
        uint32_t inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (uint32_t)o) inc += y;
        }
        if (i < p.n_tiles) toff[i] = carry + inc - c;
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        gmn = fminf(gmn, __shfl_xor_sync(0xffffffffu, gmn, o));
        gmx = fmaxf(gmx, __shfl_xor_sync(0xffffffffu, gmx, o));
        gbad |= __shfl_xor_sync(0xffffffffu, gbad, o);
    }
    if (lane == 0) {
        TensorState& st = p.state[b];
        st.xmin = gmn;
        st.xmax = gmx;
        st.nonfinite = gbad;
        st.nnz = carry;
        st.tiles_done = 0;  // re-arm for the next launch
        st.errbits = 0;
        st.status = SCZ_OK;
        if (gbad) {
            st.status = SCZ_INVALID_INPUT;
            st.scale = 1.0;
            st.zero_point = 0;
            st.fast = 0;
            st.rcp32 = 1.0f;
        } else {
            double s;
            int64_t z;
            device_compute_params(gmn, gmx, p.q_bits, &s, &z);
            st.scale = s;
            st.zero_point = z;
            // guard-band path needs fl32(1/s) normal and x*r32 finite
            st.fast = (s >= 0x1p-120 && s <= 0x1p120) ? 1u : 0u;
            st.rcp32 = (float)(1.0 / s);
        }
    }
}

// ---------------------------------------------------------------- quantize
struct QuantParams {
    const float* x;
    uint64_t total;
    uint32_t n_tiles;
    uint32_t words_pad;
    int q_bits;
    const uint32_t* bitmap;
    const uint32_t* tile_off;
    const TensorState* state;
    uint8_t* v8;          // [B][v8_stride] compacted value symbols (head of D)
    uint32_t* vhist;      // [B][256]
    uint32_t* sym_out;    // optional [B][total] full symbol array (stage API)
    uint64_t v8_stride;
};

// tensor.py:130-140 for one element: exact fp64 sequence of the reference.
// Out of line on purpose: it runs for ~0.03 % of elements and must not be
// if-converted into every element of the hot loop.
__device__ __noinline__ uint32_t quant_exact(float x, double scale, double zf, double qmax) {
    double y = __dadd_rn(__ddiv_rn((double)x, scale), zf);
    double a = floor(__dadd_rn(fabs(y), 0.5));
    double r = (y > 0.0) ? a : ((y < 0.0) ? -a : 0.0);
    r = fmin(fmax(r, 0.0), qmax);
    return (uint32_t)r;
}

// fp32 estimate y = x * fl32(1/s) + z has |error| < 2^-15.4; any
// y within QGUARD = 2^-13 of a rounding boundary k + 1/2 is recomputed exactly.
constexpr float QGUARD = 0x1p-13f;
__device__ __forceinline__ uint32_t quant_fast(float x, float r32, float zf32, int qmax,
                                               double scale, double zf, bool fast) {
    if (fast) {
        // d = y - rint(y) is exact; y lies within QGUARD of a half-integer
        // iff |d| >= 1/2 - QGUARD, and only those take the exact path
        const float y = fmaf(x, r32, zf32);
        const float rq = rintf(y);
        if (fabsf(y - rq) < 0.5f - QGUARD) {
            const int q = (int)rq;
            return (uint32_t)min(max(q, 0), qmax);
        }
    }
    return quant_exact(x, scale, zf, (double)qmax);
}

// One 8192-element tile of tensor b.  `staged`: the tile's fp32 data was
// prefetched into s_x by cp.async (a persistent launch, measured slower and
// not used: profiles/r2/attempts), else it is loaded here; on_loaded() runs
// once the data is in registers.
template <bool SYM_OUT, class OnLoaded>  // SYM_OUT: also write every element's symbol (stage API)
__device__ __forceinline__ void quantize_tile(const QuantParams& p, uint32_t tile, uint32_t b,
                                              const float4* s_x, bool staged, OnLoaded on_loaded) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const TensorState& st = p.state[b];
    const float* xb = p.x + (uint64_t)b * p.total;
    const bool aligned = ((reinterpret_cast<uintptr_t>(xb) & 15) == 0);
    const uint64_t tile_base = (uint64_t)tile * TILE;
    const uint32_t* bm = p.bitmap + (uint64_t)b * p.words_pad + (uint64_t)tile * TILE_WORDS;

    __shared__ uint32_t s_wpre[TILE_WORDS];
    __shared__ uint32_t s_wbits[TILE_WORDS];
    __shared__ uint32_t s_scan[33];
    // one histogram copy per warp (no inter-warp atomic contention), 1 KB
    // aligned so a bin address is the copy's base OR'd with 4 * symbol
    __shared__ __align__(1024) uint32_t s_hist[8][256];
    __shared__ __align__(16) uint8_t s_v[TILE + 32];  // the tile's value symbols, rank order
    const int nbins = 1 << p.q_bits;
    static_assert(8 * 256 == 2 * 4 * TILE_THREADS, "two 16-byte zero stores per thread");
    reinterpret_cast<uint4*>(&s_hist[0][0])[threadIdx.x] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(&s_hist[0][0])[threadIdx.x + TILE_THREADS] = make_uint4(0, 0, 0, 0);
    // all eight 16-byte loads in flight first (out-of-range lanes read 0:
    // their bitmap bits are 0 and the exact path re-checks the index)
    float4 vv[8];
    if (staged) {
        cp_async_wait<0>();
        __syncthreads();  // every thread's copies landed
#pragma unroll
        for (int it = 0; it < 8; ++it) vv[it] = s_x[warp * 256 + it * 32 + lane];
    } else if (aligned && tile_base + TILE <= p.total) {  // interior tile: no bounds checks
        const float4* x4 = reinterpret_cast<const float4*>(xb + tile_base + warp * 1024 + lane * 4);
#pragma unroll
        for (int it = 0; it < 8; ++it) vv[it] = __ldg(x4 + it * 32);
    } else {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            uint32_t valid;
            vv[it] = load4(xb, tile_base + warp * 1024 + it * 128 + lane * 4, p.total, aligned, &valid);
        }
    }
    on_loaded();  // the tile's data is in registers: s_x may be refilled
    uint32_t myword = bm[threadIdx.x];
    s_wbits[threadIdx.x] = myword;
    uint32_t tot;
    s_wpre[threadIdx.x] = block_exclusive_scan<TILE_THREADS>(__popc(myword), s_scan, &tot);
    // a warp reads only its own 32 words of s_wpre (written by its lanes after
    // the scan's closing barrier): a warp barrier orders them (racecheck)
    __syncwarp();
    const uint32_t base_rank = p.tile_off[(uint64_t)b * p.n_tiles + tile];
    const double scale = st.scale;
    const double zf = (double)st.zero_point;
    const float r32 = st.rcp32, zf32 = (float)st.zero_point;
    const bool fast = st.fast != 0;
    const int qmax = nbins - 1;
    uint8_t* v8 = p.v8 + (uint64_t)b * p.v8_stride;
    // values are staged at s_v + (destination & 15) so the aligned middle of
    // the copy-out is one bulk copy (block_copy_s2g_bulk)
    const uint32_t vsh = stage_shift(v8 + base_rank);

    // Branch-free over all 32 elements of the thread: the fp32 estimate for
    // every element and a store predicated on its bitmap bit.  In the fast
    // path the estimate's rint lies in [0, qmax] (y >= -1/2 and y <= qmax + 1/2
    // up to rounding, since lo <= x <= hi and z = round(-lo / s), and elements
    // within QGUARD of a half-integer are excluded), so the symbol is the low
    // byte of y + 1.5 * 2^23 and needs no clamp.  A bit per group of four
    // collects "an element is near a rounding boundary (or the scale is out of
    // the fp32 range)"; such groups are redone afterwards, the elements near a
    // boundary with the exact fp64 sequence.  The histogram is taken from the
    // staged symbols.
    uint32_t slow = fast ? 0u : 0xFFu;  // bit it: redo group it (4 elements)
    const uint32_t sv_base = (uint32_t)__cvta_generic_to_shared(s_v) + vsh;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
        const float4 v = vv[it];
        const float e[4] = {v.x, v.y, v.z, v.w};
        const int word = warp * 32 + it * 4 + (lane >> 3);
        const int bit0 = 4 * (lane & 7);
        const uint32_t wbits = s_wbits[word];
        const uint32_t nib = wbits >> bit0;  // nonzero flags (bitmap == x != 0, valid only)
        uint32_t sa = sv_base + s_wpre[word] + __popc(wbits & ((1u << bit0) - 1u));  // rank slot
        bool sl = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            // rint via the 1.5 * 2^23 magic constant (|y| < 2^22 whenever
            // `fast`): full-rate FADDs instead of FRND / F2I conversions
            const float y = fmaf(e[j], r32, zf32);
            const float t = __fadd_rn(y, 0x1.8p23f);
            const float rq = __fsub_rn(t, 0x1.8p23f);
            sl |= !(fabsf(__fsub_rn(y, rq)) < 0.5f - QGUARD);
            if constexpr (SYM_OUT) {
                // caller-supplied parameters: x may lie outside the range
                const uint32_t q = (uint32_t)min(max(__float_as_int(t) - 0x4B400000, 0), qmax);
                sts_u8_bump(sa, q, nib, 1u << j);
                const uint64_t idx = tile_base + warp * 1024 + it * 128 + lane * 4 + j;
                if (idx < p.total) p.sym_out[(uint64_t)b * p.total + idx] = q;
            } else {
                sts_u8_bump(sa, __float_as_uint(t), nib, 1u << j);
            }
        }
        slow |= (uint32_t)sl << it;
    }
    while (slow) {  // rare: exact fp64 path (tensor.py:130-140), x re-read
        const int it = __ffs(slow) - 1;
        slow &= slow - 1;
        const int word = warp * 32 + it * 4 + (lane >> 3);
        const uint32_t wbits = s_wbits[word];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t off = warp * 1024 + it * 128 + lane * 4 + j;
            if (tile_base + off >= p.total) continue;
            const float x = xb[tile_base + off];
            const float y = fmaf(x, r32, zf32);
            const float rq = __fsub_rn(__fadd_rn(y, 0x1.8p23f), 0x1.8p23f);
            if (fast && fabsf(__fsub_rn(y, rq)) < 0.5f - QGUARD) continue;
            const int bit = 4 * (lane & 7) + j;
            const uint32_t q = quant_exact(x, scale, zf, (double)qmax);
            if ((wbits >> bit) & 1u) s_v[vsh + s_wpre[word] + __popc(wbits & ((1u << bit) - 1u))] = (uint8_t)q;
            if constexpr (SYM_OUT) p.sym_out[(uint64_t)b * p.total + tile_base + off] = q;
        }
    }
    fence_proxy_async_smem();  // the staged values, for the bulk copy-out
    __syncthreads();
    // value histogram of the tile's symbols (per-warp copies): whole words
    // of four symbols, then the < 4 symbols before and after them
    {
        const uint32_t hb = (uint32_t)__cvta_generic_to_shared(&s_hist[warp][0]);
        const uint32_t sb = (uint32_t)__cvta_generic_to_shared(s_v);
        const uint32_t lo = vsh, hi = vsh + tot;
        const uint32_t wlo = min((lo + 3u) & ~3u, hi), whi = max(hi & ~3u, wlo);
        for (uint32_t i = wlo + 4 * threadIdx.x; i < whi; i += 4 * TILE_THREADS) {
            const uint32_t w4 = lds_u32(sb + i);
            red_shared_inc(hb | ((w4 << 2) & 0x3FCu));
            red_shared_inc(hb | ((w4 >> 6) & 0x3FCu));
            red_shared_inc(hb | ((w4 >> 14) & 0x3FCu));
            red_shared_inc(hb | ((w4 >> 22) & 0x3FCu));
        }
        if (threadIdx.x < wlo - lo) red_shared_inc(hb | (lds_u8(sb + lo + threadIdx.x) << 2));
        else if (threadIdx.x >= 32 && threadIdx.x - 32 < hi - whi)
            red_shared_inc(hb | (lds_u8(sb + whi + threadIdx.x - 32) << 2));
    }
    __syncthreads();
    // the tile's values go out: head / tail bytes by threads, the aligned
    // middle as one bulk copy
    block_copy_s2g_bulk(v8 + base_rank, s_v, tot);
    uint32_t* gh = p.vhist + (uint64_t)b * 256;
    for (int i = threadIdx.x; i < nbins; i += TILE_THREADS) {
        const uint32_t t = (s_hist[0][i] + s_hist[1][i]) + (s_hist[2][i] + s_hist[3][i]) +
                           (s_hist[4][i] + s_hist[5][i]) + (s_hist[6][i] + s_hist[7][i]);
        if (t) atomicAdd(gh + i, t);
    }
    if (threadIdx.x == 0) bulk_store_wait();  // the copy-out still reads s_v
}


template <bool SYM_OUT>
__global__ void __launch_bounds__(TILE_THREADS, SCZ_QUANT_MINB) k_quantize(QuantParams p) {
    pdl_wait();
    if (p.state[blockIdx.y].status != SCZ_OK) return;
    quantize_tile<SYM_OUT>(p, blockIdx.x, blockIdx.y, nullptr, false, [] {});
}

// ------------------------------------------------------- search histograms
struct ColHistParams {
    const uint32_t* bitmap;
    uint32_t words_pad;
    uint32_t n_words;      // ceil(T / 32)
    uint32_t period_words; // P / 32
    uint32_t n_rows;       // ceil(n_words / period_words)
    uint32_t rows_per_cta; // row chunk handled by one CTA
    uint32_t* hp;          // [B][P] counts of nonzeros at p mod P
    uint32_t hp_stride;
};

// H_P[j] = #{p : p mod P == j, x[p] != 0}; thread owns one bitmap word
// column of the (rows x P) view and counts its 32 bit positions.
__global__ void __launch_bounds__(128) k_colhist(ColHistParams p) {
    pdl_wait();
    const uint32_t q = blockIdx.x * 128 + threadIdx.x;
    const uint32_t b = blockIdx.z;
    const bool single = gridDim.y == 1;  // this CTA alone covers its columns
    if (q >= p.period_words && !single) return;
    const uint32_t r0 = blockIdx.y * p.rows_per_cta;
    // (in the single-CTA form, threads past the last column only take part
    // in the transposed store's barrier)
    const uint32_t r1 = q < p.period_words ? min(p.n_rows, r0 + p.rows_per_cta) : r0;
    const uint32_t* bm = p.bitmap + (uint64_t)b * p.words_pad;
    // nib[j] holds eight 4-bit counters: bit positions j, j + 4, ..., j + 28
    // of the word column, flushed into cnt[] every 15 rows (SWAR: 3
    // operations per 8 positions instead of 2 per position); rows are loaded
    // four at a time so the loads overlap
    uint32_t cnt[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) cnt[i] = 0;
    uint32_t nib[4] = {0, 0, 0, 0};
    uint32_t pending = 0;
    auto flush = [&]() {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int k = 0; k < 8; ++k) cnt[4 * k + j] += (nib[j] >> (4 * k)) & 0xFu;
            nib[j] = 0;
        }
        pending = 0;
    };
    for (uint32_t r = r0; r < r1; r += 4) {
        uint32_t w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t wi = (uint64_t)(r + u) * p.period_words + q;
            w[u] = (r + u < r1 && wi < p.n_words) ? __ldg(bm + wi) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int j = 0; j < 4; ++j) nib[j] += (w[u] >> j) & 0x11111111u;
        pending += 4;
        if (pending > 11) flush();
    }
    flush();
    if (single) {
        // the only contribution to these counters: plain stores, transposed
        // through shared memory so each warp writes 128 contiguous bytes
        // (dynamic shared memory: launches of the atomic form carry none)
        extern __shared__ uint32_t s_cnt[];  // [128 * 33]
#pragma unroll
        for (int i = 0; i < 32; ++i) s_cnt[threadIdx.x * 33 + i] = cnt[i];
        __syncthreads();
        uint32_t* hp = p.hp + (uint64_t)b * p.hp_stride + (uint64_t)blockIdx.x * 128 * 32;
        const uint32_t nw = min(128u, p.period_words - blockIdx.x * 128) * 32;
        for (uint32_t w = threadIdx.x; w < nw; w += 128) hp[w] = s_cnt[(w >> 5) * 33 + (w & 31)];
        return;
    }
    uint32_t* hp = p.hp + (uint64_t)b * p.hp_stride + q * 32;
#pragma unroll
    for (int i = 0; i < 32; ++i)
        if (cnt[i]) atomicAdd(hp + i, cnt[i]);
}

// popcount of bits [start, start + len) of a bitmap (len >= 1).
__device__ __forceinline__ uint32_t range_popc(const uint32_t* bm, uint64_t start, uint32_t len) {
    uint64_t end = start + len;
    uint64_t w0 = start >> 5, w1 = (end - 1) >> 5;
    uint32_t s = (uint32_t)(start & 31);
    if (w0 == w1) {
        uint32_t w = __ldg(bm + w0) >> s;
        uint32_t m = (len >= 32) ? 0xffffffffu : ((1u << len) - 1u);
        return __popc(w & m);
    }
    uint32_t c = __popc(__ldg(bm + w0) >> s);
    for (uint64_t w = w0 + 1; w < w1; ++w) c += __popc(__ldg(bm + w));
    uint32_t e = (uint32_t)(end & 31);
    uint32_t last = __ldg(bm + w1);
    c += __popc(e ? (last & ((1u << e) - 1u)) : last);
    return c;
}

struct RowHistParams {
    const uint32_t* bitmap;
    uint32_t words_pad;
    uint32_t n_cand;
    uint32_t cand_k[MAX_CAND];        // K per candidate
    uint32_t cand_rows[MAX_CAND];     // N per candidate
    uint32_t chunk_start[MAX_CAND + 1];  // first CTA-chunk of each candidate
    uint32_t rhist_off[MAX_CAND];     // offset of candidate's r-hist (K+1 bins)
    uint32_t rows_per_chunk;
    uint32_t* rhist;                  // [B][rhist_stride]
    uint32_t rhist_stride;
};

// Row-count histograms for every candidate K: r_i = popcount(row i).
__global__ void __launch_bounds__(256) k_rowhist(RowHistParams p) {
    pdl_wait();
    const uint32_t chunk = blockIdx.x, b = blockIdx.y;
    uint32_t c = 0;
    while (c + 1 < p.n_cand && p.chunk_start[c + 1] <= chunk) ++c;
    const uint32_t K = p.cand_k[c], N = p.cand_rows[c];
    const uint32_t nb = K + 1;
    extern __shared__ uint32_t s_h[];
    const bool use_smem = nb <= 4096;
    uint32_t* gh = p.rhist + (uint64_t)b * p.rhist_stride + p.rhist_off[c];
    if (use_smem)
        for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) s_h[i] = 0;
    __syncthreads();
    const uint32_t* bm = p.bitmap + (uint64_t)b * p.words_pad;
    const uint64_t r0 = (uint64_t)(chunk - p.chunk_start[c]) * p.rows_per_chunk;
    const uint64_t r1 = min((uint64_t)N, r0 + p.rows_per_chunk);
    for (uint64_t r = r0 + threadIdx.x; r < r0 + ((r1 - r0 + 31) & ~31ull); r += blockDim.x) {
        const bool live = r < r1;
        uint32_t v = live ? range_popc(bm, r * K, K) : 0xffffffffu;
        uint32_t peers = __match_any_sync(0xffffffffu, v);
        if (live && (threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) {
            if (use_smem) atomicAdd(&s_h[v], (uint32_t)__popc(peers));
            else atomicAdd(gh + v, (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    if (use_smem)
        for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x)
            if (s_h[i]) atomicAdd(gh + i, s_h[i]);
}

// ------------------------------------------------------------ materialise
struct MatParams {
    uint64_t total;
    uint32_t n_tiles;
    uint32_t words_pad;
    const uint32_t* bitmap;
    const uint32_t* tile_off;
    const TensorState* state;
    void* cr;             // [B][cr_stride] symbols of width sym_bytes
    uint64_t cr_stride;   // elements
    int sym_bytes;        // 1: skip tensors whose chosen width is not sizeof(S)
    int after_v;          // 1: c ++ r start at element nnz (u8: D = v ++ c ++ r contiguous)
};

template <typename S>
__device__ __forceinline__ void store_sym(void* base, uint64_t i, uint32_t v) {
    reinterpret_cast<S*>(base)[i] = (S)v;
}

// s_buf: TILE * 2 + 64 bytes of shared memory (u8: columns then row counts;
// u16: columns), shared by the width instances of one kernel
template <typename S>
__device__ __forceinline__ void materialize_body(const MatParams& p, uint8_t* s_buf) {
    const uint32_t tile = blockIdx.x, b = blockIdx.y;
    const TensorState& st = p.state[b];
    if (st.status != SCZ_OK) return;
    if (p.sym_bytes && st.sym_bytes != sizeof(S)) return;  // another width variant owns this tensor
    const uint32_t K = st.n_cols;
    const uint64_t nnz = st.nnz;
    const uint32_t* bm = p.bitmap + (uint64_t)b * p.words_pad;
    S* cr = reinterpret_cast<S*>(p.cr) + (uint64_t)b * p.cr_stride + (p.after_v ? nnz : 0);
    __shared__ uint32_t s_scan[33];
    __shared__ uint32_t s_w[TILE_WORDS + 2];  // this tile's bitmap + the next two words
    __shared__ uint8_t s_mod[64];             // i mod K for i < 64 (K <= 32)
    S* s_c0 = reinterpret_cast<S*>(s_buf);    // column indices staged in rank order
    const uint64_t word = (uint64_t)tile * TILE_WORDS + threadIdx.x;
    uint32_t w = bm[word];
    s_w[threadIdx.x] = w;
    if (threadIdx.x < 2) {
        const uint64_t nw = (uint64_t)(tile + 1) * TILE_WORDS + threadIdx.x;
        s_w[TILE_WORDS + threadIdx.x] = nw < p.words_pad ? bm[nw] : 0u;
    }
    if (threadIdx.x < 64 && K <= 32) s_mod[threadIdx.x] = (uint8_t)(threadIdx.x % K);
    uint32_t tot;
    uint32_t lrank = block_exclusive_scan<TILE_THREADS>(__popc(w), s_scan, &tot);  // syncs
    const uint32_t base_rank = p.tile_off[(uint64_t)b * p.n_tiles + tile];
    // u8 columns are staged at s_buf + (destination & 15) so the aligned
    // middle of the copy-out is one bulk copy (block_copy_s2g_bulk)
    const bool bulk = sizeof(S) == 1 && K <= 32;
    S* s_c = s_c0 + (bulk ? stage_shift(cr + base_rank) : 0u);
    // column index of every nonzero: p mod K (sparse.py:66-68)
    if (w) {
        // (32 * word) mod K without a 64-bit modulo: T < 2^31 so the fp64
        // quotient estimate is within one of the truth
        const uint32_t xw = (uint32_t)(word * 32);
        uint32_t qk = __double2uint_rz(__dmul_rn((double)xw, __drcp_rn((double)K)));
        int64_t rr = (int64_t)xw - (int64_t)qk * K;
        if (rr < 0) rr += K;
        if (rr >= K) rr -= K;
        const uint32_t m = (uint32_t)rr;
        if ((K & (K - 1)) == 0 && K <= 32) {  // K | 32: m == 0, c = bit mod K
            if constexpr (sizeof(S) == 1) {
                // all 32 bit positions, predicated (no per-lane trip count,
                // no bit scans): c = j mod K lands at the next rank slot
                uint32_t sa = (uint32_t)__cvta_generic_to_shared(s_c) + lrank;
                const uint32_t km = K - 1;
#pragma unroll
                for (int j = 0; j < 32; ++j) sts_u8_bump(sa, (uint32_t)j & km, w, 1u << j);
            } else {
                while (w) {
                    const int bit = __ffs(w) - 1;
                    w &= w - 1;
                    s_c[lrank++] = (S)(bit & (K - 1));
                }
            }
        } else {
            while (w) {
                const int bit = __ffs(w) - 1;
                w &= w - 1;
                uint32_t c = m + bit;
                c = (K <= 32) ? s_mod[c] : (c >= K ? c - K : c);
                s_c[lrank++] = (S)c;
            }
        }
    }
    // row counts for the rows starting in this tile (sparse.py:68)
    const uint64_t ts = (uint64_t)tile * TILE, te = min(ts + TILE, p.total);
    // 32-bit quotients (T < 2^31, so ts + K - 1 < 2^32; a 64-bit division
    // here was 11 % of the kernel's instructions), shifts for K = 2^k
    uint64_t i0, i1;
    if ((K & (K - 1)) == 0) {
        const uint32_t k = __ffs(K) - 1;
        i0 = ((uint32_t)ts + K - 1) >> k;
        i1 = ((uint32_t)te + K - 1) >> k;
    } else {
        i0 = ((uint32_t)ts + K - 1) / K;
        i1 = ((uint32_t)te + K - 1) / K;
    }
    if (sizeof(S) == 1 && K <= 32) {
        // u8: row counts staged too; c and r leave with 16-byte stores
        uint8_t* s_rc = s_buf + TILE + 32;  // (u8 columns use the first TILE + 32 bytes)
        const uint32_t kmask = K == 32 ? 0xffffffffu : ((1u << K) - 1u);
        const uint32_t nr = (uint32_t)(i1 - i0);
        if (K == 4) {
            // K = 4 divides the tile: thread t's bitmap word holds rows
            // 8t .. 8t + 7 as nibbles; SWAR nibble popcounts, spread to bytes
            static_assert(TILE % 4 == 0 && TILE_WORDS == TILE_THREADS, "one word per thread");
            const uint32_t ww = s_w[threadIdx.x];
            uint32_t x = ww - ((ww >> 1) & 0x55555555u);
            x = (x & 0x33333333u) + ((x >> 2) & 0x33333333u);
            const uint32_t lo = x & 0x0F0F0F0Fu, hi = (x >> 4) & 0x0F0F0F0Fu;
            reinterpret_cast<uint2*>(s_rc)[threadIdx.x] = make_uint2(__byte_perm(lo, hi, 0x5140), __byte_perm(lo, hi, 0x7362));
        } else {
            for (uint32_t j = threadIdx.x; j < nr; j += TILE_THREADS) {
                const uint32_t start = (uint32_t)((i0 + j) * K - ts);  // < TILE
                const uint32_t wi = start >> 5, sh = start & 31;
                s_rc[j] = (uint8_t)__popc(__funnelshift_r(s_w[wi], s_w[wi + 1], sh) & kmask);
            }
        }
        fence_proxy_async_smem();  // the column bytes, for the bulk copy
        __syncthreads();
        block_copy_s2g_bulk(reinterpret_cast<uint8_t*>(cr + base_rank), reinterpret_cast<const uint8_t*>(s_c0), tot);
        block_copy_s2g<TILE_THREADS>(reinterpret_cast<uint8_t*>(cr + nnz + i0), s_rc, nr);
        if (threadIdx.x == 0) bulk_store_wait();
        return;
    }
    __syncthreads();
    S* dst = cr + base_rank;
    for (uint32_t i = threadIdx.x; i < tot; i += TILE_THREADS) dst[i] = s_c[i];  // coalesced
    if (K <= 32) {
        const uint32_t kmask = K == 32 ? 0xffffffffu : ((1u << K) - 1u);
        for (uint64_t i = i0 + threadIdx.x; i < i1; i += TILE_THREADS) {
            const uint32_t start = (uint32_t)(i * K - ts);  // < TILE
            const uint32_t wi = start >> 5, sh = start & 31;
            cr[nnz + i] = (S)__popc(__funnelshift_r(s_w[wi], s_w[wi + 1], sh) & kmask);
        }
    } else {
        for (uint64_t i = i0 + threadIdx.x; i < i1; i += TILE_THREADS)
            cr[nnz + i] = (S)range_popc(bm, i * K, K);
    }
}

template <typename S>
__global__ void __launch_bounds__(TILE_THREADS) k_materialize(MatParams p) {
    pdl_wait();
    __shared__ __align__(16) uint8_t s_buf[TILE * (sizeof(S) < 2 ? 2 : sizeof(S)) + 64];
    materialize_body<S>(p, s_buf);
}

// The pipeline's launch: u8 and u16 classes in one grid (see k_rans_enc_v2_u8u16).
__global__ void __launch_bounds__(TILE_THREADS, SCZ_MAT_MINB) k_materialize_u8u16(MatParams p8, MatParams p16) {
    pdl_wait();
    __shared__ __align__(16) uint8_t s_buf[TILE * 2 + 64];
    const uint32_t w = p8.state[blockIdx.y].sym_bytes;
    if (w == 2) materialize_body<uint16_t>(p16, s_buf);
    else if (w == 1) materialize_body<uint8_t>(p8, s_buf);
}

template __global__ void k_materialize<uint8_t>(MatParams);
template __global__ void k_materialize<uint16_t>(MatParams);
template __global__ void k_materialize<uint32_t>(MatParams);

}  // namespace scz
