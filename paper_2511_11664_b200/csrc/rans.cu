// rans.cu -- rANS encode/decode kernels (K5, K7).
//
// Arithmetic per symbol is exactly rans.py:134-152 (32-bit state, L = 2^23,
// byte renormalisation, precision n).  Two layouts (FORMAT.md):
//   v1  one stream per tensor, byte-identical to rans.encode (rans.py:155-180);
//       one warp per tensor runs the serial recurrence (lanes redundant, the
//       table entries of the next 32 symbols are fetched in parallel).
//   v2  blocks of B symbols, W = 32 interleaved lanes per block, one warp per
//       block, one lane per rANS state.  Renormalisation bytes of a step are
//       placed by a warp ballot-scan (<= 2 bytes per lane per step).
#include "common.cuh"

namespace scz {

constexpr int ENC_WPB = 4;    // warps (= v2 blocks) per CTA
constexpr int DEC_WPB = 4;
constexpr int RING = 512;     // per-warp payload ring buffer (bytes)
constexpr uint32_t TAB_SMEM_MAX = 2048;  // symbols whose table fits in smem

// ---- symbol sources: D[i] for tensor b -----------------------------------
template <typename S>
struct SplitSrc {  // D = v8[0..nnz) ++ cr[0..nnz+N)
    const uint8_t* v8;
    uint64_t v8_stride;
    const S* cr;
    uint64_t cr_stride;
    __device__ __forceinline__ uint32_t at(uint32_t b, uint64_t i, uint64_t nnz) const {
        return i < nnz ? (uint32_t)v8[b * v8_stride + i] : (uint32_t)cr[b * cr_stride + (i - nnz)];
    }
    static constexpr int width = sizeof(S);
};
struct Contig8Src {  // D = v ++ c ++ r contiguous u8 (the common width)
    const uint8_t* d;
    uint64_t stride;
    __device__ __forceinline__ uint32_t at(uint32_t b, uint64_t i, uint64_t) const {
        return d[b * stride + i];
    }
    static constexpr int width = 1;
};
struct PlainSrc {  // D given as u32 (stage API)
    const uint32_t* d;
    uint64_t stride;
    __device__ __forceinline__ uint32_t at(uint32_t b, uint64_t i, uint64_t) const {
        return d[b * stride + i];
    }
    static constexpr int width = 0;  // matches any sym_bytes
};

struct EncParams {
    TensorState* state;
    const EncTab* enctab;
    uint32_t acap;
    int precision;
    uint32_t block_syms;      // v2 block size (multiple of 32)
    uint8_t* slots;           // block output slots
    uint64_t slot_cap;        // bytes per slot
    uint32_t slots_per_tensor;
    uint32_t* block_len;      // [B][slots_per_tensor]
    uint32_t tab_smem;        // table entries staged in dynamic smem (v2)
};

__device__ __forceinline__ void flag_err(TensorState& st, uint32_t bit) {
    atomicOr(&st.errbits, bit);
}
constexpr uint32_t ERR_OVERFLOW = 1, ERR_UNCODABLE = 2;

// v1: the reference's single stream.  One warp per tensor; all lanes carry
// the same state, lane j prefetches the table entry of the j-th next symbol.
template <class Src>
__global__ void __launch_bounds__(32) k_rans_enc_v1(EncParams p, Src src) {
    pdl_wait();
    const uint32_t b = blockIdx.x;
    TensorState& st = p.state[b];
    if (st.status != SCZ_OK) return;
    if (Src::width && st.sym_bytes != (uint32_t)Src::width) return;
    __shared__ EncTab s_tab[TAB_SMEM_MAX];
    const uint32_t A = st.alphabet;
    const EncTab* gt = p.enctab + (uint64_t)b * p.acap;
    const bool smem_tab = A <= TAB_SMEM_MAX;
    if (smem_tab)
        for (uint32_t i = threadIdx.x; i < A; i += 32) s_tab[i] = gt[i];
    __syncwarp();
    const EncTab* tab = smem_tab ? s_tab : gt;
    const uint32_t lane = threadIdx.x;
    const uint64_t L = st.stream_len, nnz = st.nnz;
    const int n = p.precision;
    uint8_t* slot = p.slots + (uint64_t)b * p.slots_per_tensor * p.slot_cap;
    uint8_t* tail = slot + p.slot_cap - 1;
    uint32_t x = STATE_LOW, err = 0;
    uint64_t emitted = 0;
    for (uint64_t top = L; top > 0;) {
        const uint32_t cnt = (uint32_t)(top < 32 ? top : 32);
        // lane j holds symbol top-1-j (processed j-th in this chunk)
        EncTab mine = {1, 0, 0, 0xFFFFFFFFu};
        uint32_t ok = 1;
        if (lane < cnt) {
            uint32_t sym = src.at(b, top - 1 - lane, nnz);
            if (sym >= A) {
                err |= ERR_OVERFLOW;
                ok = 0;
            } else {
                mine = tab[sym];
                if (mine.freq == 0) {
                    err |= ERR_UNCODABLE;
                    ok = 0;
                }
            }
        }
        if (__any_sync(0xffffffffu, !ok)) break;
        for (uint32_t j = 0; j < cnt; ++j) {
            EncTab t;
            t.freq = __shfl_sync(0xffffffffu, mine.freq, j);
            t.cum = __shfl_sync(0xffffffffu, mine.cum, j);
            t.rcp = __shfl_sync(0xffffffffu, mine.rcp, j);
            t.shift = __shfl_sync(0xffffffffu, mine.shift, j);
            const uint32_t bound = t.freq << (31 - n);
            if (x >= bound) {
                if (lane == 0) tail[-(int64_t)emitted] = (uint8_t)(x & 0xFF);
                x >>= 8;
                ++emitted;
                if (x >= bound) {
                    if (lane == 0) tail[-(int64_t)emitted] = (uint8_t)(x & 0xFF);
                    x >>= 8;
                    ++emitted;
                }
            }
            uint32_t q = enc_div(x, t);
            x = (q << n) + t.cum + (x - q * t.freq);
        }
        top -= cnt;
    }
    err = __reduce_or_sync(0xffffffffu, err);
    if (lane == 0) {
        uint8_t* start = slot + p.slot_cap - emitted - 4;
        start[0] = (uint8_t)x;
        start[1] = (uint8_t)(x >> 8);
        start[2] = (uint8_t)(x >> 16);
        start[3] = (uint8_t)(x >> 24);
        p.block_len[(uint64_t)b * p.slots_per_tensor] = (uint32_t)(4 + emitted);
        if (err) flag_err(st, err);
    }
}

// ---------------------------------------------------------------- decode
struct DecParams {
    const scz_info* info;        // [B] device copy
    const uint32_t* freqs;       // batch freq buffer
    const uint32_t* block_bytes; // batch block-length buffer
    const uint8_t* payload;      // batch payload buffer (256-byte aligned base)
    uint32_t* cumtab;            // scratch [B][acap + 1]
    uint32_t* blk_off;           // scratch [B][nblk_cap]
    uint32_t acap, nblk_cap;
    void* dsym;                  // out: tensor b's symbols at byte b * dsym_stride
    uint64_t dsym_stride;        // bytes (one stride for every symbol class of a batch)
    int32_t* status;             // [B]
    // v2 LUT classes: per-tensor decode tables built once in global memory
    // (k_dec_prepare slices) and bulk-copied into each decoder CTA:
    //   [2^n] u32 (f << 16) | (slot - cum)   then   [2^n] symbol (u8 / u16)
    uint8_t* lut;
    uint64_t lut_stride;         // bytes per tensor
    unsigned long long* chunk_state;  // [B][nchunk_cap] CSR look-back words, zeroed here
    uint32_t nchunk_cap;
    // 1: the v2 decoder adds the row counts of every SMALL_ROWS-row chunk of
    // u8 tensors with K in {1, 2, 4} into chunk_state (k_rows_small8 reads
    // the prefix instead of looking back)
    int chunk_sums;
    float* dq_lut;  // optional [B][256]: dequantised value of every u8 symbol (k_rows_small8)
};

constexpr uint32_t LUT_SLICE = 2048;  // slots per k_dec_prepare slice CTA

__host__ __device__ inline uint32_t lut_sym_off(int n) { return 4u << n; }

// Per tensor: validate the table (rans.py:49-56, Σ f == 2^n), build the cdf,
// scan block lengths into offsets and check them against the header.
// Slice CTA (blockIdx.x >= 1): slots [LUT_SLICE * (x - 1), LUT_SLICE * x) of
// the v2 decode tables of tensor blockIdx.y; thread t owns 8 consecutive
// slots: one binary search of the cdf, then a forward walk.
template <typename L>
__device__ void build_lut_slice(const DecParams& p, const scz_info& in, uint32_t b, uint32_t slice) {
    const int n = in.precision;
    const uint32_t A = in.alphabet;
    const uint32_t s0 = slice * LUT_SLICE;
    if (s0 >= (1u << n)) return;
    __shared__ uint32_t s_cum[4097];
    __shared__ uint32_t s_scan[33];
    const uint32_t* f = p.freqs + in.freqs_off;
    uint32_t carry = 0;
    for (uint32_t base = 0; base < A; base += 256) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t v = i < A ? f[i] : 0;
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan<256>(v, s_scan, &tot);
        if (i < A) s_cum[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) s_cum[A] = carry;
    __syncthreads();
    if (carry != (1u << n)) return;  // corrupt table: the prepare CTA flags it
    uint8_t* base = p.lut + (uint64_t)b * p.lut_stride;
    uint32_t* step = reinterpret_cast<uint32_t*>(base);
    L* sym = reinterpret_cast<L*>(base + lut_sym_off(n));
    // one layout for v1 and v2 (k_rans_dec_v1p reads f and slot - cum as the
    // two 16-bit halves of the entry)
    const bool split = false;
    uint16_t* f16 = reinterpret_cast<uint16_t*>(base);
    uint16_t* b16 = f16 + ((size_t)1 << n);
    const uint32_t slot0 = s0 + 8 * threadIdx.x;
    if (slot0 >= (1u << n)) return;
    uint32_t lo = 0, hi = A;  // last symbol with cum <= slot0
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_cum[mid] <= slot0) lo = mid;
        else hi = mid;
    }
    uint32_t e[8];
    L sy[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t sl = slot0 + k;
        while (s_cum[lo + 1] <= sl) ++lo;  // f = 0 symbols are skipped here
        e[k] = ((s_cum[lo + 1] - s_cum[lo]) << 16) | (sl - s_cum[lo]);
        sy[k] = (L)lo;
    }
    if (split) {
        uint32_t fw[4], bw[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            fw[k] = (e[2 * k] >> 16) | (e[2 * k + 1] & 0xFFFF0000u);
            bw[k] = (e[2 * k] & 0xFFFFu) | (e[2 * k + 1] << 16);
        }
        *reinterpret_cast<uint4*>(f16 + slot0) = make_uint4(fw[0], fw[1], fw[2], fw[3]);
        *reinterpret_cast<uint4*>(b16 + slot0) = make_uint4(bw[0], bw[1], bw[2], bw[3]);
    } else {
        uint4* d4 = reinterpret_cast<uint4*>(step + slot0);
        d4[0] = make_uint4(e[0], e[1], e[2], e[3]);
        d4[1] = make_uint4(e[4], e[5], e[6], e[7]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) sym[slot0 + k] = sy[k];
}

__global__ void __launch_bounds__(256) k_dec_prepare(DecParams p) {
    pdl_wait();
    const uint32_t b = blockIdx.y;
    const scz_info& in = p.info[b];
    if (blockIdx.x > 0) {
        if (p.status[b] != SCZ_OK || (in.version != 2 && in.version != 1)) return;
        if (in.sym_bytes == 1) build_lut_slice<uint8_t>(p, in, b, blockIdx.x - 1);
        else if (in.sym_bytes == 2) build_lut_slice<uint16_t>(p, in, b, blockIdx.x - 1);
        return;
    }
    __shared__ uint32_t s_scan[33];
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    if (p.dq_lut) build_dequant_lut(p.dq_lut + (uint64_t)b * 256, (double)in.zero_point, in.scale);
    if (p.chunk_state)
        for (uint32_t i = threadIdx.x; i < p.nchunk_cap; i += blockDim.x)
            p.chunk_state[(uint64_t)b * p.nchunk_cap + i] = 0ull;
    __syncthreads();
    if (p.status[b] != SCZ_OK) return;
    const uint32_t A = in.alphabet;
    const uint32_t* f = p.freqs + in.freqs_off;
    uint32_t* cum = p.cumtab + (uint64_t)b * (p.acap + 1);
    unsigned long long carry = 0;
    for (uint32_t base = 0; base < A; base += 256) {
        uint32_t i = base + threadIdx.x;
        uint32_t v = i < A ? f[i] : 0;
        uint32_t tot;
        uint32_t ex = block_exclusive_scan<256>(v, s_scan, &tot);
        if (i < A) cum[i] = (uint32_t)(carry + ex);
        carry += tot;
    }
    if (threadIdx.x == 0) cum[A] = (uint32_t)carry;
    if (carry != (1ull << in.precision) && threadIdx.x == 0) s_bad = 1;
    // block offsets
    const uint32_t W = in.version == 2 ? in.lanes : 1;
    uint32_t* off = p.blk_off + (uint64_t)b * p.nblk_cap;
    carry = 0;
    for (uint32_t base = 0; base < in.n_blocks; base += 256) {
        uint32_t i = base + threadIdx.x;
        uint32_t v = 0;
        if (i < in.n_blocks) {
            v = in.version == 2 ? p.block_bytes[in.blocks_off + i] : (uint32_t)in.payload_len;
            if (v < 4 * W) s_bad = 1;
        }
        uint32_t tot;
        uint32_t ex = block_exclusive_scan<256>(v, s_scan, &tot);
        if (i < in.n_blocks) off[i] = (uint32_t)(carry + ex);
        carry += tot;
    }
    if (threadIdx.x == 0 && carry != in.payload_len) s_bad = 1;
    __syncthreads();
    if (threadIdx.x == 0 && s_bad) p.status[b] = SCZ_CORRUPT_STREAM;
}

// slot -> symbol lookup table over [0, 2^n): thread t fills a contiguous
// range, starting from a binary search of cum.
template <typename L>
__device__ void build_lut(L* lut, const uint32_t* cum, uint32_t A, uint32_t nslots) {
    const uint32_t per = (nslots + blockDim.x - 1) / blockDim.x;
    uint32_t s0 = threadIdx.x * per;
    if (s0 >= nslots) return;
    uint32_t s1 = min(nslots, s0 + per);
    // largest sym with cum[sym] <= s0 (searchsorted right - 1)
    uint32_t lo = 0, hi = A + 1;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (cum[mid] <= s0) lo = mid;
        else hi = mid;
    }
    uint32_t sym = lo;
    for (uint32_t sl = s0; sl < s1; ++sl) {
        while (cum[sym + 1] <= sl) ++sym;
        lut[sl] = (L)sym;
    }
}

__device__ __forceinline__ uint32_t find_sym(const uint32_t* cum, uint32_t A, uint32_t slot) {
    uint32_t lo = 0, hi = A + 1;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (cum[mid] <= slot) lo = mid;
        else hi = mid;
    }
    return lo;
}

// slot -> symbol: LUT when L is u8/u16, binary search of the cdf otherwise
// (np.searchsorted(cdf, slot, 'right') - 1, rans.py:201).
template <typename L>
__device__ __forceinline__ uint32_t lookup(const L* lut, const uint32_t* cum, uint32_t A,
                                           uint32_t slot) {
    if constexpr (sizeof(L) == 4) return find_sym(cum, A, slot);
    else return lut[slot];
}

// Per-warp byte ring fed by aligned 128-byte chunks of the payload.
struct Ring {
    uint8_t* buf;
    uint64_t filled;  // absolute (payload-buffer) address up to which bytes are loaded
    __device__ __forceinline__ void fill_to(const uint8_t* payload, uint64_t want, uint32_t lane) {
        __syncwarp();  // every lane's earlier reads of the slots about to be refilled (racecheck)
        while (filled < want) {  // warp-uniform
            uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(payload + filled) + lane);
            *reinterpret_cast<uint32_t*>(buf + ((filled + 4 * lane) & (RING - 1))) = w;
            filled += 128;
        }
        __syncwarp();
    }
    __device__ __forceinline__ uint32_t byte(uint64_t a) const { return buf[a & (RING - 1)]; }
};

// v1 decode: one warp per tensor, the serial rans.decode loop (all lanes
// carry the same state; lane 0 stores).  Generic lookup (binary search) when
// the table does not fit a LUT.
template <typename S, typename L>
__global__ void __launch_bounds__(32) k_rans_dec_v1(DecParams p) {
    pdl_wait();
    const uint32_t b = blockIdx.x;
    const scz_info& in = p.info[b];
    if (p.status[b] != SCZ_OK || in.version != 1 || in.sym_bytes != sizeof(S)) return;
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* ringbuf = smem;
    uint2* s_tab = reinterpret_cast<uint2*>(smem + RING);
    const uint32_t A = in.alphabet;
    const int n = in.precision;
    const uint32_t nslots = 1u << n;
    const bool tab_smem = A <= TAB_SMEM_MAX;
    L* lut = reinterpret_cast<L*>(smem + RING + (tab_smem ? A : 0) * sizeof(uint2));
    const uint32_t* f = p.freqs + in.freqs_off;
    const uint32_t* cum = p.cumtab + (uint64_t)b * (p.acap + 1);
    if (tab_smem)
        for (uint32_t i = threadIdx.x; i < A; i += 32) s_tab[i] = make_uint2(f[i], cum[i]);
    if constexpr (sizeof(L) < 4) build_lut<L>(lut, cum, A, nslots);
    __syncwarp();
    const uint32_t lane = threadIdx.x;
    const uint64_t Ls = 2 * in.nnz + in.n_rows;
    const uint64_t blen = in.payload_len;
    const uint64_t a0 = in.payload_off;
    Ring ring{ringbuf, a0 & ~127ull};
    ring.fill_to(p.payload, a0 + 128, lane);
    uint32_t x = ring.byte(a0) | (ring.byte(a0 + 1) << 8) | (ring.byte(a0 + 2) << 16) |
                 (ring.byte(a0 + 3) << 24);
    uint64_t pos = 4;
    const uint32_t mask = nslots - 1;
    S* out = reinterpret_cast<S*>(reinterpret_cast<uint8_t*>(p.dsym) + (uint64_t)b * p.dsym_stride);
    bool bad = false;
    for (uint64_t i = 0; i < Ls; ++i) {
        const uint32_t slot = x & mask;
        const uint32_t sym = lookup<L>(lut, cum, A, slot);
        uint2 fc = tab_smem ? s_tab[sym] : make_uint2(f[sym], cum[sym]);
        x = fc.x * (x >> n) + slot - fc.y;
        while (x < STATE_LOW) {
            if (pos >= blen) {
                bad = true;
                break;
            }
            x = (x << 8) | ring.byte(a0 + pos);
            ++pos;
        }
        if (bad) break;
        if (lane == 0) out[i] = (S)sym;
        if (ring.filled < a0 + pos + 64) ring.fill_to(p.payload, a0 + pos + 64 + 256, lane);
    }
    if (!bad) bad = (x != STATE_LOW) || pos != blen;
    if (bad && lane == 0) p.status[b] = SCZ_CORRUPT_STREAM;
}

#define SCZ_INST_DEC(S, L) template __global__ void k_rans_dec_v1<S, L>(DecParams);
SCZ_INST_DEC(uint8_t, uint8_t)
SCZ_INST_DEC(uint16_t, uint16_t)
SCZ_INST_DEC(uint32_t, uint32_t)

#define SCZ_INST_ENC(SRC) template __global__ void k_rans_enc_v1<SRC>(EncParams, SRC);
SCZ_INST_ENC(Contig8Src)
SCZ_INST_ENC(SplitSrc<uint8_t>)
SCZ_INST_ENC(SplitSrc<uint16_t>)
SCZ_INST_ENC(SplitSrc<uint32_t>)
SCZ_INST_ENC(PlainSrc)

}  // namespace scz
