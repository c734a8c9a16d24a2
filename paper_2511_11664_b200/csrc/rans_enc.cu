// rans_enc.cu -- v2 interleaved-lane rANS encoder (K5).
//
// One warp codes one FORMAT.md v2 block; lane j owns state j and the
// block-local symbols i = j (mod 32).  Steps run in descending order; per
// step every lane renormalises (<= 2 bytes, rans.py:139-142), the warp places
// the bytes with one ballot-scan (lanes descending, low byte first), and the
// state transform uses the exact reciprocal of the frequency.
// Symbols are fetched 8 steps ahead into a rotating register queue (they do
// not depend on the state); the per-symbol table lives in shared memory.
// Emitted bytes are written backwards from the end of the block's slot, so
// the finished block is contiguous: [32 LE states][bytes in decoder order].
//
// Only the highest step of a block can be partial, so it is peeled; the
// remaining steps are full and branch-free.  CHECK adds the reference's
// AlphabetOverflow / UncodableSymbol detection (rans.py:176-179, 189-190) for
// caller-supplied tables (stage API); the pipeline's own tables cannot fail.
#include "common.cuh"

namespace scz {

constexpr int ENC2_WPB = 4;                  // warps (= blocks) per CTA
constexpr uint32_t ENC_TAB_SMEM_MAX = 8192;  // table entries staged in smem (128 KB)

// In-kernel packing (pipeline launches; payload == nullptr for the stage
// API): once a warp has coded its block it publishes the block's byte length,
// finds the block's payload offset by decoupled look-back over the tensor's
// earlier blocks (chunk_prefix), and copies the block from its slot into the
// tensor's payload region [b * pcap, b * pcap + payload_len).  The tensor's
// last block then knows the payload length and writes the header (scz_info).
struct PackParams {
    uint8_t* payload;          // [B][pcap]
    uint64_t pcap;
    unsigned long long* lb;    // [B][slots_per_tensor] look-back words (zeroed)
    scz_info* info;            // [B]
    uint64_t total;
    int q_bits;
    int write_failed;          // this launch writes the headers of failed tensors
};

// The header of tensor b from its device state (container.py:32-70 fields).
__device__ __forceinline__ void write_info(scz_info& in, const TensorState& st, int32_t status, int format,
                                           int q_bits, int precision, uint64_t total, uint32_t block_syms,
                                           uint32_t nb, uint64_t plen, uint64_t payload_off, uint32_t acap,
                                           uint32_t slots_per_tensor, uint32_t b) {
    in.status = status;
    in.version = (uint8_t)format;
    in.q_bits = (uint8_t)q_bits;
    in.precision = (uint8_t)precision;
    in.sym_bytes = (uint8_t)st.sym_bytes;
    in.total = total;
    in.n_rows = st.n_rows;
    in.n_cols = st.n_cols;
    in.nnz = st.nnz;
    in.scale = st.scale;
    in.zero_point = st.zero_point;
    in.alphabet = st.alphabet;
    in.lanes = format == 2 ? 32 : 1;
    in.block_syms = format == 2 ? block_syms : (uint32_t)st.stream_len;
    in.n_blocks = nb;
    in.payload_len = plen;
    in.payload_off = payload_off;
    in.freqs_off = (uint64_t)b * acap;
    in.blocks_off = (uint64_t)b * slots_per_tensor;
    in.search_flags = st.search_flags;
    in.n_evaluated = st.n_evaluated;
}

// status after the encoder's overflow / uncodable flags (rans.py:176-179)
__device__ __forceinline__ int32_t final_status(const TensorState& st, uint32_t errbits) {
    if (st.status != SCZ_OK) return st.status;
    if (errbits & 1u) return SCZ_ALPHABET_OVERFLOW;
    if (errbits & 2u) return SCZ_UNCODABLE_SYMBOL;
    return SCZ_OK;
}

// Copy len bytes src -> dst (any alignments) with one warp: bytes up to a
// 16-byte aligned destination, then 16-byte stores assembled from aligned
// 16-byte loads (funnel-shifted), then the tail.  src is a slot (padded: the
// 16 bytes after the last are readable).  Two chunks per lane in flight: at
// B = 1 this copy sits on the latency path, one L2 round trip per round.
__device__ __forceinline__ void warp_copy_bytes(uint8_t* dst, const uint8_t* src, uint32_t len, uint32_t lane) {
    uint32_t head = (uint32_t)((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15);
    head = head < len ? head : len;
    if (lane < head) dst[lane] = src[lane];
    const uint8_t* s2 = src + head;
    uint4* d2 = reinterpret_cast<uint4*>(dst + head);
    const uint32_t n16 = (len - head) >> 4;
    const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(s2) & 15);  // byte shift
    const uint4* sw = reinterpret_cast<const uint4*>(reinterpret_cast<uintptr_t>(s2) & ~(uintptr_t)15);
    // 16 bytes starting at byte sh (1..15, warp-uniform) of the pair (a, b)
    const uint32_t q = sh >> 2, r = (sh & 3) * 8;
    auto pick = [q, r](const uint4& a, const uint4& b) -> uint4 {
        switch (q) {
            case 0: return make_uint4(__funnelshift_r(a.x, a.y, r), __funnelshift_r(a.y, a.z, r),
                                      __funnelshift_r(a.z, a.w, r), __funnelshift_r(a.w, b.x, r));
            case 1: return make_uint4(__funnelshift_r(a.y, a.z, r), __funnelshift_r(a.z, a.w, r),
                                      __funnelshift_r(a.w, b.x, r), __funnelshift_r(b.x, b.y, r));
            case 2: return make_uint4(__funnelshift_r(a.z, a.w, r), __funnelshift_r(a.w, b.x, r),
                                      __funnelshift_r(b.x, b.y, r), __funnelshift_r(b.y, b.z, r));
            default: return make_uint4(__funnelshift_r(a.w, b.x, r), __funnelshift_r(b.x, b.y, r),
                                       __funnelshift_r(b.y, b.z, r), __funnelshift_r(b.z, b.w, r));
        }
    };
    for (uint32_t c0 = 0; c0 < n16; c0 += 64) {
        uint4 a[2], bb[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint32_t c = c0 + 32 * k + lane;
            if (c < n16) {
                a[k] = sw[c];
                bb[k] = sh ? sw[c + 1] : a[k];
            }
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint32_t c = c0 + 32 * k + lane;
            if (c < n16) d2[c] = sh ? pick(a[k], bb[k]) : a[k];
        }
    }
    for (uint32_t i = head + 16 * n16 + lane; i < len; i += 32) dst[i] = src[i];
}

template <typename S>
struct SplitCursor {
    const uint8_t* v;
    const S* c;
    uint32_t split;
    __device__ __forceinline__ uint32_t at(uint32_t i) const {
        return i < split ? (uint32_t)__ldg(v + i) : (uint32_t)__ldg(c + i);
    }
};
struct PlainCursor {
    const uint32_t* d;
    __device__ __forceinline__ uint32_t at(uint32_t i) const { return __ldg(d + i); }
};

template <typename S>
__device__ __forceinline__ SplitCursor<S> make_cursor(const SplitSrc<S>& src, uint32_t b, uint64_t base,
                                                      uint64_t nnz, uint32_t len) {
    SplitCursor<S> k;
    k.v = src.v8 + b * src.v8_stride + base;
    // c[i] addresses cr[base + i - nnz]; formed as an integer to allow base < nnz
    k.c = reinterpret_cast<const S*>(reinterpret_cast<uintptr_t>(src.cr + b * src.cr_stride) +
                                     (int64_t)(base - nnz) * (int64_t)sizeof(S));
    const uint64_t rest = base >= nnz ? 0 : nnz - base;
    k.split = (uint32_t)(rest < len ? rest : len);
    return k;
}
__device__ __forceinline__ PlainCursor make_cursor(const PlainSrc& src, uint32_t b, uint64_t base, uint64_t,
                                                   uint32_t) {
    return PlainCursor{src.d + b * src.stride + base};
}
struct Byte8Cursor {
    const uint8_t* d;
    __device__ __forceinline__ uint32_t at(uint32_t i) const { return __ldg(d + i); }
};
__device__ __forceinline__ Byte8Cursor make_cursor(const Contig8Src& src, uint32_t b, uint64_t base, uint64_t,
                                                   uint32_t) {
    return Byte8Cursor{src.d + b * src.stride + base};
}

struct EncLane {
    uint32_t x;
    uint32_t emitted;  // bytes emitted by the warp so far (warp-uniform)
    uint32_t err;
};

__device__ __forceinline__ void enc_apply(EncLane& L, const EncTab& t, bool live, int n, int sh_bound,
                                          uint32_t gtm, uint8_t* slot_end);

// One step for one lane.  `live` false keeps the lane idle (partial step).
template <bool SMEM, bool CHECK>
__device__ __forceinline__ void enc_step(EncLane& L, uint32_t sym, bool live, const EncTab* s_tab,
                                         const EncTab* gt, uint32_t A, int n, int sh_bound, uint32_t gtm,
                                         uint8_t* slot_end) {
    EncTab t = {1u, 0u, 0u, 0xFFFFFFFFu};
    if (CHECK) {
        if (live && sym >= A) {
            L.err |= 1u;
            live = false;
        }
    }
    if (live || !CHECK) {
        if constexpr (SMEM) {
            t = s_tab[live ? sym : 0];
        } else {
            const uint4 g = __ldg(reinterpret_cast<const uint4*>(gt) + (live ? sym : 0));
            t = EncTab{g.x, g.y, g.z, g.w};
        }
    }
    if (CHECK) {
        if (live && t.freq == 0) {
            L.err |= 2u;
            live = false;
        }
    }
    enc_apply(L, t, live, n, sh_bound, gtm, slot_end);
}

// The state transform and byte placement with the symbol's table entry given.
__device__ __forceinline__ void enc_apply(EncLane& L, const EncTab& t, bool live, int n, int sh_bound,
                                          uint32_t gtm, uint8_t* slot_end) {
    const uint32_t bound = t.freq << sh_bound;  // ((L >> n) << 8) * f
    const bool e1 = live && L.x >= bound;
    const bool e2 = live && (L.x >> 8) >= bound;
    const uint32_t b1 = __ballot_sync(0xffffffffu, e1);
    const uint32_t b2 = __ballot_sync(0xffffffffu, e2);
    const uint32_t pos = L.emitted + __popc(b1 & gtm) + __popc(b2 & gtm) + 1;
    if (e1) slot_end[-(int32_t)pos] = (uint8_t)L.x;
    if (e2) slot_end[-(int32_t)pos - 1] = (uint8_t)(L.x >> 8);
    L.emitted += __popc(b1) + __popc(b2);
    uint32_t x = L.x >> ((e1 ? 8u : 0u) + (e2 ? 8u : 0u));
    const uint32_t q = (t.shift == 0xFFFFFFFFu) ? x : (__umulhi(x, t.rcp) >> t.shift);
    x = (q << n) + t.cum + (x - q * t.freq);
    if (live) L.x = x;
}

// The u8 pipeline path's step: table entries pre-transformed at staging
// (freq -> bound = f << (31 - n), cum -> bias, shift -> shift | cmpl << 16
// with cmpl = 2^n - f; f = 1 as rcp = 2^32 - 1, shift 0, bias = cum + 2^n - 1),
// so x' = x + bias + q * cmpl with q = umulhi(x, rcp) >> shift equals
// (x / f << n) + cum + x % f (rans.py:143-144) for every f >= 1 -- three
// dependent operations on the state.  Bytes go to a per-warp shared ring
// (ob, RB bytes, same backwards order as the slot), flushed in 16-byte chunks.
constexpr uint32_t ENC_RB = 2048;
__device__ __forceinline__ EncTab enc_tab_fast(const EncTab& e, int n) {
    EncTab f;
    f.freq = e.freq << (31 - n);
    if (e.shift == 0xFFFFFFFFu) {  // f <= 1
        f.cum = e.cum + (1u << n) - 1u;
        f.rcp = 0xFFFFFFFFu;
        f.shift = ((1u << n) - 1u) << 16;
    } else {
        f.cum = e.cum;
        f.rcp = e.rcp;
        f.shift = e.shift | (((1u << n) - e.freq) << 16);
    }
    return f;
}
// obs: the warp's ring as a 32-bit shared address (plus the masked position;
// not OR'd: static shared offsets start after the reserved 1 KB, so the
// ring base is not ENC_RB-aligned in the address space).
__device__ __forceinline__ void enc_apply_ring(EncLane& L, const EncTab& t, bool live, uint32_t gtm, uint32_t obs) {
    const bool e1 = live && L.x >= t.freq;
    const bool e2 = live && (L.x >> 8) >= t.freq;  // implies e1
    const uint32_t b1 = __ballot_sync(0xffffffffu, e1);
    const uint32_t b2 = __ballot_sync(0xffffffffu, e2);
    // bytes before this lane's first: ring positions -(n + 1), -(n + 2)
    const uint32_t n = L.emitted + __popc(b1 & gtm) + __popc(b2 & gtm);
    sts_u8_if(obs + (~n & (ENC_RB - 1)), L.x, e1);
    sts_u8_if(obs + (~(n + 1) & (ENC_RB - 1)), L.x >> 8, e2);
    L.emitted += __popc(b1) + __popc(b2);
    uint32_t x = L.x;
    if (e1) x >>= 8;  // two predicated shifts (e2 implies e1)
    if (e2) x >>= 8;
    const uint32_t q = __funnelshift_r(__umulhi(x, t.rcp), 0u, t.shift);
    const uint32_t xn = x + t.cum + q * (t.shift >> 16);
    if (live) L.x = xn;
}

template <class Src, bool SMEM, bool CHECK>
__device__ __forceinline__ void enc_v2_body(const EncParams& p, const Src& src, const PackParams& pk) {
    // grid (tensor, block group): a tensor's block groups are dispatched B CTAs
    // apart, so a group's look-back predecessors started well before it, and
    // the idle groups past a tensor's block count all sit at the grid's tail
    const uint32_t b = blockIdx.x;
    TensorState& st = p.state[b];
    if (st.status != SCZ_OK) {
        if (pk.payload && pk.write_failed && blockIdx.y == 0 && threadIdx.x == 0)
            write_info(pk.info[b], st, st.status, 2, pk.q_bits, p.precision, pk.total, p.block_syms, 0, 0,
                       (uint64_t)b * pk.pcap, p.acap, p.slots_per_tensor, b);
        return;
    }
    if (Src::width && st.sym_bytes != (uint32_t)Src::width) return;  // other width variant
    const uint64_t L = st.stream_len;
    const uint32_t nblk = L ? ceil_div_u32(L, p.block_syms) : 1;
    const uint32_t blk0 = blockIdx.y * ENC2_WPB;
    if (blk0 >= nblk) return;
    extern __shared__ EncTab s_tab[];  // A entries when SMEM (host: A <= p.tab_smem)
    const uint32_t A = st.alphabet;
    const EncTab* gt = p.enctab + (uint64_t)b * p.acap;
    constexpr bool RING = std::is_same<Src, Contig8Src>::value && SMEM && !CHECK;
    if constexpr (SMEM) {
        for (uint32_t i = threadIdx.x; i < A; i += blockDim.x)
            s_tab[i] = RING ? enc_tab_fast(gt[i], p.precision) : gt[i];
        __syncthreads();
    }
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t blk = blk0 + warp;
    if (blk >= nblk) return;
    const uint64_t base = (uint64_t)blk * p.block_syms;
    const uint32_t len = (uint32_t)min((uint64_t)p.block_syms, L - base);
    const auto cur = make_cursor(src, b, base, st.nnz, len);
    const int steps = (int)((len + 31) / 32);
    const int n = p.precision, sh_bound = 31 - n;
    const uint32_t gtm = lanemask_gt();
    uint8_t* slot_end = p.slots + ((uint64_t)b * p.slots_per_tensor + blk + 1) * p.slot_cap;
    EncLane E{STATE_LOW, 0u, 0u};
    if constexpr (RING) {
        // u8 symbols staged through a per-warp 2 x 1 KB shared ring (chunk g =
        // steps [32g, 32g + 32) = block bytes [1024g, 1024g + 1024)), fetched
        // one chunk ahead with cp.async; the table entry of the next step is
        // loaded while the current one is coded.  Output bytes collect in a
        // per-warp shared ring and leave in 16-byte chunks every 16 steps.
        __shared__ __align__(16) uint8_t s_ring[ENC2_WPB][2][1024];
        __shared__ __align__(16) uint8_t s_ob[ENC2_WPB][ENC_RB];
        uint8_t* ob = s_ob[warp];
        const uint32_t obs = (uint32_t)__cvta_generic_to_shared(ob);
        uint32_t flushed = 0;  // bytes already in the slot (multiple of 16)
        auto flush = [&]() {   // every complete 16-byte chunk since the last flush
            const uint32_t upto = E.emitted & ~15u;
            for (uint32_t c = flushed + 16 * lane; c < upto; c += 512)
                *reinterpret_cast<uint4*>(slot_end - c - 16) =
                    *reinterpret_cast<const uint4*>(ob + ((0u - c - 16) & (ENC_RB - 1)));
            flushed = upto;
        };
        const uint8_t* gsym = cur.d;
        auto fetch = [&](int g) {
            if (g >= 0) {
                uint8_t* dst = s_ring[warp][g & 1] + 16 * lane;
                const uint8_t* src = gsym + (size_t)g * 1024 + 16 * lane;
                cp_async16(dst, src);
                cp_async16(dst + 512, src + 512);
            }
            cp_async_commit();
        };
        if (steps > 0) {
            const int s_top = steps - 1, g_top = s_top >> 5;
            fetch(g_top);
            fetch(g_top - 1);
            for (int g = g_top; g >= 0; --g) {
                cp_async_wait<1>();
                __syncwarp();
                const uint8_t* rs = s_ring[warp][g & 1] + lane;
#pragma unroll 1
                for (int h = 1; h >= 0; --h) {  // half-chunks of 16 steps
                    const int lo = g * 32 + 16 * h;
                    int s = min(lo + 15, s_top);
                    if (s < lo) continue;
                    EncTab t;
                    if (s == s_top) {  // the highest step may be partial
                        const bool act = (uint32_t)s * 32 + lane < len;
                        t = s_tab[act ? rs[(s & 31) * 32] : 0];
                        enc_apply_ring(E, t, act, gtm, obs);
                        --s;
                    }
                    // groups of four steps: the four table entries are loaded
                    // up front (symbols do not depend on the state)
#pragma unroll 1
                    for (; s - 3 >= lo; s -= 4) {
                        // s - 3 .. s lie in one half-chunk: no wrap, one base
                        const uint8_t* rp = rs + (s & 31) * 32;
                        const EncTab t0 = s_tab[rp[0]];
                        const EncTab t1 = s_tab[rp[-32]];
                        const EncTab t2 = s_tab[rp[-64]];
                        const EncTab t3 = s_tab[rp[-96]];
                        enc_apply_ring(E, t0, true, gtm, obs);
                        enc_apply_ring(E, t1, true, gtm, obs);
                        enc_apply_ring(E, t2, true, gtm, obs);
                        enc_apply_ring(E, t3, true, gtm, obs);
                    }
                    for (; s >= lo; --s) enc_apply_ring(E, s_tab[rs[(s & 31) * 32]], true, gtm, obs);
                    __syncwarp();
                    flush();
                }
                __syncwarp();
                fetch(g - 2);
            }
        }
        cp_async_wait<0>();
        // the last partial chunk, byte by byte
        const uint32_t k = flushed + lane;
        if (k < E.emitted) slot_end[-(int32_t)k - 1] = ob[(0u - k - 1) & (ENC_RB - 1)];
    } else if (steps > 0) {
        // the highest step may be partial: peel it
        const int s_top = steps - 1;
        const uint32_t i_top = (uint32_t)s_top * 32 + lane;
        const bool act = i_top < len;
        // queue of the next 8 (full) steps' symbols: q[k] = step s_top - 1 - k
        uint32_t q[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int s = s_top - 1 - k;
            q[k] = s >= 0 ? cur.at((uint32_t)s * 32 + lane) : 0u;
        }
        enc_step<SMEM, CHECK>(E, act ? cur.at(i_top) : 0u, act, s_tab, gt, A, n, sh_bound, gtm, slot_end);
        int s0 = s_top - 1;  // next step to code; q[k] holds step s0 - k
        for (; s0 >= 7; s0 -= 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t sym = q[k];
                const int sp = s0 - k - 8;  // clamped: a harmless in-block load when sp < 0
                q[k] = cur.at((uint32_t)max(sp, 0) * 32 + lane);
                enc_step<SMEM, CHECK>(E, sym, true, s_tab, gt, A, n, sh_bound, gtm, slot_end);
            }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k <= s0) enc_step<SMEM, CHECK>(E, q[k], true, s_tab, gt, A, n, sh_bound, gtm, slot_end);
    }
    // block bytes: 32 little-endian states, then the emitted bytes (decoder order)
    const uint32_t blen = 4 * 32 + E.emitted;
    uint8_t* start = slot_end - blen;
    start[4 * lane + 0] = (uint8_t)E.x;
    start[4 * lane + 1] = (uint8_t)(E.x >> 8);
    start[4 * lane + 2] = (uint8_t)(E.x >> 16);
    start[4 * lane + 3] = (uint8_t)(E.x >> 24);
    if (CHECK) E.err = __reduce_or_sync(0xffffffffu, E.err);
    if (lane == 0) {
        p.block_len[(uint64_t)b * p.slots_per_tensor + blk] = blen;
        if (CHECK && E.err) atomicOr(&st.errbits, E.err);
    }
    if (pk.payload) {
        __threadfence();  // error bits before the length is published
        __syncwarp();     // the slot bytes of every lane are visible to the warp
        const uint32_t excl = chunk_prefix(pk.lb + (uint64_t)b * p.slots_per_tensor, blk, blen);
        warp_copy_bytes(pk.payload + (uint64_t)b * pk.pcap + excl, start, blen, lane);
        if (blk == nblk - 1 && lane == 0) {
            __threadfence();  // every block published: their error bits are visible
            const uint32_t eb = *(volatile uint32_t*)&st.errbits;
            write_info(pk.info[b], st, final_status(st, eb), 2, pk.q_bits, p.precision, pk.total, p.block_syms,
                       nblk, (uint64_t)excl + blen, (uint64_t)b * pk.pcap, p.acap, p.slots_per_tensor, b);
        }
    }
}

template <class Src, bool SMEM, bool CHECK>
__global__ void __launch_bounds__(ENC2_WPB * 32) k_rans_enc_v2(EncParams p, Src src, PackParams pk) {
    pdl_wait();
    enc_v2_body<Src, SMEM, CHECK>(p, src, pk);
}

// The pipeline's launch: u8 and u16 symbol classes in one grid (a tensor's
// class is known only after k_select), so no launch is spent on an empty
// class.  u32 tensors (K > 65535) go to k_rans_enc_v2<SplitSrc<uint32_t>>.
template <bool SMEM>
__global__ void __launch_bounds__(ENC2_WPB * 32, 10)
    k_rans_enc_v2_u8u16(EncParams p, Contig8Src s8, SplitSrc<uint16_t> s16, PackParams pk) {
    pdl_wait();
    const TensorState& st = p.state[blockIdx.x];
    if (st.status == SCZ_OK && st.sym_bytes == 2) enc_v2_body<SplitSrc<uint16_t>, SMEM, false>(p, s16, pk);
    else enc_v2_body<Contig8Src, SMEM, false>(p, s8, pk);  // also writes failed tensors' headers
}
template __global__ void k_rans_enc_v2_u8u16<true>(EncParams, Contig8Src, SplitSrc<uint16_t>, PackParams);
template __global__ void k_rans_enc_v2_u8u16<false>(EncParams, Contig8Src, SplitSrc<uint16_t>, PackParams);

#define SCZ_INST_ENC2(SRC, CHK)                                                              \
    template __global__ void k_rans_enc_v2<SRC, true, CHK>(EncParams, SRC, PackParams);     \
    template __global__ void k_rans_enc_v2<SRC, false, CHK>(EncParams, SRC, PackParams);
SCZ_INST_ENC2(Contig8Src, false)
SCZ_INST_ENC2(SplitSrc<uint8_t>, false)
SCZ_INST_ENC2(SplitSrc<uint16_t>, false)
SCZ_INST_ENC2(SplitSrc<uint32_t>, false)
SCZ_INST_ENC2(PlainSrc, true)

}  // namespace scz
