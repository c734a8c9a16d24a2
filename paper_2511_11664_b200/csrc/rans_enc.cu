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
#ifdef SCZ_ENC_PROBE
// diagnostics build: %globaltimer stamps per block (first 512 blocks of
// tensor 0): start, table staged, coded, looked back, copied, done
__device__ unsigned long long g_enc_probe[512][8];
#define ENC_STAMP(blk, i)                                                                      \
    do {                                                                                       \
        if ((threadIdx.x & 31) == 0 && blockIdx.x == 0 && (blk) < 512) {                       \
            unsigned long long t_;                                                            \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
            g_enc_probe[(blk)][(i)] = t_;                                                     \
        }                                                                                      \
    } while (0)
#else
#define ENC_STAMP(blk, i) do { } while (0)
#endif
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
#ifndef SCZ_COPY_K
#define SCZ_COPY_K 2
#endif
    constexpr int CK_ = SCZ_COPY_K;  // chunks per lane in flight
    for (uint32_t c0 = 0; c0 < n16; c0 += 32 * CK_) {
        uint4 a[CK_], bb[CK_];
#pragma unroll
        for (int k = 0; k < CK_; ++k) {
            const uint32_t c = c0 + 32 * k + lane;
            if (c < n16) {
                a[k] = sw[c];
                bb[k] = sh ? sw[c + 1] : a[k];
            }
        }
#pragma unroll
        for (int k = 0; k < CK_; ++k) {
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
// dependent operations on the state.
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
// The u8 pipeline path (RING): symbols staged per warp in shared memory by
// cp.async, three 1 KB chunks (32 steps each) in flight ahead of the coder;
// table entries of the next four steps loaded while the current four are
// coded; emitted bytes go DOWN a per-warp 2 KB shared window from its top
// (the byte of warp-order position k of a step lands at base - 1 - k, so the
// window holds the bytes already in decoder order) and leave in 16-byte
// chunks every 16 steps, after which the < 16 leftover bytes move back to the
// top.  No address masking in the step: position = base - (bytes of the
// higher lanes), one IADD3; the second byte's store has an immediate offset.
constexpr uint32_t ENC_OB = 2048;    // output window per warp (16 steps emit <= 1024 bytes)
constexpr uint32_t ENC_SCH = 1024;   // symbol chunk: 32 steps x 32 lanes
constexpr int ENC_NSCH = 3;          // symbol chunks per warp (two in flight ahead)

template <bool PRED>
__device__ __forceinline__ void enc_step_lin(uint32_t& x, uint32_t& base, const EncTab& t, uint32_t gtm,
                                             bool live) {
    const uint32_t x8 = x >> 8;
    const bool e1 = (!PRED || live) && x >= t.freq;   // t.freq holds the bound f << (31 - n)
    const bool e2 = (!PRED || live) && x8 >= t.freq;  // implies e1
    const uint32_t b1 = __ballot_sync(0xffffffffu, e1);
    const uint32_t b2 = __ballot_sync(0xffffffffu, e2);
    const uint32_t pos = base - __popc(b1 & gtm) - __popc(b2 & gtm);
    asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.shared.u8 [%0+-1], %1;\n}\n" ::"r"(pos), "r"(x),
                 "r"((uint32_t)e1)
                 : "memory");
    asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.shared.u8 [%0+-2], %1;\n}\n" ::"r"(pos), "r"(x8),
                 "r"((uint32_t)e2)
                 : "memory");
    base -= __popc(b1) + __popc(b2);
    uint32_t xs = e1 ? x8 : x;
    if (e2) xs >>= 8;
    const uint32_t q = __funnelshift_r(__umulhi(xs, t.rcp), 0u, t.shift);
    const uint32_t xn = q * (t.shift >> 16) + (xs + t.cum);
    x = (!PRED || live) ? xn : x;
}

__device__ __forceinline__ EncTab lds_tab16(uint32_t saddr) {
    EncTab t;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(t.freq), "=r"(t.cum), "=r"(t.rcp), "=r"(t.shift)
                 : "r"(saddr));
    return t;
}

__device__ __forceinline__ void enc_v2_ring(EncLane& E, const uint8_t* gsym, uint32_t len, int steps,
                                            const EncTab* s_tab, uint8_t* slot_end, uint32_t warp, uint32_t lane,
                                            uint32_t gtm) {
    __shared__ __align__(16) uint8_t s_sym[ENC2_WPB][ENC_NSCH][ENC_SCH];
    __shared__ __align__(16) uint8_t s_ob[ENC2_WPB][ENC_OB];
    // shared addresses pinned in registers (opaque copies: otherwise the
    // compiler re-derives the shared window base, S2R included, per load)
    const uint32_t tab_s = opaque_u32(smem_u32(s_tab));
    const uint32_t ob_s = opaque_u32(smem_u32(s_ob[warp]));
    const uint32_t top = ob_s + ENC_OB;
    const uint32_t sym_s = opaque_u32(smem_u32(s_sym[warp][0]) + lane);
    uint32_t base = top;   // window bytes [base, rtop) are pending
    uint32_t rtop = top;   // [rtop, top) already went to the slot
    uint32_t flushed = 0;  // bytes already in the slot (multiple of 16)
    // the window is flushed (at a 16-step boundary) only once less than one
    // interval's worst case (16 steps x 32 lanes x 2 bytes) is left below base
    const uint32_t low = ob_s + 1024;
    uint32_t x = E.x;
    // window byte at address a goes to slot_end - flushed - (rtop - a): the
    // complete 16-byte chunks below rtop leave; when less than one flush
    // interval (16 steps, <= 1024 bytes) of room is left below base, the
    // < 16 leftover bytes move up to the top
    auto flush = [&]() {
        __syncwarp();
        const uint32_t nfl = (rtop - base) & ~15u;
        for (uint32_t c = 16 * lane; c < nfl; c += 512) {
            uint4 v;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "r"(rtop - c - 16)
                         : "memory");
            *reinterpret_cast<uint4*>(slot_end - flushed - c - 16) = v;
        }
        flushed += nfl;
        rtop -= nfl;
        if (base < ob_s + 1024) {
            const uint32_t rem = rtop - base;
            const uint32_t v = lane < rem ? lds_u8(base + lane) : 0u;
            __syncwarp();
            if (lane < rem) sts_u8_if(top - rem + lane, v, true);
            rtop = top;
            base = top - rem;
        }
        __syncwarp();
    };
    auto fetch = [&](int g) {
        if (g >= 0) {
            uint8_t* dst = s_sym[warp][g % ENC_NSCH] + 16 * lane;
            const uint8_t* src = gsym + (size_t)g * ENC_SCH + 16 * lane;
            cp_async16(dst, src);
            cp_async16(dst + 512, src + 512);
        }
        cp_async_commit();
    };
    if (steps > 0) {
        int cg = (steps - 1) >> 5;  // chunk being read (landed)
        fetch(cg);
        fetch(cg - 1);
        fetch(cg - 2);
        cp_async_wait<2>();
        __syncwarp();
        uint32_t symc = sym_s + (uint32_t)(cg % ENC_NSCH) * ENC_SCH;
        // chunk of step s: leaving chunk cg frees its slot for chunk cg - 3
        auto ensure = [&](int s) {
            if ((s >> 5) != cg) {
                __syncwarp();
                fetch(cg - 3);
                --cg;
                cp_async_wait<2>();
                __syncwarp();
                symc = sym_s + (uint32_t)(cg % ENC_NSCH) * ENC_SCH;
            }
        };
        auto sym_at = [&](int s) -> uint32_t { return symc + (uint32_t)(s & 31) * 32; };
        int s = steps - 1;
        if (len & 31u) {  // the highest step of the tensor's last block is partial
            const bool act = (uint32_t)s * 32 + lane < len;
            const EncTab t = lds_tab16(tab_s + 16 * (act ? lds_u8(sym_at(s)) : 0u));
            enc_step_lin<true>(x, base, t, gtm, act);
            if ((s & 15) == 0 && base < low) flush();
            --s;
        }
        for (; s >= 0 && (s & 31) != 31; --s) {  // align the rest to whole 32-step symbol chunks
            ensure(s);
            enc_step_lin<false>(x, base, lds_tab16(tab_s + 16 * lds_u8(sym_at(s))), gtm, true);
            if ((s & 15) == 0 && base < low) flush();
        }
        // groups of sixteen steps (s = 15 mod 16: never across a 32-step
        // symbol chunk; a flush boundary only at the end), four table entries
        // in flight: entry k of the next quarter loads right after step k of
        // this one used its registers, four steps ahead of its use.  The
        // successors of the first three quarters share the chunk of s, so
        // only the last quarter checks for a chunk change.
        if (s >= 31) {
            ensure(s);
            const uint32_t a = sym_at(s);
            uint32_t y0 = lds_u8(a), y1 = lds_u8(a - 32), y2 = lds_u8(a - 64), y3 = lds_u8(a - 96);
            EncTab t0 = lds_tab16(tab_s + 16 * y0), t1 = lds_tab16(tab_s + 16 * y1);
            EncTab t2 = lds_tab16(tab_s + 16 * y2), t3 = lds_tab16(tab_s + 16 * y3);
            auto quarter = [&]() {
                enc_step_lin<false>(x, base, t0, gtm, true);
                t0 = lds_tab16(tab_s + 16 * y0);
                enc_step_lin<false>(x, base, t1, gtm, true);
                t1 = lds_tab16(tab_s + 16 * y1);
                enc_step_lin<false>(x, base, t2, gtm, true);
                t2 = lds_tab16(tab_s + 16 * y2);
                enc_step_lin<false>(x, base, t3, gtm, true);
                t3 = lds_tab16(tab_s + 16 * y3);
            };
            auto load_y = [&](uint32_t an) {
                y0 = lds_u8(an);
                y1 = lds_u8(an - 32);
                y2 = lds_u8(an - 64);
                y3 = lds_u8(an - 96);
            };
#pragma unroll 1
            for (;;) {
                load_y(sym_at(s - 4));
                quarter();
                load_y(sym_at(s - 8));
                quarter();
                load_y(sym_at(s - 12));
                quarter();
                load_y(sym_at(s - 16));
                quarter();
                if (base < low) flush();  // s - 15 = 0 mod 16
                load_y(sym_at(s - 20));
                quarter();
                load_y(sym_at(s - 24));
                quarter();
                load_y(sym_at(s - 28));
                quarter();
                const int sn = s - 32;
                const bool more = sn >= 31;
                if (more) {
                    ensure(sn);
                    load_y(sym_at(sn));
                }
                // unconditional: after the last group these reload entries
                // of the last symbols (harmless, unused)
                quarter();
                if (base < low) flush();  // s - 31 = 0 mod 32
                s = sn;
                if (!more) break;
            }
        }
    }
    cp_async_wait<0>();
    flush();  // every complete 16-byte chunk
    // the last (< 16) bytes, then the emitted count
    const uint32_t pend = rtop - base;
    if (lane < pend) slot_end[-(int32_t)(flushed + pend) + (int32_t)lane] = (uint8_t)lds_u8(base + lane);
    E.emitted = flushed + pend;
    E.x = x;
}

// The block's bytes -- 32 little-endian states, then the emitted bytes in
// decoder order -- end at slot_end; publish the length, find the block's
// payload offset by decoupled look-back, copy it there, drop the slot's L2
// lines, and (last block) write the tensor's header.
template <bool CHECK>
__device__ __forceinline__ void enc_v2_block_tail(const EncParams& p, const PackParams& pk, TensorState& st,
                                                  uint32_t b, uint32_t blk, uint32_t nblk, uint8_t* slot_end,
                                                  EncLane E, uint32_t lane) {
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
        ENC_STAMP(blk, 3);
        const uint32_t excl = chunk_prefix(pk.lb + (uint64_t)b * p.slots_per_tensor, blk, blen);
        ENC_STAMP(blk, 4);
        warp_copy_bytes(pk.payload + (uint64_t)b * pk.pcap + excl, start, blen, lane);
        ENC_STAMP(blk, 5);
        // the slot is dead now: drop its L2 lines without a write-back to HBM
        // (slots are 128-byte aligned; the lines below `start` hold only this
        // slot's unused head)
        __syncwarp();
        for (uintptr_t a = (reinterpret_cast<uintptr_t>(start) & ~(uintptr_t)127) + 128 * lane;
             a < reinterpret_cast<uintptr_t>(slot_end); a += 128 * 32)
            asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(a) : "memory");
        ENC_STAMP(blk, 6);
        if (blk == nblk - 1 && lane == 0) {
            __threadfence();  // every block published: their error bits are visible
            const uint32_t eb = *(volatile uint32_t*)&st.errbits;
            write_info(pk.info[b], st, final_status(st, eb), 2, pk.q_bits, p.precision, pk.total, p.block_syms,
                       nblk, (uint64_t)excl + blen, (uint64_t)b * pk.pcap, p.acap, p.slots_per_tensor, b);
        }
    }
}

template <class Src, bool SMEM, bool CHECK>
__device__ __forceinline__ void enc_v2_body(const EncParams& p, const Src& src, const PackParams& pk) {
    // grid (tensor, block group): a tensor's block groups are dispatched B CTAs
    // apart, so a group's look-back predecessors started well before it, and
    // the idle groups past a tensor's block count all sit at the grid's tail
    const uint32_t b = blockIdx.x;
    ENC_STAMP(blockIdx.y * ENC2_WPB + (threadIdx.x >> 5), 0);
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
        ENC_STAMP(blk, 1);
        enc_v2_ring(E, cur.d, len, steps, s_tab, slot_end, warp, lane, gtm);
        ENC_STAMP(blk, 2);
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
    enc_v2_block_tail<CHECK>(p, pk, st, b, blk, nblk, slot_end, E, lane);
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
#ifndef SCZ_ENC2_MINB
#define SCZ_ENC2_MINB 8
#endif
__global__ void __launch_bounds__(ENC2_WPB * 32, SCZ_ENC2_MINB)
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
