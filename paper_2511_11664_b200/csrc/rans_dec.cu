// rans_dec.cu -- v2 interleaved-lane rANS decoder (K7).
//
// One warp decodes one FORMAT.md v2 block; lane j owns state j.  Per step:
//   slot = x & (2^n - 1);  sym = LUT[slot];  (f, cum) = tab[sym]
//   x = f * (x >> n) + slot - cum                      (rans.py:147-152)
// then every lane's refill count (2 if x < 2^15, 1 if x < 2^23) is placed by
// one ballot-scan and the bytes come from a per-warp ring in shared memory.
// The ring is fed by cp.async copies issued 2-4 chunks ahead, so global
// latency never sits on the state recurrence.  All in-loop addressing is
// 32-bit; the slot LUT (u8/u16) and the table are shared by the CTA's warps.
#include "common.cuh"

namespace scz {

constexpr uint32_t SMALL_ROWS_DEC = 2048;  // == SMALL_ROWS (decode.cu)
constexpr int DEC2_WPB = 16;         // warps (= blocks) per CTA, throughput mode
constexpr int DEC2_WPB_SMALL = 4;    // latency mode (grid would not fill the GPU)
constexpr int DCHUNK = 256;          // bytes per cp.async chunk (8 per lane)
constexpr int DRING = 4 * DCHUNK;    // per-warp ring
constexpr int DRING_STRIDE = DRING + 16;  // + a mirror of the ring's first 8 bytes (no wrap on the 2nd word)
constexpr uint32_t DEC_BIG_F = 256;  // symbols with more slots are filled CTA-wide

// Shared-memory layout (LUT classes, L = u8 / u16):
//   rings  [WPB][DRING + 16] bytes (bytes DRING.. mirror bytes 0..7)
//   step   [2^n] u32 (f << 16) | (slot - cum): the state update in one load
//   sym    [2^n] L   slot -> symbol (off the state recurrence)
// The two tables are built once per tensor by k_dec_prepare and arrive with
// one bulk copy (TMA) while the payload ring is being primed.
template <typename S, typename L, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_rans_dec_v2(DecParams p) {
    pdl_wait();
    const uint32_t b = blockIdx.y;
    const scz_info& in = p.info[b];
    if (p.status[b] != SCZ_OK || in.version != 2 || in.sym_bytes != sizeof(S)) return;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t s_bar;
    const uint32_t A = in.alphabet;
    const int n = in.precision;
    const uint32_t nslots = 1u << n;
    const uint32_t* gf = p.freqs + in.freqs_off;
    const uint32_t* gcum = p.cumtab + (uint64_t)b * (p.acap + 1);
    const uint32_t blk0 = blockIdx.x * WPB;
    if (blk0 >= in.n_blocks) return;  // whole CTA idle
    uint8_t* rings = smem;
    uint32_t* lstep = reinterpret_cast<uint32_t*>(smem + WPB * DRING_STRIDE);
    const L* lsym = reinterpret_cast<const L*>(reinterpret_cast<const uint8_t*>(lstep) + lut_sym_off(n));
    if constexpr (sizeof(L) < 4) {
        if (threadIdx.x == 0) {
            mbar_init(&s_bar, 1);
            const uint32_t bytes = (lut_sym_off(n) + nslots * (uint32_t)sizeof(L) + 15u) & ~15u;
            mbar_expect_tx(&s_bar, bytes);
            bulk_g2s(lstep, p.lut + (uint64_t)b * p.lut_stride, bytes, &s_bar);
        }
        __syncthreads();  // s_bar initialised before any warp polls it
    }
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t blk = blk0 + warp;
    if (blk >= in.n_blocks) return;
    const uint64_t Ls = 2 * in.nnz + in.n_rows;
    const uint64_t base = (uint64_t)blk * in.block_syms;
    const uint32_t len = (uint32_t)min((uint64_t)in.block_syms, Ls - base);
    const uint32_t blen = p.block_bytes[in.blocks_off + blk];
    const uint64_t a0 = in.payload_off + p.blk_off[(uint64_t)b * p.nblk_cap + blk];
    const uint64_t cbase = a0 & ~(uint64_t)(DCHUNK - 1);
    const uint8_t* gsrc = p.payload + cbase + 8 * lane;
    uint8_t* ring = rings + warp * DRING_STRIDE;
    uint8_t* rdst = ring + 8 * lane;
    uint32_t cur = (uint32_t)(a0 - cbase);  // byte offset from cbase
    const uint32_t end = cur + blen;
    // chunk c (bytes [256c, 256c + 256) from cbase) lives in ring slot c & 3;
    // chunks starting at or beyond `end` are never fetched (a 256-aligned
    // chunk holding a valid byte never leaves that byte's allocation)
    auto fetch = [&](uint32_t c) {
        if (c * DCHUNK < end) {
            cp_async8(rdst + (c & 3) * DCHUNK, gsrc + (size_t)c * DCHUNK);
            if ((c & 3) == 0 && lane == 0) cp_async8(ring + DRING, gsrc + (size_t)c * DCHUNK);  // mirror
        }
        cp_async_commit();
    };
    fetch(0);
    fetch(1);
    fetch(2);
    fetch(3);
    cp_async_wait<2>();  // chunks 0 and 1 landed
    __syncwarp();
    auto rb = [&](uint32_t a) -> uint32_t { return ring[a & (DRING - 1)]; };
    uint32_t x = rb(cur + 4 * lane) | (rb(cur + 4 * lane + 1) << 8) | (rb(cur + 4 * lane + 2) << 16) |
                 (rb(cur + 4 * lane + 3) << 24);
    cur += 128;
    uint32_t k = 0;  // chunk holding `cur`; chunks <= k + 1 have landed
    // A step consumes <= 64 bytes, so four steps stay inside chunks k, k + 1
    // (landed) and cross at most one chunk boundary: the ring is advanced
    // once per four steps, keeping the branch off three of four recurrences.
    auto advance = [&]() {
        if ((cur >> 8) != k) {  // warp-uniform, taken about once per 7 steps
            __syncwarp();
            ++k;
            fetch(k + 3);
            cp_async_wait<2>();
            __syncwarp();
        }
    };
    advance();
    if constexpr (sizeof(L) < 4) mbar_wait(&s_bar, 0);
    const uint32_t mask = nslots - 1;
    const uint32_t ltm = lanemask_lt();
    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
    S* out = reinterpret_cast<S*>(reinterpret_cast<uint8_t*>(p.dsym) + (uint64_t)b * p.dsym_stride) + base + lane;
    const uint32_t steps = (len + 31) / 32;
    // One step: pop the lane's symbol (rans.py:147-152) and refill.  A
    // stream that runs past its block end keeps decoding ring garbage and is
    // rejected by the final cur == end check (rans.py:203-205 underrun).
    auto step = [&](bool active) -> uint32_t {
        uint32_t sym = 0;
        bool p1 = false, p2 = false;  // refill 1 byte (x < 2^23) / 2 bytes (x < 2^15)
        if (active) {
            const uint32_t slot = x & mask;
            if constexpr (sizeof(L) < 4) {
                const uint32_t e = lstep[slot];
                sym = lsym[slot];
                x = (e >> 16) * (x >> n) + (e & 0xffffu);
            } else {
                uint32_t lo = 0, hi = A + 1;  // np.searchsorted(cdf, slot, 'right') - 1
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (gcum[mid] <= slot) lo = mid;
                    else hi = mid;
                }
                sym = lo;
                x = gf[sym] * (x >> n) + slot - gcum[sym];
            }
            p1 = x < STATE_LOW;
            p2 = x < (1u << 15);
        }
        const uint32_t b1 = __ballot_sync(0xffffffffu, p1);
        const uint32_t b2 = __ballot_sync(0xffffffffu, p2);
        const uint32_t a = cur + __popc(b1 & ltm) + __popc(b2 & ltm);
        // bytes a, a + 1 from two aligned words (the second one may be the
        // mirror past the ring's end); PRMT shifts them into x
        const uint32_t wa = ring_s + (a & (DRING - 4));
        const uint32_t w0 = lds_u32(wa);
        const uint32_t w1 = lds_u32(wa + 4);
        const uint32_t v = __funnelshift_r(w0, w1, a * 8);  // the shift is taken mod 32
        const uint32_t sel = p2 ? 0x1045u : (p1 ? 0x2104u : 0x3210u);
        x = __byte_perm(x, v, sel);
        cur += __popc(b1) + __popc(b2);
        return sym;
    };
    if constexpr (sizeof(S) == 1) {
        // u8 symbols collect in a per-warp 16-step shared buffer and leave
        // with one 16-byte store per lane (instead of a byte store per step)
        __shared__ __align__(16) uint8_t s_sym[WPB][16 * 32];
        uint8_t* ob = s_sym[warp];
        uint8_t* gout = reinterpret_cast<uint8_t*>(p.dsym) + (uint64_t)b * p.dsym_stride + base;  // 16-aligned
        const uint32_t full = len / 32;
        uint32_t s = 0;
        for (; s + 16 <= full; s += 16) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
#pragma unroll
                for (int u = 0; u < 4; ++u) ob[(4 * q + u) * 32 + lane] = (uint8_t)step(true);
                advance();
            }
            __syncwarp();
            *reinterpret_cast<uint4*>(gout + (size_t)s * 32 + 16 * lane) =
                *reinterpret_cast<const uint4*>(ob + 16 * lane);
            __syncwarp();
        }
        for (uint32_t j = s; j < steps; ++j) {
            const bool act = j * 32 + lane < len;  // only the last step can be partial
            const uint32_t sym = step(act);
            if (act) ob[(j - s) * 32 + lane] = (uint8_t)sym;
            if (j < full) advance();
        }
        __syncwarp();
        const uint32_t rem = len - s * 32;  // symbols still in the buffer (< 512)
        for (uint32_t i = lane; i < rem; i += 32) gout[(size_t)s * 32 + i] = ob[i];
        __syncwarp();
    } else if (steps > 0) {
        const uint32_t full = len / 32;
        uint32_t s = 0;
        for (; s + 4 <= full; s += 4) {
            *out = (S)step(true); out += 32;
            *out = (S)step(true); out += 32;
            *out = (S)step(true); out += 32;
            *out = (S)step(true); out += 32;
            advance();
        }
        for (; s < full; ++s) {
            *out = (S)step(true); out += 32;
            advance();
        }
        if (full < steps) {  // partial last step
            const bool act = full * 32 + lane < len;
            const uint32_t sym = step(act);
            if (act) *out = (S)sym;
        }
    }
    cp_async_wait<0>();
    // Row-count sums per SMALL_ROWS-row chunk for k_rows_small8 (u8, K in
    // {1, 2, 4}): the block's symbols in the r segment [2 nnz, 2 nnz + N)
    // are re-read (just written by this warp) and added per chunk.
    if (sizeof(S) == 1 && p.chunk_sums && (in.n_cols == 1 || in.n_cols == 2 || in.n_cols == 4)) {
        const uint64_t r0 = 2 * in.nnz;
        const uint64_t lo = max(base, r0), hi = base + len;
        if (lo < hi) {
            __syncwarp();  // every lane's symbol stores are visible to the warp
            const uint8_t* d8 = reinterpret_cast<const uint8_t*>(p.dsym) + (uint64_t)b * p.dsym_stride;
            unsigned long long* cs = p.chunk_state + (uint64_t)b * p.nchunk_cap;
            for (uint64_t c = (lo - r0) / SMALL_ROWS_DEC; r0 + c * SMALL_ROWS_DEC < hi; ++c) {
                const uint64_t a = max(lo, r0 + c * SMALL_ROWS_DEC);
                const uint64_t e = min(hi, r0 + (c + 1) * SMALL_ROWS_DEC);
                uint32_t acc = 0;
                // aligned words covering [a, e), bytes outside masked off
                for (uint64_t w = (a >> 2) + lane; w <= ((e - 1) >> 2); w += 32) {
                    uint32_t v = reinterpret_cast<const uint32_t*>(d8)[w];
                    const uint64_t wb = w << 2;
                    if (wb < a) v &= 0xFFFFFFFFu << (8 * (uint32_t)(a - wb));
                    if (wb + 4 > e) v &= 0xFFFFFFFFu >> (8 * (uint32_t)(wb + 4 - e));
                    acc = __dp4a(v, 0x01010101u, acc);
                }
                acc = warp_sum(acc);
                if (lane == 0 && acc) atomicAdd(cs + c, (unsigned long long)acc);
            }
        }
    }
    // rans.py:211-212: every lane back at L and every byte consumed
    const bool bad = __any_sync(0xffffffffu, x != STATE_LOW) || cur != end;
    if (bad && lane == 0) p.status[b] = SCZ_CORRUPT_STREAM;
}

#define SCZ_DEC2(S, L)                                                      \
    template __global__ void k_rans_dec_v2<S, L, DEC2_WPB>(DecParams);       \
    template __global__ void k_rans_dec_v2<S, L, DEC2_WPB_SMALL>(DecParams);
SCZ_DEC2(uint8_t, uint8_t)
SCZ_DEC2(uint16_t, uint16_t)
SCZ_DEC2(uint32_t, uint32_t)
#undef SCZ_DEC2

// dynamic shared memory of k_rans_dec_v2 for a batch (max over tensors)
inline size_t dec_v2_smem(int wpb, size_t lwidth, int n, uint32_t) {
    size_t s = (size_t)wpb * DRING_STRIDE;
    if (lwidth < 4) s += ((((size_t)1 << n) * (4 + lwidth)) + 15) & ~(size_t)15;
    return (s + 15) & ~(size_t)15;
}

}  // namespace scz
