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

constexpr int DEC2_WPB = 16;         // warps (= blocks) per CTA
constexpr int DCHUNK = 256;          // bytes per cp.async chunk (8 per lane)
constexpr int DRING = 4 * DCHUNK;    // per-warp ring

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <typename S, typename L>
__global__ void __launch_bounds__(DEC2_WPB * 32) k_rans_dec_v2(DecParams p) {
    const uint32_t b = blockIdx.y;
    const scz_info& in = p.info[b];
    if (p.status[b] != SCZ_OK || in.version != 2 || in.sym_bytes != sizeof(S)) return;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t A = in.alphabet;
    const int n = in.precision;
    const uint32_t nslots = 1u << n;
    const uint32_t* gf = p.freqs + in.freqs_off;
    const uint32_t* gcum = p.cumtab + (uint64_t)b * (p.acap + 1);
    const uint32_t blk0 = blockIdx.x * DEC2_WPB;
    if (blk0 >= in.n_blocks) return;  // whole CTA idle
    uint8_t* rings = smem;
    // classes (dec_class): u8/u16 LUT with the (f, cum) table in smem, or
    // binary search over the cdf in global memory for huge alphabets / n = 16
    uint2* tab = reinterpret_cast<uint2*>(smem + DEC2_WPB * DRING);   // A entries
    L* lut = reinterpret_cast<L*>(tab + A);                            // 2^n entries
    if constexpr (sizeof(L) < 4) {
        for (uint32_t i = threadIdx.x; i < A; i += blockDim.x) tab[i] = make_uint2(gf[i], gcum[i]);
        __syncthreads();
        // warp w writes the slot ranges of symbols w, w + nw, ... (coalesced)
        const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (uint32_t s = warp; s < A; s += nw) {
            const uint32_t c0 = tab[s].y, c1 = c0 + tab[s].x;
            for (uint32_t sl = c0 + lane; sl < c1; sl += 32) lut[sl] = (L)s;
        }
        __syncthreads();
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
    uint8_t* ring = rings + warp * DRING;
    uint8_t* rdst = ring + 8 * lane;
    // chunk c (absolute offset 256c from cbase) lives in ring slot c & 3
    cp_async8(rdst + 0 * DCHUNK, gsrc + 0 * DCHUNK); cp_async_commit();
    cp_async8(rdst + 1 * DCHUNK, gsrc + 1 * DCHUNK); cp_async_commit();
    cp_async8(rdst + 2 * DCHUNK, gsrc + 2 * DCHUNK); cp_async_commit();
    cp_async8(rdst + 3 * DCHUNK, gsrc + 3 * DCHUNK); cp_async_commit();
    cp_async_wait<2>();  // chunks 0 and 1 landed
    __syncwarp();
    uint32_t cur = (uint32_t)(a0 - cbase);  // byte offset from cbase
    const uint32_t end = cur + blen;
    auto rb = [&](uint32_t a) -> uint32_t { return ring[a & (DRING - 1)]; };
    uint32_t x = rb(cur + 4 * lane) | (rb(cur + 4 * lane + 1) << 8) | (rb(cur + 4 * lane + 2) << 16) |
                 (rb(cur + 4 * lane + 3) << 24);
    cur += 128;
    uint32_t k = 0;  // chunk holding `cur`; chunks <= k + 1 have landed
    // a step consumes <= 64 bytes < one chunk, so at most one chunk boundary
    auto advance = [&]() {
        if ((cur >> 8) != k) {  // warp-uniform, taken about once per 7 steps
            __syncwarp();
            ++k;
            cp_async8(rdst + ((k + 3) & 3) * DCHUNK, gsrc + (k + 3) * DCHUNK);
            cp_async_commit();
            cp_async_wait<2>();
            __syncwarp();
        }
    };
    advance();
    const uint32_t mask = nslots - 1;
    const uint32_t ltm = lanemask_lt();
    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
    S* out = reinterpret_cast<S*>(p.dsym) + (uint64_t)b * p.dsym_stride + base + lane;
    const uint32_t steps = (len + 31) / 32;
    bool bad = false;
    // One step: pop the lane's symbol (rans.py:147-152) and refill.
    auto step = [&](bool active) -> bool {
        uint32_t cnt = 0, sym = 0;
        if (active) {
            const uint32_t slot = x & mask;
            if constexpr (sizeof(L) < 4) {
                sym = lut[slot];
                const uint2 fc = tab[sym];
                x = fc.x * (x >> n) + slot - fc.y;
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
            cnt = (x < (1u << 15)) ? 2u : ((x < STATE_LOW) ? 1u : 0u);
        }
        const uint32_t b1 = __ballot_sync(0xffffffffu, cnt >= 1);
        const uint32_t b2 = __ballot_sync(0xffffffffu, cnt == 2);
        const uint32_t tot = __popc(b1) + __popc(b2);
        if (cur + tot > end) return false;  // rans.py:203-205 underrun
        const uint32_t a = cur + __popc(b1 & ltm) + __popc(b2 & ltm);
        uint32_t r0, r1;  // both bytes read unconditionally (cheap), selected below
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(r0) : "r"(ring_s + (a & (DRING - 1))));
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(r1) : "r"(ring_s + ((a + 1) & (DRING - 1))));
        x = cnt == 2 ? ((x << 16) | (r0 << 8) | r1) : (cnt == 1 ? ((x << 8) | r0) : x);
        cur += tot;
        if (active) *out = (S)sym;
        out += 32;
        advance();
        return true;
    };
    if (steps > 0) {
        const uint32_t full = len / 32;
        uint32_t s = 0;
        for (; s < full; ++s)
            if (!step(true)) {
                bad = true;
                break;
            }
        if (!bad && s < steps && !step(s * 32 + lane < len)) bad = true;  // partial last step
    }
    cp_async_wait<0>();
    // rans.py:211-212: every lane back at L and every byte consumed
    if (!bad) bad = __any_sync(0xffffffffu, x != STATE_LOW) || cur != end;
    if (bad && lane == 0) p.status[b] = SCZ_CORRUPT_STREAM;
}

template __global__ void k_rans_dec_v2<uint8_t, uint8_t>(DecParams);
template __global__ void k_rans_dec_v2<uint16_t, uint16_t>(DecParams);
template __global__ void k_rans_dec_v2<uint32_t, uint32_t>(DecParams);

// dynamic shared memory of k_rans_dec_v2 for a batch (max over tensors)
inline size_t dec_v2_smem(size_t lwidth, int n, uint32_t maxA) {
    size_t s = (size_t)DEC2_WPB * DRING;
    if (lwidth < 4) s += (size_t)maxA * sizeof(uint2) + ((size_t)1 << n) * lwidth;
    return (s + 15) & ~(size_t)15;
}

}  // namespace scz
