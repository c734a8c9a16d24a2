// rans_v1.cu -- v1 (the reference's wire format) rANS stream kernels for the
// pipeline's u8 / u16 symbol classes (K5, K7).
//
// A v1 payload is ONE rANS stream per tensor (rans.py:155-213): every state
// depends on the previous one, so a stream is a serial chain and its time is
// (symbols) x (latency of one step).  These kernels therefore spend the GPU
// on shortening that chain, not on parallelism inside a stream: one CTA per
// tensor, one thread (lane 0) runs the recurrence with nothing but
// register ALU work and shared-memory loads on it, and everything else is
// moved off the chain:
//   * input bytes / symbols arrive in shared memory by TMA bulk copies issued
//     two to three 4 KB chunks ahead (mbarrier per ring slot);
//   * outputs leave shared memory by TMA bulk stores of completed 4 KB
//     halves (one instruction per 4 KB instead of a store per symbol);
//   * decode: the slot table is split into f[2^n] u16, bias[2^n] u16 and
//     sym[2^n] (built by k_dec_prepare), so the state update is one IMAD on
//     two independent 16-bit loads; the refill takes the next two payload
//     bytes (an off-chain funnel shift of two ring words) with one funnel
//     shift of 0, 8 or 16 bits (rans.py:205-210);
//   * encode: the table entry of the next symbols is loaded two steps ahead
//     (symbols do not depend on the state); renormalisation and the division
//     use the pre-transformed entry of rans_enc.cu (x' = x + bias + q * cmpl,
//     q = umulhi(x, rcp) >> shift, exact for x < 2^31).
// The batch's streams run concurrently (one CTA each), so a batch of B
// tensors costs about one stream's chain.  Byte-identical to rans.encode /
// rans.decode (tests/test_gpu_parity.py, tests/test_gpu_bench_path.py).
#include "common.cuh"

namespace scz {

constexpr uint32_t V1_CH = 4096;                 // bytes per staged input chunk
constexpr uint32_t V1_NCH = 4;                   // input ring slots
constexpr uint32_t V1_RING = V1_CH * V1_NCH;     // 16 KB input ring
constexpr uint32_t V1_OUT = 8192;                // output ring (two 4 KB halves)
constexpr uint32_t V1_HALF = V1_OUT / 2;

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// shared -> global bulk copy (TMA store), completion tracked by bulk groups
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// Input ring owned by one thread: chunk c = bytes [c * V1_CH, (c + 1) * V1_CH)
// of a 16-byte aligned source region with `end` valid bytes goes to slot
// c % V1_NCH.  Chunks at or past `end` are never fetched (and never waited
// for); a fetch stops at the 16-byte boundary after `end`, which never leaves
// the allocation holding the last valid byte.
struct ChunkRing {
    uint8_t* buf;
    uint64_t* bar;
    const uint8_t* src;
    uint32_t end;
    uint32_t phase;  // bit s: parity of the next completion of slot s
    __device__ __forceinline__ void issue(int c) {
        if (c < 0) return;
        const uint32_t lo = (uint32_t)c * V1_CH;
        if (lo >= end) return;
        const uint32_t hi = min(lo + V1_CH, (end + 15u) & ~15u);
        const uint32_t s = (uint32_t)c % V1_NCH;
        fence_proxy_async_smem();  // earlier generic reads of the slot before the async write
        mbar_expect_tx(&bar[s], hi - lo);
        bulk_g2s(buf + s * V1_CH, src + lo, hi - lo, &bar[s]);
    }
    __device__ __forceinline__ void wait(int c) {
        if (c < 0 || (uint32_t)c * V1_CH >= end) return;
        const uint32_t s = (uint32_t)c % V1_NCH;
        mbar_wait(&bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
    }
};

// ---------------------------------------------------------------- decode
// Shared memory: input ring [V1_RING] | output ring [V1_OUT] |
//                f [2^n] u16 | bias [2^n] u16 | sym [2^n] L   (k_dec_prepare)
inline size_t dec_v1_smem(int n, size_t lwidth) {
    return V1_RING + V1_OUT + ((((size_t)1 << n) * (4 + lwidth) + 15) & ~(size_t)15);
}

template <typename S, typename L>
__global__ void __launch_bounds__(32) k_rans_dec_v1_fast(DecParams p) {
    pdl_wait();
    const uint32_t b = blockIdx.x;
    const scz_info& in = p.info[b];
    if (p.status[b] != SCZ_OK || in.version != 1 || in.sym_bytes != sizeof(S)) return;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[V1_NCH + 1];
    const int n = in.precision;
    const uint32_t nslots = 1u << n;
    uint8_t* ring = smem;
    uint8_t* oring = smem + V1_RING;
    uint8_t* lut = oring + V1_OUT;
    const uint32_t lane = threadIdx.x;
    const uint64_t Ls = 2 * in.nnz + in.n_rows;
    const uint64_t a0 = in.payload_off;
    const uint64_t gbase = a0 & ~15ull;
    const uint32_t off0 = (uint32_t)(a0 - gbase);
    const uint32_t end = off0 + (uint32_t)in.payload_len;
    uint8_t* gout = reinterpret_cast<uint8_t*>(p.dsym) + (uint64_t)b * p.dsym_stride;  // 16-aligned
    constexpr uint32_t HS = V1_HALF / sizeof(S);  // symbols per output half
    uint32_t x = 0, pos = 0;
    if (lane == 0) {
        for (uint32_t i = 0; i <= V1_NCH; ++i) mbar_init(&bars[i], 1);
        const uint32_t lut_bytes = ((nslots * (4u + (uint32_t)sizeof(L))) + 15u) & ~15u;
        mbar_expect_tx(&bars[V1_NCH], lut_bytes);
        bulk_g2s(lut, p.lut + (uint64_t)b * p.lut_stride, lut_bytes, &bars[V1_NCH]);
        ChunkRing rg{ring, bars, p.payload + gbase, end, 0u};
        for (int c = 0; c < (int)V1_NCH; ++c) rg.issue(c);
        rg.wait(0);
        rg.wait(1);
        int k = 0;  // chunk holding pos; chunks k, k + 1 have landed
        const uint32_t ring_s = smem_u32(ring);
        const uint32_t out_s = smem_u32(oring);
        // the two payload words at byte a (ring coordinates), funnel-shifted
        auto bytes_at = [&](uint32_t a) -> uint32_t {
            const uint32_t wa = a & ~3u;
            const uint32_t w0 = lds_u32(ring_s + (wa & (V1_RING - 1)));
            const uint32_t w1 = lds_u32(ring_s + ((wa + 4) & (V1_RING - 1)));
            return __funnelshift_r(w0, w1, (a & 3u) * 8);  // byte a in bits 0-7
        };
        x = bytes_at(off0);  // 4-byte little-endian initial state (rans.py:193)
        pos = off0 + 4;
        // explicit 32-bit shared addresses: f, bias and symbol of a slot are
        // three loads whose addresses are one op each from the slot
        const uint32_t lf = smem_u32(lut), lb = lf + 2 * nslots, ls = lf + 4 * nslots;
        const uint32_t mask = nslots - 1;
        mbar_wait(&bars[V1_NCH], 0);
        // one symbol: rans.py:199-210
        auto pop = [&](uint32_t i) {
            const uint32_t slot = x & mask;
            const uint32_t f = lds_u16(lf + 2 * slot);
            const uint32_t bias = lds_u16(lb + 2 * slot);
            const uint32_t sym = sizeof(L) == 1 ? lds_u8(ls + slot) : lds_u16(ls + 2 * slot);
            const uint32_t v = bytes_at(pos);                  // the next payload bytes (off the chain)
            const uint32_t wbe = __byte_perm(v, 0u, 0x0123u);  // next byte in bits 24-31
            const uint32_t xn = f * (x >> n) + bias;
            // refill 0, 1 or 2 bytes (x < 2^15 -> 2 for n <= 16): both shifted
            // candidates and both tests in parallel, then two selects
            const uint32_t x1 = __funnelshift_l(wbe, xn, 8), x2 = __funnelshift_l(wbe, xn, 16);
            const bool r1 = xn < STATE_LOW, r2 = xn < (1u << 15);
            x = r1 ? (r2 ? x2 : x1) : xn;
            pos += (r1 ? 1u : 0u) + (r2 ? 1u : 0u);
            if (sizeof(S) == 1) {
                asm volatile("st.shared.u8 [%0], %1;\n" ::"r"(out_s + (i & (V1_OUT - 1))), "r"(sym) : "memory");
            } else {
                asm volatile("st.shared.u16 [%0], %1;\n" ::"r"(out_s + 2u * (i & (V1_OUT / 2 - 1))), "r"(sym)
                             : "memory");
            }
        };
        uint32_t half = 0;  // output half being filled
        const uint32_t L32 = (uint32_t)Ls, L4 = L32 & ~3u;
        uint32_t i = 0;
        for (; i < L4; i += 4) {
            pop(i);
            pop(i + 1);
            pop(i + 2);
            pop(i + 3);
            if ((i + 4) % HS == 0) {  // a half is complete: TMA store it
                fence_proxy_async_smem();
                bulk_s2g(gout + (size_t)(i + 4 - HS) * sizeof(S), oring + half * V1_HALF, V1_HALF);
                half ^= 1u;
                bulk_wait_read<1>();  // the other half's previous store has read it
            }
            // four symbols move pos by <= 8 bytes and read <= 8 bytes past it:
            // one chunk check per four symbols keeps chunks k, k + 1 landed
            if ((int)(pos / V1_CH) != k) {
                ++k;
                rg.wait(k + 1);
                rg.issue(k + 3);
            }
        }
        for (; i < L32; ++i) pop(i);
        bulk_wait_all();
    }
    __syncwarp();
    x = __shfl_sync(0xffffffffu, x, 0);
    pos = __shfl_sync(0xffffffffu, pos, 0);
    // the partial last half
    const uint64_t done = Ls - Ls % HS;
    const uint32_t rem = (uint32_t)(Ls - done);
    const uint32_t half = (uint32_t)((done / HS) & 1u);
    const S* src = reinterpret_cast<const S*>(oring + half * V1_HALF);
    S* dst = reinterpret_cast<S*>(gout) + done;
    for (uint32_t i = lane; i < rem; i += 32) dst[i] = src[i];
    // rans.py:211-212: the final state is L and every byte was consumed
    if (lane == 0 && (x != STATE_LOW || pos != end)) p.status[b] = SCZ_CORRUPT_STREAM;
}

template __global__ void k_rans_dec_v1_fast<uint8_t, uint8_t>(DecParams);
template __global__ void k_rans_dec_v1_fast<uint16_t, uint16_t>(DecParams);

// ---------------------------------------------------------------- encode
// u8 symbol class (D = v ++ c ++ r contiguous u8, A <= 256): the pipeline's
// common v1 case.  Symbols are coded in reverse (rans.py:170); emitted byte
// j of the stream lands at slot_end - 1 - j, so the finished stream
// [4 state bytes][bytes in decoder order] ends at the slot's end.
__global__ void __launch_bounds__(32) k_rans_enc_v1_fast(EncParams p, Contig8Src src) {
    pdl_wait();
    const uint32_t b = blockIdx.x;
    TensorState& st = p.state[b];
    if (st.status != SCZ_OK || st.sym_bytes != 1) return;
    __shared__ __align__(16) uint8_t s_ring[V1_RING];
    __shared__ __align__(16) uint8_t s_out[V1_OUT];
    __shared__ __align__(16) EncTab s_tab[256];
    __shared__ __align__(8) uint64_t bars[V1_NCH];
    const uint32_t lane = threadIdx.x;
    const uint32_t A = st.alphabet;  // <= 256 for the u8 class
    const EncTab* gt = p.enctab + (uint64_t)b * p.acap;
    const int n = p.precision;
    for (uint32_t i = lane; i < A; i += 32) {  // bound / bias / rcp / shift | cmpl << 16 (rans_enc.cu)
        const EncTab e = gt[i];
        EncTab f;
        f.freq = e.freq << (31 - n);
        if (e.shift == 0xFFFFFFFFu) {
            f.cum = e.cum + (1u << n) - 1u;
            f.rcp = 0xFFFFFFFFu;
            f.shift = ((1u << n) - 1u) << 16;
        } else {
            f.cum = e.cum;
            f.rcp = e.rcp;
            f.shift = e.shift | (((1u << n) - e.freq) << 16);
        }
        s_tab[i] = f;
    }
    __syncwarp();
    const uint32_t L = (uint32_t)st.stream_len;
    uint8_t* slot_end = p.slots + ((uint64_t)b * p.slots_per_tensor + 1) * p.slot_cap;  // 16-aligned
    uint32_t x = STATE_LOW, E = 0;
    if (lane == 0) {
        for (uint32_t i = 0; i < V1_NCH; ++i) mbar_init(&bars[i], 1);
        ChunkRing rg{s_ring, bars, src.d + (uint64_t)b * src.stride, L, 0u};
        const int kt = (int)((L - 1) / V1_CH);
        rg.issue(kt);
        rg.issue(kt - 1);
        int k = kt + 1;  // chunk of the prefetch index; chunks k, (k - 1 in flight) ...
        const uint32_t ring_s = smem_u32(s_ring);
        const uint32_t out_s = smem_u32(s_out);
        const uint32_t tab_s = smem_u32(s_tab);
        auto lds_tab = [&](uint32_t sym) -> uint4 {
            uint4 t;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                         : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w)
                         : "r"(tab_s + 16 * sym));
            return t;
        };
        // chunk bookkeeping for the lowest index j of the next symbols read
        auto enter = [&](uint32_t j) {
            if ((int)(j / V1_CH) != k) {  // entered chunk k - 1
                --k;
                rg.wait(k);
                rg.issue(k - 2);
            }
        };
        // one symbol (rans.py:139-144) with its table entry t =
        // {bound, bias, rcp, shift | cmpl << 16}
        auto push = [&](const uint4& t) {
            const bool e1 = x >= t.x;
            const uint32_t a = x >> 8;
            const bool e2 = a >= t.x;  // implies e1
            if ((E & (V1_HALF - 1)) >= V1_HALF - 2) bulk_wait_read<0>();  // may enter a half still being stored
            sts_u8_if(out_s + (~E & (V1_OUT - 1)), x, e1);
            sts_u8_if(out_s + (~(E + 1) & (V1_OUT - 1)), a, e2);
            const uint32_t En = E + (e1 ? 1u : 0u) + (e2 ? 1u : 0u);
            if ((En ^ E) & ~(V1_HALF - 1)) {  // half E / V1_HALF complete: TMA store it
                const uint32_t m = E / V1_HALF;
                fence_proxy_async_smem();
                bulk_s2g(slot_end - (uint64_t)(m + 1) * V1_HALF, s_out + ((m & 1u) ? 0u : V1_HALF), V1_HALF);
            }
            E = En;
            const uint32_t xr = e2 ? (a >> 8) : (e1 ? a : x);
            const uint32_t q = __funnelshift_r(__umulhi(xr, t.z), 0u, t.w);
            x = q * (t.w >> 16) + (xr + t.y);
        };
        // the top (L mod 4) symbols one by one, then aligned groups of four:
        // the four table entries of the next group load while this group codes
        const uint32_t L4 = L & ~3u;
        for (uint32_t i = L; i > L4;) {
            --i;
            enter(i);
            push(lds_tab(lds_u8(ring_s + (i & (V1_RING - 1)))));
        }
        auto load4 = [&](uint32_t j, uint4* t) {  // symbols j .. j + 3 (j % 4 == 0)
            enter(j);
            const uint32_t w = lds_u32(ring_s + (j & (V1_RING - 1)));
            t[0] = lds_tab(w >> 24);
            t[1] = lds_tab((w >> 16) & 0xFFu);
            t[2] = lds_tab((w >> 8) & 0xFFu);
            t[3] = lds_tab(w & 0xFFu);
        };
        // Fast form for four symbols that cannot leave the current output
        // half (<= 8 bytes, checked once per four): no per-symbol checks, the
        // bytes go to a descending ring offset r (byte E at r = ~E mod 8192)
        // with predicated stores at r and r - 1.
        auto push_fast = [&](const uint4& t, uint32_t& r) {
            const bool e1 = x >= t.x;
            const uint32_t a = x >> 8;
            const bool e2 = a >= t.x;
            // explicit 32-bit shared addresses (a C store to s_out[r] makes the
            // compiler rebuild the shared window base per store)
            asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.shared.u8 [%0], %1;\n}\n" ::"r"(
                             out_s + r),
                         "r"(x), "r"((uint32_t)e1));
            asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.shared.u8 [%0+-1], %1;\n}\n" ::"r"(
                             out_s + r),
                         "r"(a), "r"((uint32_t)e2));
            r -= (e1 ? 1u : 0u) + (e2 ? 1u : 0u);
            const uint32_t xr = e2 ? (a >> 8) : (e1 ? a : x);
            const uint32_t q = __funnelshift_r(__umulhi(xr, t.z), 0u, t.w);
            x = q * (t.w >> 16) + (xr + t.y);
        };
        auto push4 = [&](const uint4* t) {
            if ((E & (V1_HALF - 1)) <= V1_HALF - 9) {
                uint32_t r = ~E & (V1_OUT - 1);
                const uint32_t r0 = r;
                push_fast(t[0], r);
                push_fast(t[1], r);
                push_fast(t[2], r);
                push_fast(t[3], r);
                E += r0 - r;
            } else {
                push(t[0]);
                push(t[1]);
                push(t[2]);
                push(t[3]);
            }
        };
        uint4 ta[4], tb[4];
        if (L4) {
            load4(L4 - 4, ta);
            for (int j = (int)L4 - 4; j >= 0; j -= 8) {
                if (j >= 4) load4(j - 4, tb);
                push4(ta);
                if (j < 4) break;
                if (j >= 8) load4(j - 8, ta);
                push4(tb);
            }
        }
        bulk_wait_all();
    }
    __syncwarp();
    x = __shfl_sync(0xffffffffu, x, 0);
    E = __shfl_sync(0xffffffffu, E, 0);
    // bytes of the last, partial half, then the 4 little-endian state bytes
    const uint32_t j0 = E & ~(V1_HALF - 1);
    for (uint32_t j = j0 + lane; j < E; j += 32) slot_end[-(int64_t)j - 1] = s_out[~j & (V1_OUT - 1)];
    if (lane < 4) slot_end[-(int64_t)E - 4 + lane] = (uint8_t)(x >> (8 * lane));
    if (lane == 0) p.block_len[(uint64_t)b * p.slots_per_tensor] = 4 + E;
}

}  // namespace scz
