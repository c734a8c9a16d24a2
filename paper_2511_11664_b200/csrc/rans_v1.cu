// rans_v1.cu -- v1 (the reference's wire format) rANS stream kernels for the
// pipeline's symbol classes (K5, K7).
//
// A v1 payload is ONE rANS stream per tensor (rans.py:155-213): every state
// depends on the previous one, so a stream is a serial chain and its time is
// (symbols) x (cycles of one step on the chain).  One CTA per tensor, split
// by role so that a single thread -- the chain -- issues nothing but the
// state recurrence, and everything else runs beside it on other warps:
//
//   encode (3 warps):
//     warp 1  feeder   loads the symbols of 8 chunks (64 symbols each, in
//                      coding order: descending index, rans.py:170) with 16
//                      loads in flight per lane, gathers their encoder table
//                      entries (pre-transformed: bound, bias, rcp, shift, and
//                      cmpl = 2^n - f in a separate array) into a 16-chunk
//                      queue in shared memory;
//     warp 0  chain    lane 0 runs x' = x + bias + q * cmpl with
//                      q = umulhi(x_r, rcp) >> shift on the queued entries
//                      and records the state before every symbol;
//     warp 2  emitter  recomputes each symbol's renormalisation from the
//                      recorded state (<= 2 bytes, rans.py:139-142), places
//                      the bytes of 32 symbols at once with a warp ballot
//                      scan into an 8 KB output ring and TMA-stores each
//                      completed 4 KB half.
//   decode (3 warps):
//     warp 1  feeder   TMA-stages the payload and expands it into a ring of
//                      big-endian 4-byte windows P[q] = bytes q .. q+3, so the
//                      chain's refill is one load + one funnel shift;
//     warp 0  chain    lane 0: slot = x & (2^n - 1); f, slot - cum from the
//                      2^n-slot table (two 16-bit loads of one entry);
//                      x' = f (x >> n) + bias; refill 0, 1 or 2 bytes with
//                      both candidates formed in parallel (rans.py:199-210);
//                      records the slot;
//     warp 2  emitter  slot -> symbol through the table's symbol column,
//                      symbols into an output ring, TMA stores of halves.
//
// Roles hand chunks over through mbarriers, one per queue slot and
// direction (full / free), as TMA pipelines do.  Byte-identical to rans.encode / rans.decode
// (tests/test_gpu_parity.py, tests/test_gpu_bench_path.py).
#include "common.cuh"

namespace scz {

constexpr uint32_t V1_OUT = 8192;                // output ring (two 4 KB halves)
constexpr uint32_t V1_HALF = V1_OUT / 2;
#ifndef SCZ_V1_C
#define SCZ_V1_C 64
#endif
constexpr uint32_t V1_C = SCZ_V1_C;              // symbols per chunk
constexpr uint32_t V1_NQ = 1024 / V1_C;          // chunks in the queue
constexpr uint32_t V1_G = 512 / V1_C;            // chunks per encoder feeder group (16 loads per lane)
constexpr int V1_THREADS = 96;                   // chain, feeder, emitter warps

// (fence_proxy_async_smem: common.cuh)
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

// Role hand-over: one mbarrier per queue slot and direction ("full" /
// "free"), phase parity = lap of the slot.  Producers arrive after their
// writes (release), consumers try_wait.parity (acquire); an mbarrier phase
// cannot run ahead of its consumer, so parities never alias.
// (mbar_arrive: common.cuh)

// Input ring owned by one warp (lane 0 issues, every lane waits): chunk c =
// bytes [c * CH, (c + 1) * CH) of a 16-byte aligned source region with `end`
// valid bytes goes to slot c % NS.  Chunks at or past `end` are never fetched
// (and never waited for); a fetch stops at the 16-byte boundary after `end`,
// which never leaves the allocation holding the last valid byte.
template <uint32_t CH, uint32_t NS>
struct ChunkRing {
    uint8_t* buf;
    uint64_t* bar;
    const uint8_t* src;
    uint32_t end;
    uint32_t phase;  // bit s: parity of the next completion of slot s
    __device__ __forceinline__ void issue(int c) {
        if (c < 0) return;
        const uint32_t lo = (uint32_t)c * CH;
        if (lo >= end) return;
        const uint32_t hi = min(lo + CH, (end + 15u) & ~15u);
        const uint32_t s = (uint32_t)c % NS;
        fence_proxy_async_smem();  // earlier generic reads of the slot before the async write
        mbar_expect_tx(&bar[s], hi - lo);
        bulk_g2s(buf + s * CH, src + lo, hi - lo, &bar[s]);
    }
    __device__ __forceinline__ void wait(int c) {
        if (c < 0 || (uint32_t)c * CH >= end) return;
        const uint32_t s = (uint32_t)c % NS;
        mbar_wait(&bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
    }
};

// ---------------------------------------------------------------- encode
// Coding order k = 0 .. L-1 visits D[L-1-k] (rans.py:170).  Emitted byte j of
// the stream lands at slot_end - 1 - j, so the finished stream [4 state bytes]
// [bytes in decoder order] ends at the slot's end.
template <class Src>
__global__ void __launch_bounds__(V1_THREADS) k_rans_enc_v1p(EncParams p, Src src) {
    // launched without PDL (capi.cu launch_plain) and no early trigger: the
    // next kernel launches when this one completes, so nothing parks on the
    // SMs while the chains run
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const uint32_t b = blockIdx.x;
    TensorState& st = p.state[b];
    if (st.status != SCZ_OK) return;
    if (Src::width && st.sym_bytes != (uint32_t)Src::width) return;  // other symbol class
    __shared__ __align__(16) uint4 s_ent[V1_NQ][V1_C];  // bound, bias, rcp, shift
    __shared__ __align__(8) uint2 s_cm[V1_NQ][V1_C];    // cmpl = 2^n - f, bound << 8 (saturated)
    __shared__ uint32_t s_xs[V1_NQ][V1_C];              // state before the symbol
    __shared__ __align__(128) uint8_t s_out[V1_OUT];
    __shared__ uint32_t s_final;                        // the final state
    __shared__ __align__(8) uint64_t b_fed[V1_NQ], b_chn[V1_NQ], b_free[V1_NQ];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t L = (uint32_t)st.stream_len;
    const uint32_t nch = (L + V1_C - 1) / V1_C;
    const int n = p.precision;
    if (threadIdx.x < V1_NQ) {
        mbar_init(&b_fed[threadIdx.x], 32);  // the feeder's lanes
        mbar_init(&b_chn[threadIdx.x], 1);   // the chain thread
        mbar_init(&b_free[threadIdx.x], 32); // the emitter's lanes
    }
    __syncthreads();
    uint8_t* slot_end = p.slots + ((uint64_t)b * p.slots_per_tensor + 1) * p.slot_cap;  // 16-aligned
    uint32_t E = 0;  // emitter: bytes emitted so far
    if (warp == 1) {
        // ---- feeder: symbols -> table entries, 8 chunks per round
        const EncTab* gt = p.enctab + (uint64_t)b * p.acap;
        const uint64_t nnz = st.nnz;
        const uint32_t one = 1u << n;
        for (uint32_t g0 = 0; g0 < nch; g0 += V1_G) {
            const uint32_t g1 = min(g0 + V1_G, nch);
            for (uint32_t c = max(g0, V1_NQ); c < g1; ++c) mbar_wait(&b_free[c % V1_NQ], ((c / V1_NQ) - 1) & 1u);
            constexpr uint32_t NL = V1_G * V1_C / 32;  // symbols per lane per group
            uint32_t sym[NL];
#pragma unroll
            for (uint32_t j = 0; j < NL; ++j) {
                const uint32_t k = g0 * V1_C + j * 32 + lane;
                sym[j] = k < L ? src.at(b, L - 1 - k, nnz) : 0u;
            }
#pragma unroll
            for (uint32_t j = 0; j < NL; ++j) {
                const uint32_t k = g0 * V1_C + j * 32 + lane;
                if (k < L) {
                    const uint4 e = __ldg(reinterpret_cast<const uint4*>(gt) + sym[j]);  // freq, cum, rcp, shift
                    uint4 t;
                    uint2 cm;
                    t.x = e.x << (31 - n);  // bound ((L >> n) << 8) * f
                    cm.y = t.x >= (1u << 24) ? 0xFFFFFFFFu : t.x << 8;  // x >= bound2 <=> (x >> 8) >= bound
                    if (e.w == 0xFFFFFFFFu) {  // f = 1: q = x, x' = x + cum + (2^n - 1) x
                        t.y = e.y + one - 1u;
                        t.z = 0xFFFFFFFFu;
                        t.w = 0u;
                        cm.x = one - 1u;
                    } else {
                        t.y = e.y;
                        t.z = e.z;
                        t.w = e.w;
                        cm.x = one - e.x;
                    }
                    const uint32_t c = k / V1_C, i = k % V1_C;
                    s_ent[c % V1_NQ][i] = t;
                    s_cm[c % V1_NQ][i] = cm;
                }
            }
            for (uint32_t c = g0; c < g1; ++c) mbar_arrive(&b_fed[c % V1_NQ]);
        }
    } else if (warp == 0) {
        // ---- chain: the state recurrence (rans.py:139-144), one thread
        if (lane == 0) {
            uint32_t x = STATE_LOW;
            for (uint32_t c = 0; c < nch; ++c) {
                const uint32_t s = c % V1_NQ;
                mbar_wait(&b_fed[s], (c / V1_NQ) & 1u);
                // entries are loaded V1_D steps ahead of their use (explicit
                // shared addresses, volatile: the issue order is as written)
                const uint32_t ent_s = smem_u32(s_ent[s]), cm_s = smem_u32(s_cm[s]), xs_s = smem_u32(s_xs[s]);
                auto code = [&](const uint4& t, uint2 cm, uint32_t k) {
                    asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(xs_s + 4 * k), "r"(x) : "memory");
                    // The next state for each renormalisation outcome (0, 1 or 2
                    // bytes: x, x >> 8, x >> 16 coded) is formed in parallel and
                    // the tests only select one at the end: the select is off
                    // the multiply chain (asm keeps the compiler from hoisting
                    // it in front of the multiplies).
                    auto cand = [&](uint32_t xr) -> uint32_t {
                        uint32_t y;
                        asm("{\n .reg .b32 h, q, r;\n mul.hi.u32 h, %1, %2;\n shf.r.wrap.b32 q, h, 0, %3;\n"
                            " add.u32 r, %1, %4;\n mad.lo.u32 %0, q, %5, r;\n}\n"
                            : "=r"(y)
                            : "r"(xr), "r"(t.z), "r"(t.w), "r"(t.y), "r"(cm.x));
                        return y;
                    };
                    const bool e1 = x >= t.x;
                    const bool e2 = x >= cm.y;  // (x >> 8) >= bound; implies e1
                    const uint32_t y0 = cand(x), y1 = cand(x >> 8), y2 = cand(x >> 16);
                    x = e2 ? y2 : (e1 ? y1 : y0);
                };
                auto lds64 = [](uint32_t a) -> uint2 {
                    uint2 t;
                    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n" : "=r"(t.x), "=r"(t.y) : "r"(a) : "memory");
                    return t;
                };
                auto lds128 = [](uint32_t a) -> uint4 {
                    uint4 t;
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                                 : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w)
                                 : "r"(a)
                                 : "memory");
                    return t;
                };
                const uint32_t m = min(V1_C, L - c * V1_C);
                if (m == V1_C) {
                    constexpr uint32_t V1_D = 4;
                    uint4 tq[V1_D];
                    uint2 cq[V1_D];
#pragma unroll
                    for (uint32_t d = 0; d < V1_D; ++d) {
                        tq[d] = lds128(ent_s + 16 * d);
                        cq[d] = lds64(cm_s + 8 * d);
                    }
#pragma unroll
                    for (uint32_t k = 0; k < V1_C; ++k) {
                        const uint4 t = tq[k % V1_D];
                        const uint2 cm = cq[k % V1_D];
                        if (k + V1_D < V1_C) {
                            tq[k % V1_D] = lds128(ent_s + 16 * (k + V1_D));
                            cq[k % V1_D] = lds64(cm_s + 8 * (k + V1_D));
                        }
                        code(t, cm, k);
                    }
                } else {
                    for (uint32_t k = 0; k < m; ++k) code(lds128(ent_s + 16 * k), lds64(cm_s + 8 * k), k);
                }
                mbar_arrive(&b_chn[s]);
            }
            s_final = x;
        }
    } else {
        // ---- emitter: renormalisation bytes of 32 symbols per ballot scan
        const uint32_t ltm = lanemask_lt();
        const uint32_t out_s = smem_u32(s_out);
        for (uint32_t c = 0; c < nch; ++c) {
            const uint32_t s = c % V1_NQ;
            mbar_wait(&b_chn[s], (c / V1_NQ) & 1u);
#pragma unroll
            for (uint32_t h = 0; h < V1_C / 32; ++h) {
                const uint32_t k = h * 32 + lane;
                const bool valid = c * V1_C + k < L;
                const uint32_t x = s_xs[s][k], bnd = s_ent[s][k].x;
                const bool e1 = valid && x >= bnd;
                const bool e2 = valid && (x >> 8) >= bnd;
                const uint32_t b1 = __ballot_sync(0xffffffffu, e1), b2 = __ballot_sync(0xffffffffu, e2);
                const uint32_t En = E + __popc(b1) + __popc(b2);
                const uint32_t j = E + __popc(b1 & ltm) + __popc(b2 & ltm);
                const bool cross = (E / V1_HALF) != (En / V1_HALF);  // warp-uniform
                if (cross) {
                    // the half being entered reuses the buffer of the half two
                    // back: its TMA store must have finished reading it
                    if (lane == 0) bulk_wait_read<0>();
                    __syncwarp();
                }
                sts_u8_if(out_s + (~j & (V1_OUT - 1)), x, e1);
                sts_u8_if(out_s + (~(j + 1) & (V1_OUT - 1)), x >> 8, e2);
                if (cross) {  // half E / V1_HALF is complete: TMA store it
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        const uint32_t mh = E / V1_HALF;
                        bulk_s2g(slot_end - (uint64_t)(mh + 1) * V1_HALF, s_out + ((mh & 1u) ? 0u : V1_HALF),
                                 V1_HALF);
                    }
                }
                E = En;
            }
            mbar_arrive(&b_free[s]);
        }
    }
    __syncthreads();
    if (warp == 2) {
        const uint32_t x = s_final;
        // bytes of the last, partial half, then the 4 little-endian state bytes
        const uint32_t j0 = E & ~(V1_HALF - 1);
        for (uint32_t j = j0 + lane; j < E; j += 32) slot_end[-(int64_t)j - 1] = s_out[~j & (V1_OUT - 1)];
        if (lane < 4) slot_end[-(int64_t)E - 4 + lane] = (uint8_t)(x >> (8 * lane));
        if (lane == 0) {
            p.block_len[(uint64_t)b * p.slots_per_tensor] = 4 + E;
            bulk_wait_all();
        }
    }
}

template __global__ void k_rans_enc_v1p<Contig8Src>(EncParams, Contig8Src);
template __global__ void k_rans_enc_v1p<SplitSrc<uint16_t>>(EncParams, SplitSrc<uint16_t>);
template __global__ void k_rans_enc_v1p<SplitSrc<uint32_t>>(EncParams, SplitSrc<uint32_t>);

// ---------------------------------------------------------------- decode
// Shared memory (dynamic):
//   lut   [2^n] u32 (f << 16) | (slot - cum), then [2^n] symbol (L)  (k_dec_prepare, TMA)
//   P     [V1D_PRING + V1D_PMIR] u32: P[q mod PRING] = bytes q..q+3 of the
//         payload, big-endian; positions [0, PMIR) of every PRING-aligned lap
//         are mirrored past the ring end (a chunk's reads never wrap)
//   raw   [V1D_NR][V1D_RCH] payload bytes (TMA ring)
//   slots [V1_NQ][V1_C] u16
//   out   [V1_OUT] symbol ring
constexpr uint32_t V1D_PCH = 256;                 // positions per P chunk
constexpr uint32_t V1D_NP = 8;                    // P chunks in the ring
constexpr uint32_t V1D_PRING = V1D_PCH * V1D_NP;  // positions in the ring
constexpr uint32_t V1D_PMIR = 2 * V1_C + 32;      // > 2 V1_C: one chunk's refills
constexpr uint32_t V1D_RCH = 2048;                // raw TMA chunk (bytes)
constexpr uint32_t V1D_NR = 4;

__host__ __device__ inline size_t dec_v1p_lut_bytes(int n, size_t lwidth) { return (((size_t)1 << n) * (4 + lwidth) + 15) & ~(size_t)15; }
inline size_t dec_v1p_smem(int n, size_t lwidth) {
    return dec_v1p_lut_bytes(n, lwidth) + 4 * (V1D_PRING + V1D_PMIR) + V1D_NR * V1D_RCH + 2 * V1_NQ * V1_C + V1_OUT;
}

template <typename S, typename L>
__global__ void __launch_bounds__(V1_THREADS) k_rans_dec_v1p(DecParams p) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // see k_rans_enc_v1p
    const uint32_t b = blockIdx.x;
    const scz_info& in = p.info[b];
    if (p.status[b] != SCZ_OK || in.version != 1 || in.sym_bytes != sizeof(S)) return;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[V1D_NR + 1];
    __shared__ uint32_t s_fin[2];  // final state, final position
    __shared__ __align__(8) uint64_t b_pfull[V1D_NP], b_pfree[V1D_NP], b_schn[V1_NQ], b_sfree[V1_NQ];
    const int n = in.precision;
    const uint32_t nslots = 1u << n;
    const uint32_t lut_bytes = (uint32_t)dec_v1p_lut_bytes(n, sizeof(L));
    uint8_t* lut = smem;
    uint32_t* P = reinterpret_cast<uint32_t*>(smem + lut_bytes);
    uint8_t* raw = reinterpret_cast<uint8_t*>(P + V1D_PRING + V1D_PMIR);
    uint16_t* slots = reinterpret_cast<uint16_t*>(raw + V1D_NR * V1D_RCH);
    uint8_t* oring = reinterpret_cast<uint8_t*>(slots + V1_NQ * V1_C);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t Ls = (uint32_t)(2 * in.nnz + in.n_rows);
    const uint32_t plen = (uint32_t)in.payload_len;  // >= 4 (host check)
    const uint32_t nch = (Ls + V1_C - 1) / V1_C;
    const uint32_t npch = (plen + V1D_PCH - 1) / V1D_PCH;
    if (threadIdx.x < V1D_NP) {
        mbar_init(&b_pfull[threadIdx.x], 32);  // the feeder's lanes
        mbar_init(&b_pfree[threadIdx.x], 1);   // the chain thread
    }
    if (threadIdx.x < V1_NQ) {
        mbar_init(&b_schn[threadIdx.x], 1);    // the chain thread
        mbar_init(&b_sfree[threadIdx.x], 32);  // the emitter's lanes
    }
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i <= V1D_NR; ++i) mbar_init(&bars[i], 1);
        mbar_expect_tx(&bars[V1D_NR], lut_bytes);
        bulk_g2s(lut, p.lut + (uint64_t)b * p.lut_stride, lut_bytes, &bars[V1D_NR]);
    }
    __syncthreads();
    const uint32_t HS = V1_HALF / sizeof(S);  // symbols per output half
    uint8_t* gout = reinterpret_cast<uint8_t*>(p.dsym) + (uint64_t)b * p.dsym_stride;  // 16-aligned
    if (warp == 1) {
        // ---- feeder: payload -> big-endian 4-byte windows
        const uint64_t a0 = in.payload_off;
        const uint64_t gbase = a0 & ~15ull;
        const uint32_t off0 = (uint32_t)(a0 - gbase);
        const uint32_t rend = off0 + plen;
        ChunkRing<V1D_RCH, V1D_NR> rg{raw, bars, p.payload + gbase, rend, 0u};
        if (lane == 0) {
            rg.issue(0);
            rg.issue(1);
        }
        int rw = 0;  // next raw chunk to wait for
        const uint32_t raw_s = smem_u32(raw);
        for (uint32_t g = 0; g < npch; ++g) {
            if (g >= V1D_NP) mbar_wait(&b_pfree[g % V1D_NP], ((g / V1D_NP) - 1) & 1u);
            // raw bytes [off0 + 256 g, off0 + 256 g + 259) (clamped to the payload)
            const int hi = (int)(min(off0 + g * V1D_PCH + V1D_PCH + 2, rend - 1) / V1D_RCH);
            while (rw <= hi) {
                rg.wait(rw);
                __syncwarp();
                if (lane == 0) rg.issue(rw + 2);  // reuses the slot of rw - 2 (no longer read)
                ++rw;
            }
            const uint32_t q0 = g * V1D_PCH + 8 * lane;  // this lane's 8 positions
            uint32_t by[11];
#pragma unroll
            for (uint32_t t = 0; t < 11; ++t) {
                const uint32_t q = q0 + t;
                by[t] = q < plen ? lds_u8(raw_s + ((off0 + q) & (V1D_NR * V1D_RCH - 1))) : 0u;
            }
            const uint32_t pi = q0 % V1D_PRING;
#pragma unroll
            for (uint32_t u = 0; u < 8; ++u) {
                const uint32_t w = (by[u] << 24) | (by[u + 1] << 16) | (by[u + 2] << 8) | by[u + 3];
                P[pi + u] = w;
                if (pi + u < V1D_PMIR) P[V1D_PRING + pi + u] = w;
            }
            mbar_arrive(&b_pfull[g % V1D_NP]);
        }
    } else if (warp == 0) {
        // ---- chain: the state recurrence (rans.py:199-210), one thread
        if (lane == 0) {
            const uint32_t mask = nslots - 1;
            const uint32_t lut_s = smem_u32(lut), P_s = smem_u32(P);
            const uint32_t slots_s = smem_u32(slots);
            uint32_t waited = 1, released = 0;  // P chunks waited for / handed back
            mbar_wait(&b_pfull[0], 0);
            const uint32_t x0 = lds_u32(P_s);
            const uint32_t x = __byte_perm(x0, 0u, 0x0123u);  // 4-byte little-endian initial state (rans.py:193)
            uint32_t ea = lut_s + 4 * (x & mask), xs = x >> n;  // entry address of x's slot, x >> n
            uint32_t pos = 4;
            mbar_wait(&bars[V1D_NR], 0);  // the table
            for (uint32_t c = 0; c < nch; ++c) {
                const uint32_t s = c % V1_NQ;
                if (c >= V1_NQ) mbar_wait(&b_sfree[s], ((c / V1_NQ) - 1) & 1u);
                // this chunk refills at most 2 V1_C bytes: windows up to pos + 2 V1_C
                const uint32_t need = min((pos + 2 * V1_C) / V1D_PCH, npch - 1) + 1;
                for (; waited < need; ++waited) mbar_wait(&b_pfull[waited % V1D_NP], (waited / V1D_NP) & 1u);
                for (; released < pos / V1D_PCH; ++released) mbar_arrive(&b_pfree[released % V1D_NP]);
                const uint32_t pa0 = P_s + 4 * (pos % V1D_PRING);
                uint32_t pa = pa0;
                uint32_t v = lds_u32(pa);
                const uint32_t sl_s = slots_s + 2 * V1_C * s;
                // The chain carries the next table entry's address and x >> n
                // instead of x: the three refill candidates (0, 1, 2 bytes)
                // get their entry addresses in parallel, and the refill test
                // only selects one of them (asm keeps the compiler from
                // folding the select back in front of the address math).
                auto addr_of = [&](uint32_t c) -> uint32_t {
                    uint32_t a;
                    asm("{\n .reg .b32 t;\n and.b32 t, %1, %2;\n mad.lo.u32 %0, t, 4, %3;\n}\n"
                        : "=r"(a)
                        : "r"(c), "r"(mask), "r"(lut_s));
                    return a;
                };
                auto step = [&](uint32_t k) {
                    const uint32_t f = lds_u16(ea + 2), bias = lds_u16(ea);
                    asm volatile("st.shared.u16 [%0], %1;\n" ::"r"(sl_s + 2 * k), "r"((ea - lut_s) >> 2) : "memory");
                    const uint32_t xn = f * xs + bias;
                    const uint32_t x1 = __funnelshift_l(v, xn, 8), x2 = __funnelshift_l(v, xn, 16);
                    const bool r1 = xn < STATE_LOW, r2 = xn < (1u << 15);  // r2 implies r1
                    const uint32_t a0 = addr_of(xn), a1 = addr_of(x1), a2 = addr_of(x2);
                    ea = r1 ? (r2 ? a2 : a1) : a0;
                    xs = r1 ? (r2 ? (x2 >> n) : (x1 >> n)) : (xn >> n);
                    pa += (r1 ? 4u : 0u) + (r2 ? 4u : 0u);
                    v = lds_u32(pa);  // the next refill's window (off the state chain)
                };
                const uint32_t m = min(V1_C, Ls - c * V1_C);
                if (m == V1_C) {
#pragma unroll
                    for (uint32_t k = 0; k < V1_C; ++k) step(k);
                } else {
                    for (uint32_t k = 0; k < m; ++k) step(k);
                }
                pos += (pa - pa0) >> 2;
                mbar_arrive(&b_schn[s]);
            }
            s_fin[0] = (xs << n) | ((ea - lut_s) >> 2);  // the final state
            s_fin[1] = pos;
        }
    } else {
        // ---- emitter: slot -> symbol, output ring, TMA stores of halves
        mbar_wait(&bars[V1D_NR], 0);
        const L* lsym = reinterpret_cast<const L*>(lut + lut_sym_off(n));
        S* ob = reinterpret_cast<S*>(oring);
        for (uint32_t c = 0; c < nch; ++c) {
            const uint32_t s = c % V1_NQ;
            mbar_wait(&b_schn[s], (c / V1_NQ) & 1u);
#pragma unroll
            for (uint32_t h = 0; h < V1_C / 32; ++h) {
                const uint32_t k = h * 32 + lane;
                const uint32_t i = c * V1_C + k;
                if (i < Ls) ob[i % (2 * HS)] = (S)lsym[slots[s * V1_C + k]];
            }
            mbar_arrive(&b_sfree[s]);
            const uint32_t iend = (c + 1) * V1_C;
            if (iend % HS == 0 && iend <= Ls) {  // a half is complete: TMA store it
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    const uint32_t half = (iend / HS - 1) & 1u;
                    bulk_s2g(gout + (size_t)(iend - HS) * sizeof(S), oring + half * V1_HALF, V1_HALF);
                    bulk_wait_read<1>();  // the other half's previous store has read it
                }
                __syncwarp();
            }
        }
    }
    __syncthreads();
    if (warp == 2) {
        // the partial last half
        const uint32_t done = Ls - Ls % HS;
        const uint32_t rem = Ls - done;
        const uint32_t half = (done / HS) & 1u;
        const S* srcp = reinterpret_cast<const S*>(oring + half * V1_HALF);
        S* dst = reinterpret_cast<S*>(gout) + done;
        for (uint32_t i = lane; i < rem; i += 32) dst[i] = srcp[i];
        // rans.py:211-212: the final state is L and every byte was consumed
        if (lane == 0) {
            if (s_fin[0] != STATE_LOW || s_fin[1] != plen) p.status[b] = SCZ_CORRUPT_STREAM;
            bulk_wait_all();
        }
    }
}

template __global__ void k_rans_dec_v1p<uint8_t, uint8_t>(DecParams);
template __global__ void k_rans_dec_v1p<uint16_t, uint16_t>(DecParams);

}  // namespace scz
