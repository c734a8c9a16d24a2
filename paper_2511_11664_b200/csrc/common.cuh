// common.cuh -- shared device definitions for libsczip_b200 (sm_100a).
//
// Layout conventions:
//  * a batch is B tensors of T float32 each, contiguous ([B][T]);
//  * the zero bitmap of tensor b is bitmap[b * words_pad .. ], bit (p & 31)
//    of word (p >> 5) set iff x[p] != 0.0f (the ~zero_mask of tensor.py:139);
//  * D = v ++ c ++ r (sparse.py:98-101) is never materialised whole: values
//    live in v8 (u8, rank-ordered), columns and row counts in cr (u8/u16/u32);
//  * per-tensor scalars live in TensorState; per-tensor variable-length
//    outputs in fixed-stride slots (stride recorded in the launch params).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/sczip_b200.h"

namespace scz {

constexpr int TILE = 8192;             // elements per stats/quantize tile
constexpr int TILE_THREADS = 256;      // 32 elements per thread
constexpr int TILE_WORDS = TILE / 32;  // bitmap words per tile
constexpr uint32_t STATE_LOW = 1u << 23;  // rans.py:26
constexpr int MAX_CAND = 256;          // feasible reshape candidates per launch (K <= 2^Q <= 256 bounds their count)

// Per-tensor device state written by the encode kernels (internal, not ABI).
struct TensorState {
    float xmin, xmax;      // fp32 min/max (tensor.py:127)
    uint32_t nonfinite;    // FeatureTensor check (tensor.py:48)
    uint32_t tiles_done;   // last-CTA ticket
    double scale;          // compute_params (tensor.py:101-122)
    int64_t zero_point;
    float rcp32;           // fl32(1/scale) for the guard-band quantiser
    uint32_t fast;         // 1 if the fp32 guard-band path is valid for this scale
    uint64_t nnz;
    uint32_t n_rows, n_cols;
    uint32_t alphabet;
    uint32_t cand_index;   // chosen candidate
    uint64_t stream_len;   // l_D = 2 nnz + N
    int32_t status;
    uint32_t search_flags;
    uint32_t n_evaluated;
    uint32_t n_blocks;
    uint32_t sym_bytes;    // width of the c/r symbols of the chosen K (1, 2, 4)
    uint32_t errbits;      // encoder flags (ERR_OVERFLOW | ERR_UNCODABLE)
    uint32_t sel_pending;  // lazy search: the first pass did not stop, price the rest
};

struct EncTab {  // per-symbol encoder table entry (16 B)
    uint32_t freq;
    uint32_t cum;
    uint32_t rcp;    // ceil(2^(31+l) / f), l = ceil(log2 f)   (f >= 2)
    uint32_t shift;  // l - 1 ; 0xFFFFFFFF marks f == 1 (q = x)
};

__host__ __device__ inline uint32_t ceil_div_u32(uint64_t a, uint64_t b) {
    return (uint32_t)((a + b - 1) / b);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint32_t lanemask_gt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_gt;" : "=r"(m));
    return m;
}

// Exact floor(x / f) for x < 2^31, f >= 1 (Granlund-Montgomery).
__device__ __forceinline__ uint32_t enc_div(uint32_t x, const EncTab& t) {
    if (t.shift == 0xFFFFFFFFu) return x;
    return __umulhi(x, t.rcp) >> t.shift;
}

__host__ __device__ inline void make_enc_tab(uint32_t f, uint32_t cum, EncTab* t) {
    t->freq = f;
    t->cum = cum;
    if (f <= 1) {
        t->rcp = 0;
        t->shift = 0xFFFFFFFFu;
        return;
    }
    uint32_t l = 0;
    while ((1u << l) < f) ++l;  // l = ceil(log2 f), f <= 2^16
    uint64_t m = ((1ull << (31 + l)) + f - 1) / f;
    t->rcp = (uint32_t)m;
    t->shift = l - 1;
}

// Block-wide exclusive scan of one uint32 per thread (blockDim.x <= 1024,
// multiple of 32).  Returns the exclusive prefix; *total gets the sum.
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp,
                                                         uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = (lane < NT / 32) ? s_warp[lane] : 0;
        uint32_t ws = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, ws, o);
            if (lane >= o) ws += y;
        }
        if (lane < NT / 32) s_warp[lane] = ws - w;
        if (lane == NT / 32 - 1) s_warp[32] = ws;
    }
    __syncthreads();
    uint32_t r = s_warp[warp] + x - v;
    *total = s_warp[32];
    __syncthreads();
    return r;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Decoupled look-back (single-pass scan) over the chunks of one tensor
// (CSR decode: row-count sums; v2 encoder: block byte lengths).  Word =
// flag << 32 | value; flag 1: the chunk's own value, flag 2: inclusive
// prefix.  Chunks of a tensor are consecutive blockIdx.x of one grid (or
// consecutive warps of one CTA) and start in order, so every predecessor
// makes progress.  Called by one full warp; it inspects 32 predecessors per
// round.  The words are zeroed before the launch.
__device__ uint32_t chunk_prefix(unsigned long long* st, uint32_t chunk, uint32_t local) {
    const uint32_t lane = threadIdx.x & 31;
    const volatile unsigned long long* vs = st;
    if (chunk == 0) {
        if (lane == 0) atomicExch(st, (2ull << 32) | local);
        return 0;
    }
    if (lane == 0) atomicExch(st + chunk, (1ull << 32) | local);
    uint32_t excl = 0;
    for (int j = (int)chunk - 1;; j -= 32) {
        const int idx = j - (int)lane;  // lane 0: nearest predecessor
        unsigned long long w = idx >= 0 ? vs[idx] : (2ull << 32);
        // back off while predecessors are still running, so waiting warps
        // leave the issue slots to the ones doing work
        for (uint32_t ns = 32; __any_sync(0xffffffffu, (w >> 32) == 0); ns = ns < 1024 ? 2 * ns : ns) {
            __nanosleep(ns);
            if ((w >> 32) == 0) w = vs[idx];
        }
        const uint32_t inc = __ballot_sync(0xffffffffu, (w >> 32) == 2);
        if (inc) {
            const uint32_t first = __ffs(inc) - 1;
            excl += warp_sum(lane <= first ? (uint32_t)w : 0u);
            break;
        }
        excl += warp_sum((uint32_t)w);
    }
    if (lane == 0) atomicExch(st + chunk, (2ull << 32) | (excl + local));
    return excl;
}

// Copy len bytes from shared memory (16-byte aligned, >= len + 4 bytes
// readable) to global memory at any alignment: a head to the first 16-byte
// boundary of dst, then 16-byte stores assembled from funnel-shifted shared
// words, then the tail.  All NT threads of the block call it.
template <int NT>
__device__ __forceinline__ void block_copy_s2g(uint8_t* dst, const uint8_t* s_src, uint32_t len) {
    uint32_t head = (uint32_t)((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15);
    head = head < len ? head : len;
    if (threadIdx.x < head) dst[threadIdx.x] = s_src[threadIdx.x];
    const uint32_t n16 = (len - head) >> 4;
    const uint32_t sh = (head & 3) * 8;
    for (uint32_t c = threadIdx.x; c < n16; c += NT) {
        const uint32_t o = head + 16 * c;
        const uint32_t* w = reinterpret_cast<const uint32_t*>(s_src) + (o >> 2);
        const uint32_t a0 = w[0], a1 = w[1], a2 = w[2], a3 = w[3], a4 = w[4];
        *reinterpret_cast<uint4*>(dst + o) = make_uint4(__funnelshift_r(a0, a1, sh), __funnelshift_r(a1, a2, sh),
                                                        __funnelshift_r(a2, a3, sh), __funnelshift_r(a3, a4, sh));
    }
    for (uint32_t i = head + 16 * n16 + threadIdx.x; i < len; i += NT) dst[i] = s_src[i];
}

// Shared-memory byte store / word load through an explicit 32-bit shared
// address (from __cvta_generic_to_shared once per kernel): keeps the compiler
// from re-deriving the shared window base per access in register-tight loops.
__device__ __forceinline__ void sts_u8_if(uint32_t saddr, uint32_t v, bool pred) {
    asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.shared.u8 [%0], %1;\n}\n" ::"r"(saddr),
                 "r"(v), "r"((uint32_t)pred)
                 : "memory");
}
// Compaction step: if (flags & mask) { smem[saddr] = v (low byte); ++saddr; }
__device__ __forceinline__ void sts_u8_bump(uint32_t& saddr, uint32_t v, uint32_t flags, uint32_t mask) {
    asm volatile(
        "{\n .reg .pred p;\n .reg .b32 t;\n and.b32 t, %2, %3;\n setp.ne.u32 p, t, 0;\n"
        " @p st.shared.u8 [%0], %1;\n @p add.u32 %0, %0, 1;\n}\n"
        : "+r"(saddr)
        : "r"(v), "r"(flags), "r"(mask)
        : "memory");
}
// value of every u8 symbol: fl32((i - z) * s) in fp64 (tensor.py dequantise)
__device__ __forceinline__ void build_dequant_lut(float* lut, double z, double scale) {
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x)
        lut[i] = __double2float_rn(__dmul_rn(__dsub_rn((double)i, z), scale));
}
__device__ __forceinline__ void red_shared_inc(uint32_t saddr) {
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(saddr) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(saddr) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t saddr) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];\n" : "=r"(v) : "r"(saddr) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t saddr) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];\n" : "=r"(v) : "r"(saddr) : "memory");
    return v;
}

// cp.async (Ampere-style LDGSTS) helpers: global -> shared without registers
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// mbarrier + bulk (TMA 1-D) copies: one thread moves a whole table into
// shared memory; the CTA waits on the barrier's transaction count.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// A value the compiler must keep in a register (it cannot rematerialise the
// output of a volatile asm): used for 32-bit shared addresses in hot loops.
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
    uint32_t r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {  // release.cta
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

// Copy len bytes staged in shared memory at s_stage + (dst & 15) -- the
// staging offset makes shared and global addresses agree mod 16 -- to global
// dst: the < 16-byte head and tail by threads 0-15 and 32-47, the aligned
// middle with one bulk copy (TMA) issued by thread 0.  Every thread that
// wrote the staging area runs fence_proxy_async_smem() before the barrier
// that precedes this call; thread 0 runs bulk_store_wait() before the CTA
// exits (the copy still reads shared memory).
__device__ __forceinline__ uint32_t stage_shift(const void* dst) {
    return (uint32_t)(reinterpret_cast<uintptr_t>(dst) & 15);
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void block_copy_s2g_bulk(uint8_t* dst, const uint8_t* s_stage, uint32_t len) {
    const uint32_t sh = stage_shift(dst);
    const uint8_t* s = s_stage + sh;
    uint32_t head = (16 - sh) & 15;
    head = head < len ? head : len;
    const uint32_t mid = (len - head) & ~15u, t0 = head + mid;
    if (threadIdx.x < head) dst[threadIdx.x] = s[threadIdx.x];
    if (threadIdx.x >= 32 && threadIdx.x - 32 < len - t0) dst[t0 + threadIdx.x - 32] = s[t0 + threadIdx.x - 32];
    if (threadIdx.x == 0 && mid) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst + head),
                     "r"(smem_u32(s + head)), "r"(mid)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
}
__device__ __forceinline__ void bulk_store_wait() {
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

// Programmatic dependent launch: pipeline kernels are launched with the
// PDL attribute; each one waits here, before touching memory, until the
// predecessor grid has completed and flushed, then at once allows its own
// dependent grid to launch (it becomes resident and parks in its own wait,
// so its launch latency hides behind this kernel instead of following it).
// Every PDL kernel calls this first, before any early return, so completion
// is transitive along the chain.  Both are no-ops without the attribute.
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

}  // namespace scz
