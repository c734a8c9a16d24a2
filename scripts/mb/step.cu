#include <cstdio>
#include <cstdint>
#define N_IT 20000
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) { uint32_t v; asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a)); return v; }
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a)); return v; }
__global__ void k(uint32_t* out, long long* cyc, uint32_t b, uint32_t b2, uint32_t rcp, uint32_t sh, uint32_t cm, uint32_t bias) {
    __shared__ uint32_t tab[1 << 13];
    __shared__ uint32_t P[4096];
    for (int i = threadIdx.x; i < (1 << 13); i += blockDim.x) tab[i & 8191] = ((uint32_t)(100 + (i % 300)) << 16) | (i % 100);
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) P[i] = i * 2654435761u;
    __syncthreads();
    if (threadIdx.x) return;
    long long t0, t1;
    uint32_t x = (1u << 23) + 12345;
    // ---- encoder A: predicates
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N_IT; ++i) {
        const bool e1 = x >= b, e2 = x >= b2;
        const uint32_t xr = e2 ? (x >> 16) : (e1 ? (x >> 8) : x);
        const uint32_t q = __funnelshift_r(__umulhi(xr, rcp), 0u, sh);
        x = q * cm + (xr + bias);
        x = (x & 0x3fffffff) | 0x800000;
    }
    t1 = clock64(); cyc[0] = t1 - t0; out[0] = x;
    // ---- encoder B: unsigned max of the three differences
    const uint32_t nb = 0u - b, bb = b + bias;
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N_IT; ++i) {
        const uint32_t d0 = x + nb, d1 = (x >> 8) + nb, d2 = (x >> 16) + nb;
        const uint32_t m = max(max(d0, d1), d2);
        const uint32_t xr = m + b;
        const uint32_t q = __funnelshift_r(__umulhi(xr, rcp), 0u, sh);
        x = q * cm + (m + bb);
        x = (x & 0x3fffffff) | 0x800000;
    }
    t1 = clock64(); cyc[1] = t1 - t0; out[1] = x;
    // ---- bare clamp op overhead (LOP3 per step)
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N_IT; ++i) { x = (x & 0x3fffffff) | 0x800000; x = x * 3 + 1; }
    t1 = clock64(); cyc[2] = t1 - t0; out[2] = x;
    // ---- decoder A: predicates
    const uint32_t tab_s = (uint32_t)__cvta_generic_to_shared(tab), P_s = (uint32_t)__cvta_generic_to_shared(P);
    uint32_t pa = P_s;
    x = (1u << 23) + 777;
    uint32_t v = lds_u32(pa);
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N_IT; ++i) {
        const uint32_t slot = x & 8191;
        const uint32_t ea = tab_s + 4 * slot;
        const uint32_t f = lds_u16(ea + 2), bi = lds_u16(ea);
        const uint32_t xn = f * (x >> 13) + bi;
        const uint32_t x1 = __funnelshift_l(v, xn, 8), x2 = __funnelshift_l(v, xn, 16);
        const bool r1 = xn < (1u << 23), r2 = xn < (1u << 15);
        x = r1 ? (r2 ? x2 : x1) : xn;
        pa += (r1 ? 4u : 0u) + (r2 ? 4u : 0u);
        pa = P_s + ((pa - P_s) & 16383);
        v = lds_u32(pa);
    }
    t1 = clock64(); cyc[3] = t1 - t0; out[3] = x;
    // ---- decoder B: sign-bit shift count
    x = (1u << 23) + 777; pa = P_s; v = lds_u32(pa);
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N_IT; ++i) {
        const uint32_t slot = x & 8191;
        const uint32_t ea = tab_s + 4 * slot;
        const uint32_t f = lds_u16(ea + 2), bi = lds_u16(ea);
        const uint32_t xn = f * (x >> 13) + bi;
        const uint32_t s = ((xn - (1u << 23)) >> 31) + ((xn - (1u << 15)) >> 31);
        x = __funnelshift_l(v, xn, s * 8);
        pa += 4 * s;
        pa = P_s + ((pa - P_s) & 16383);
        v = lds_u32(pa);
    }
    t1 = clock64(); cyc[4] = t1 - t0; out[4] = x;
    // ---- decoder C: clz
    x = (1u << 23) + 777; pa = P_s; v = lds_u32(pa);
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N_IT; ++i) {
        const uint32_t slot = x & 8191;
        const uint32_t ea = tab_s + 4 * slot;
        const uint32_t f = lds_u16(ea + 2), bi = lds_u16(ea);
        const uint32_t xn = f * (x >> 13) + bi;
        const uint32_t s8 = (__clz(xn) - 1) & 24;
        x = __funnelshift_l(v, xn, s8);
        pa += s8 >> 1;
        pa = P_s + ((pa - P_s) & 16383);
        v = lds_u32(pa);
    }
    t1 = clock64(); cyc[5] = t1 - t0; out[5] = x;
    // ---- decoder D: table-only chain (slot -> lds -> imad), no refill
    x = (1u << 23) + 777;
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N_IT; ++i) {
        const uint32_t slot = x & 8191;
        const uint32_t ea = tab_s + 4 * slot;
        const uint32_t f = lds_u16(ea + 2), bi = lds_u16(ea);
        x = f * (x >> 13) + bi;
        x |= 0x800000;
    }
    t1 = clock64(); cyc[6] = t1 - t0; out[6] = x;

    // ---- encoder C: three candidates in parallel, select last
    x = (1u << 23) + 12345;
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N_IT; ++i) {
        const bool e1 = x >= b, e2 = x >= b2;
        const uint32_t a1 = x >> 8, a2 = x >> 16;
        const uint32_t q0 = __funnelshift_r(__umulhi(x, rcp), 0u, sh);
        const uint32_t q1 = __funnelshift_r(__umulhi(a1, rcp), 0u, sh);
        const uint32_t q2 = __funnelshift_r(__umulhi(a2, rcp), 0u, sh);
        const uint32_t y0 = q0 * cm + (x + bias), y1 = q1 * cm + (a1 + bias), y2 = q2 * cm + (a2 + bias);
        x = e2 ? y2 : (e1 ? y1 : y0);
        x = (x & 0x3fffffff) | 0x800000;
    }
    t1 = clock64(); cyc[7] = t1 - t0; out[7] = x;
    // ---- decoder E: select the table address (candidates' addresses in parallel)
    x = (1u << 23) + 777; pa = P_s; v = lds_u32(pa);
    uint32_t xs = x >> 13, ea = tab_s + 4 * (x & 8191);
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N_IT; ++i) {
        const uint32_t f = lds_u16(ea + 2), bi = lds_u16(ea);
        const uint32_t xn = f * xs + bi;
        const uint32_t x1 = __funnelshift_l(v, xn, 8), x2 = __funnelshift_l(v, xn, 16);
        const bool r1 = xn < (1u << 23), r2 = xn < (1u << 15);
        const uint32_t e0 = tab_s + 4 * (xn & 8191), e1 = tab_s + 4 * (x1 & 8191), e2 = tab_s + 4 * (x2 & 8191);
        ea = r1 ? (r2 ? e2 : e1) : e0;
        xs = r1 ? (r2 ? (x2 >> 13) : (x1 >> 13)) : (xn >> 13);
        pa += (r1 ? 4u : 0u) + (r2 ? 4u : 0u);
        pa = P_s + ((pa - P_s) & 16383);
        v = lds_u32(pa);
    }
    t1 = clock64(); cyc[8] = t1 - t0; out[8] = xs + ea;
}
int main() {
    uint32_t* o; long long* c; cudaMalloc(&o, 64); cudaMalloc(&c, 8 * 16);
    // f = 100, n = 14: bound = f << 17, rcp for f = 100: l = 7, rcp = ceil(2^38 / 100), shift 6
    uint32_t f = 100, b = f << 17, b2 = (b >= (1u << 24)) ? 0x80000000u : b << 8;
    unsigned long long m = ((1ull << 38) + f - 1) / f;
    for (int r = 0; r < 2; ++r) k<<<1, 32>>>(o, c, b, b2, (uint32_t)m, 6, (1u << 14) - f, 5);
    cudaDeviceSynchronize();
    long long h[16]; cudaMemcpy(h, c, 128, cudaMemcpyDeviceToHost);
    const char* nm[] = {"enc A (predicates)", "enc B (umax)", "clamp+imad only", "dec A (predicates)", "dec B (sign bits)", "dec C (clz)", "dec table-only", "enc C (3 cand)", "dec E (addr select)"};
    for (int i = 0; i < 9; ++i) printf("%-22s %.2f cycles per step\n", nm[i], (double)h[i] / N_IT);
    return 0;
}
