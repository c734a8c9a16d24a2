#include <cstdio>
#include <cstdint>
#define N_IT 20000
// one chain per CTA (lane 0 of warp 0), optional helper warps that spin on smem
__global__ void k(uint32_t* out, long long* cyc, uint32_t b, uint32_t b2, uint32_t rcp, uint32_t sh, uint32_t cm, uint32_t bias, int helpers_busy) {
    __shared__ volatile uint32_t flag;
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    if (threadIdx.x >= 32) {  // helper warps
        if (helpers_busy) { uint32_t acc = threadIdx.x; while (!flag) { acc = acc * 3 + 1; } out[1000 + threadIdx.x] = acc; }
        else { while (!flag) __nanosleep(200); }
        return;
    }
    if (threadIdx.x) return;
    uint32_t x = (1u << 23) + 12345 + blockIdx.x;
    long long t0 = clock64();
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
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x] = x;
    flag = 1;
}
int main() {
    uint32_t* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8 * 1024);
    uint32_t f = 100, b = f << 17, b2 = (b >= (1u << 24)) ? 0x80000000u : b << 8;
    unsigned long long m = ((1ull << 38) + f - 1) / f;
    for (int hb = 0; hb < 2; ++hb)
    for (int nw : {1, 3}) for (int nb : {148, 296, 444, 592}) {
        k<<<nb, nw * 32>>>(o, c, b, b2, (uint32_t)m, 6, (1u << 14) - f, 5, hb);
        cudaDeviceSynchronize();
        long long h[1024]; cudaMemcpy(h, c, nb * 8, cudaMemcpyDeviceToHost);
        double mx = 0, sum = 0; for (int i = 0; i < nb; ++i) { sum += h[i]; if (h[i] > mx) mx = h[i]; }
        printf("helpers %s warps/CTA %d CTAs %d: mean %.1f max %.1f cycles/step\n", hb ? "busy" : "sleep", nw, nb, sum / nb / N_IT, mx / N_IT);
    }
    return 0;
}
