#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* out, uint32_t a0, uint32_t b0, int iters, long long* cyc) {
    uint32_t x = a0, y = b0;
    __shared__ uint32_t sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = (i * 2654435761u) & 4095;
    __syncthreads();
    long long t0, t1;
    // 1 IMAD chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = x * b0 + y; x = x * b0 + y; x = x * b0 + y; x = x * b0 + y; }
    t1 = clock64(); cyc[0] = t1 - t0; out[0] = x;
    // 2 IMAD.HI chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = __umulhi(x, b0) + y; x = __umulhi(x, b0) + y; x = __umulhi(x, b0) + y; x = __umulhi(x, b0) + y; }
    t1 = clock64(); cyc[1] = t1 - t0; out[1] = x;
    // 3 SHF.R.W chain (funnel)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = __funnelshift_r(x, y, x); x = __funnelshift_r(x, y, x); x = __funnelshift_r(x, y, x); x = __funnelshift_r(x, y, x); }
    t1 = clock64(); cyc[2] = t1 - t0; out[2] = x;
    // 4 LDS chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = sm[x & 4095]; x = sm[x & 4095]; x = sm[x & 4095]; x = sm[x & 4095]; }
    t1 = clock64(); cyc[3] = t1 - t0; out[3] = x;
    // 5 compare + select chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = (x >= b0) ? x + y : x ^ y; x = (x >= b0) ? x + y : x ^ y; x = (x >= b0) ? x + y : x ^ y; x = (x >= b0) ? x + y : x ^ y; }
    t1 = clock64(); cyc[4] = t1 - t0; out[4] = x;
    // 6 IADD3/LOP chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = (x ^ y) + b0; x = (x ^ y) + b0; x = (x ^ y) + b0; x = (x ^ y) + b0; }
    t1 = clock64(); cyc[5] = t1 - t0; out[5] = x;
    // 7 SHF.R.U32 (variable) chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = (x >> (y & 7)) | b0; x = (x >> (y & 7)) | b0; x = (x >> (y & 7)) | b0; x = (x >> (y & 7)) | b0; }
    t1 = clock64(); cyc[6] = t1 - t0; out[6] = x;
}
int main() {
    uint32_t* o; long long* c; cudaMalloc(&o, 64); cudaMalloc(&c, 8 * 8);
    int iters = 10000;
    k<<<1, 32>>>(o, 12345, 2654435761u, iters, c);
    k<<<1, 32>>>(o, 12345, 2654435761u, iters, c);
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    const char* nm[] = {"imad", "imad.hi+iadd", "shf.r.w", "lds", "isetp+sel(+iadd)", "lop3+iadd", "shf+lop"};
    for (int i = 0; i < 7; ++i) printf("%-20s %.2f cycles per op\n", nm[i], (double)h[i] / (iters * 4));
    return 0;
}
