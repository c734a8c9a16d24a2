#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* out, long long spin) {
    uint32_t wid, sm;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    if ((threadIdx.x & 31) == 0) out[(blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32) * 2] = wid, out[(blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32) * 2 + 1] = sm;
    long long t0 = clock64(); while (clock64() - t0 < spin) {}
}
int main() {
    uint32_t* d; cudaMalloc(&d, 1 << 20);
    for (int wpb : {3, 4, 6}) {
        int B = 256;
        k<<<B, wpb * 32, 34000>>>(d, 2000000);
        cudaDeviceSynchronize();
        uint32_t h[256 * 6 * 2]; cudaMemcpy(h, d, B * wpb * 8, cudaMemcpyDeviceToHost);
        // per SM: SMSPs of warp 0 of each CTA
        int cnt[148][4] = {}; int ctas[148] = {};
        for (int b = 0; b < B; ++b) { uint32_t wid = h[(b * wpb) * 2], sm = h[(b * wpb) * 2 + 1]; cnt[sm][wid % 4]++; ctas[sm]++; }
        int coll = 0, multi = 0;
        for (int s = 0; s < 148; ++s) { if (ctas[s] > 1) multi++; for (int q = 0; q < 4; ++q) if (cnt[s][q] > 1) coll++; }
        printf("wpb %d: SMs with >1 CTA %d, SMSP collisions of warp 0 %d; sample warpids of CTA 0..5:", wpb, multi, coll);
        for (int b = 0; b < 6; ++b) printf(" (sm %u w %u)", h[(b * wpb) * 2 + 1], h[(b * wpb) * 2]);
        printf("\n");
    }
    return 0;
}
