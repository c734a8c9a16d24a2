#include <cstdio>
#include <cstdint>
#define N 20000
__global__ void k(uint32_t* out, long long* cyc, uint32_t seed) {
    uint32_t x = seed + threadIdx.x;
    long long t0, t1;
    // 1: ISETP -> VOTE -> (use)
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) { uint32_t b = __ballot_sync(0xffffffffu, (x & 1) != 0); x = b + threadIdx.x; }
    t1 = clock64(); cyc[0] = t1 - t0; out[0] = x;
    // 2: POPC chain
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) { x = __popc(x) + 0x12345u; }
    t1 = clock64(); cyc[1] = t1 - t0; out[1] = x;
    // 3: SHFL chain
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) { x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1; }
    t1 = clock64(); cyc[2] = t1 - t0; out[2] = x;
    // 4: ISETP -> VOTE -> POPC(& mask) -> IADD chain (the placement chain)
    const uint32_t ltm = (1u << (threadIdx.x & 31)) - 1;
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) { uint32_t b = __ballot_sync(0xffffffffu, x > 0x80000000u); x = x * 0x9E3779B1u + __popc(b & ltm); }
    t1 = clock64(); cyc[3] = t1 - t0; out[3] = x;
    // 5: reduce.add (REDUX) chain
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) { x = __reduce_add_sync(0xffffffffu, x & 0xff) + threadIdx.x; }
    t1 = clock64(); cyc[4] = t1 - t0; out[4] = x;
}
int main() {
    uint32_t* o; long long* c; cudaMalloc(&o, 64); cudaMalloc(&c, 64);
    k<<<1, 32>>>(o, c, 7); k<<<1, 32>>>(o, c, 7); cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    const char* nm[] = {"vote (+iadd)", "popc (+iadd)", "shfl (+iadd)", "isetp+vote+lop+popc+imad", "redux.add (+lop,iadd)"};
    for (int i = 0; i < 5; ++i) printf("%-28s %.1f cycles per iteration\n", nm[i], (double)h[i] / N);
    return 0;
}
