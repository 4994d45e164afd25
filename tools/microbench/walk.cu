// walk.cu -- static unrolled walk over 64 window positions with a warp-uniform
// occupancy mask; each set position does 5 FFMA2.  Compares ptxas's
// if-converted (predicated) code against explicit skip branches, for mask
// densities 0.1 / 0.3 / 0.5.  Reports SM cycles per *useful* FFMA2 (ideal: 0.5
// per SMSP-issue... i.e. 2 pipe cycles / 4 SMSPs = 0.5).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void walk_kernel(float2* out, const unsigned long long* masks, int nmask, int reps, long long* cycles) {
    float2 acc[16];
#pragma unroll
    for (int i = 0; i < 16; i++) acc[i] = make_float2(threadIdx.x * 1e-3f, i);
    const float2 w0 = make_float2(0.999f, 1.001f), w1 = make_float2(1.0001f, 0.9999f);
    long long t0 = clock64();
    for (int r = 0; r < reps; r++) {
        unsigned long long m = masks[r % nmask];
        if (MODE == 1) m = __shfl_sync(0xffffffffu, m, 0);   // non-uniform-looking register
#pragma unroll
        for (int p = 0; p < 64; p++) {
            if ((m >> p) & 1ull) {
                const float2 vv = make_float2(1.0f + p * 1e-3f, 1.0f + p * 1e-3f);
                acc[p % 16] = __ffma2_rn(vv, w0, acc[p % 16]);
                acc[(p + 3) % 16] = __ffma2_rn(vv, w1, acc[(p + 3) % 16]);
                acc[(p + 5) % 16] = __ffma2_rn(vv, w0, acc[(p + 5) % 16]);
                acc[(p + 7) % 16] = __ffma2_rn(vv, w1, acc[(p + 7) % 16]);
                acc[(p + 11) % 16] = __ffma2_rn(vv, w0, acc[(p + 11) % 16]);
                if (MODE == 2) asm volatile("nanosleep.u32 0;");   // un-predicable: keeps the branch
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) s += acc[i].x + acc[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = make_float2(s, s);
}

int main() {
    const int nmask = 256, reps = 2000;
    unsigned long long h[nmask];
    float2* out;
    unsigned long long* dm;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * sizeof(float2));
    cudaMalloc(&dm, sizeof h);
    cudaMalloc(&cyc, 8);
    unsigned s = 12345;
    printf("[");
    bool first = true;
    for (double rho : {0.1, 0.3, 0.5}) {
        long long bits = 0;
        for (int i = 0; i < nmask; i++) {
            unsigned long long m = 0;
            for (int b = 0; b < 64; b++) {
                s = s * 1664525u + 1013904223u;
                if ((s >> 8) % 1000 < rho * 1000) m |= 1ull << b;
            }
            h[i] = m;
            bits += __builtin_popcountll(m);
        }
        cudaMemcpy(dm, h, sizeof h, cudaMemcpyHostToDevice);
        const double useful = 5.0 * (double)bits / nmask * reps;   // FFMA2 per warp
        for (int mode = 0; mode < 3; mode++) {
            for (int warps : {8, 16}) {
                if (mode == 0) walk_kernel<0><<<148, 32 * warps>>>(out, dm, nmask, reps, cyc);
                if (mode == 1) walk_kernel<1><<<148, 32 * warps>>>(out, dm, nmask, reps, cyc);
                if (mode == 2) walk_kernel<2><<<148, 32 * warps>>>(out, dm, nmask, reps, cyc);
                cudaDeviceSynchronize();
                long long c = 0;
                cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
                printf("%s{\"rho\": %.1f, \"mode\": %d, \"warps\": %d, \"sm_cycles_per_useful_ffma2\": %.3f}",
                       first ? "" : ", ", rho, mode, warps, (double)c / (useful * warps));
                first = false;
            }
        }
    }
    printf("]\n");
    return 0;
}
