// brx_chain.cu -- cost of a warp-uniform brx.idx dispatch chain on sm_100a:
// a list of case indices in shared memory, each case body 4 FFMA2, threaded
// dispatch (load next entry -> brx).  Reports cycles per dispatch at several
// warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void brx_kernel(float2* out, int n, int reps, long long* cycles) {
    __shared__ int lst[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) lst[i] = (i * 7 + 3) % 8;
    lst[n] = 8;   // sentinel
    __syncthreads();
    unsigned long long a0 = 0, a1 = 0, a2 = 0, a3 = 0, w = 0x3f8000003f800000ull;
    const unsigned base = (unsigned)__cvta_generic_to_shared(lst);
    long long t0 = clock64();
    for (int r = 0; r < reps; r++) {
        asm volatile(
            "{\n"
            ".reg .b32 p, c; .reg .b64 vv;\n"
            "mov.b32 p, %5;\n"
            "mov.b64 vv, %4;\n"
            "$T%=: .branchtargets $C0%=, $C1%=, $C2%=, $C3%=, $C4%=, $C5%=, $C6%=, $C7%=, $D%=;\n"
            "ld.shared.b32 c, [p]; add.u32 p, p, 4; brx.idx.uni c, $T%=;\n"
            "$C0%=: fma.rn.f32x2 %0, vv, %4, %0; fma.rn.f32x2 %1, vv, %4, %1; fma.rn.f32x2 %2, vv, %4, %2; fma.rn.f32x2 %3, vv, %4, %3; ld.shared.b32 c, [p]; add.u32 p, p, 4; brx.idx.uni c, $T%=;\n"
            "$C1%=: fma.rn.f32x2 %1, vv, %4, %1; fma.rn.f32x2 %2, vv, %4, %2; fma.rn.f32x2 %3, vv, %4, %3; fma.rn.f32x2 %0, vv, %4, %0; ld.shared.b32 c, [p]; add.u32 p, p, 4; brx.idx.uni c, $T%=;\n"
            "$C2%=: fma.rn.f32x2 %2, vv, %4, %2; fma.rn.f32x2 %3, vv, %4, %3; fma.rn.f32x2 %0, vv, %4, %0; fma.rn.f32x2 %1, vv, %4, %1; ld.shared.b32 c, [p]; add.u32 p, p, 4; brx.idx.uni c, $T%=;\n"
            "$C3%=: fma.rn.f32x2 %3, vv, %4, %3; fma.rn.f32x2 %0, vv, %4, %0; fma.rn.f32x2 %1, vv, %4, %1; fma.rn.f32x2 %2, vv, %4, %2; ld.shared.b32 c, [p]; add.u32 p, p, 4; brx.idx.uni c, $T%=;\n"
            "$C4%=: fma.rn.f32x2 %0, vv, %4, %0; fma.rn.f32x2 %2, vv, %4, %2; fma.rn.f32x2 %1, vv, %4, %1; fma.rn.f32x2 %3, vv, %4, %3; ld.shared.b32 c, [p]; add.u32 p, p, 4; brx.idx.uni c, $T%=;\n"
            "$C5%=: fma.rn.f32x2 %1, vv, %4, %1; fma.rn.f32x2 %3, vv, %4, %3; fma.rn.f32x2 %0, vv, %4, %0; fma.rn.f32x2 %2, vv, %4, %2; ld.shared.b32 c, [p]; add.u32 p, p, 4; brx.idx.uni c, $T%=;\n"
            "$C6%=: fma.rn.f32x2 %2, vv, %4, %2; fma.rn.f32x2 %0, vv, %4, %0; fma.rn.f32x2 %3, vv, %4, %3; fma.rn.f32x2 %1, vv, %4, %1; ld.shared.b32 c, [p]; add.u32 p, p, 4; brx.idx.uni c, $T%=;\n"
            "$C7%=: fma.rn.f32x2 %3, vv, %4, %3; fma.rn.f32x2 %1, vv, %4, %1; fma.rn.f32x2 %2, vv, %4, %2; fma.rn.f32x2 %0, vv, %4, %0; ld.shared.b32 c, [p]; add.u32 p, p, 4; brx.idx.uni c, $T%=;\n"
            "$D%=:\n"
            "}\n"
            : "+l"(a0), "+l"(a1), "+l"(a2), "+l"(a3)
            : "l"(w), "r"(base));
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = make_float2(__uint_as_float((unsigned)(a0 ^ a1)), __uint_as_float((unsigned)(a2 ^ a3)));
}

int main() {
    const int n = 1000, reps = 50;
    float2* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * sizeof(float2));
    cudaMalloc(&cyc, 8);
    printf("[");
    for (int warps : {1, 4, 8, 16, 32}) {
        brx_kernel<<<148, 32 * warps>>>(out, n, reps, cyc);
        cudaDeviceSynchronize();
        long long c = 0;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%s{\"warps_per_sm\": %d, \"cycles_per_dispatch_per_warp\": %.1f, \"sm_cycles_per_dispatch\": %.2f}",
               warps == 1 ? "" : ", ", warps, (double)c / (n * reps), (double)c / (n * reps) / warps);
    }
    printf("]\n");
    return 0;
}
