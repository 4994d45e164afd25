// tc_probe.cu -- layout probe for tcgen05.mma kind::tf32 with no-swizzle descriptors:
// one CTA, D (128 x 64) = A (128 x 16) * B (64 x 16)^T, integer data (exact), several
// descriptor/layout variants; prints the max error of each against a CPU reference.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(unsigned a, unsigned lbo, unsigned sbo) {
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__global__ void probe(const float* A, const float* B, float* D, int var) {
    // A: [128][16] row-major (m, k); B: [64][16] (n, k); D: [128][64]
    __shared__ __align__(1024) float sa[128 * 16];
    __shared__ __align__(1024) float sb[64 * 16];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ unsigned tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool aK = var & 1;
    // A layout
    for (int i = tid; i < 128 * 16; i += 128) {
        const int m = i / 16, k = i % 16;
        int off;
        if (aK) off = ((k / 4) * (128 / 8) * 128 + (m / 8) * 128 + (m % 8) * 16 + (k % 4) * 4) / 4;  // K-major
        else off = ((k / 8) * (128 / 4) * 128 + (m / 4) * 128 + (k % 8) * 16 + (m % 4) * 4) / 4;     // MN-major
        sa[off] = A[i];
    }
    for (int i = tid; i < 64 * 16; i += 128) {
        const int n = i / 16, k = i % 16;
        sb[((k / 4) * (64 / 8) * 128 + (n / 8) * 128 + (n % 8) * 16 + (k % 4) * 4) / 4] = B[i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tm = tbase;
    if (tid == 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((aK ? 0u : 1u) << 15) | (0u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
        for (int ks = 0; ks < 2; ks++) {
            unsigned alb, asb, aaddr;
            if (aK) { alb = (128 / 8) * 128; asb = 128; aaddr = su32(sa) + 2 * ks * alb; }
            else { alb = (128 / 4) * 128; asb = 128; aaddr = su32(sa) + ks * alb; }
            if (var & 2) { unsigned t = alb; alb = asb; asb = t; }
            unsigned blb = (64 / 8) * 128, bsb = 128;
            const unsigned baddr = su32(sb) + 2 * ks * blb;
            if (var & 4) { unsigned t = blb; blb = bsb; bsb = t; }
            const uint64_t da = desc(aaddr, alb, asb), db = desc(baddr, blb, bsb);
            const unsigned acc = ks ? 1u : 0u;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    }
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t r[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(tm + ((unsigned)(warp * 32) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; j++) D[(warp * 32 + lane) * 64 + c0 + j] = __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
}

int main() {
    float hA[128 * 16], hB[64 * 16], hD[128 * 64], ref[128 * 64];
    for (int i = 0; i < 128 * 16; i++) hA[i] = (float)((i * 7 + 3) % 9 - 4);
    for (int i = 0; i < 64 * 16; i++) hB[i] = (float)((i * 5 + 1) % 7 - 3);
    for (int m = 0; m < 128; m++)
        for (int n = 0; n < 64; n++) {
            float s = 0;
            for (int k = 0; k < 16; k++) s += hA[m * 16 + k] * hB[n * 16 + k];
            ref[m * 64 + n] = s;
        }
    float *A, *B, *D;
    cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
    cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
    for (int var = 0; var < 8; var++) {
        cudaMemset(D, 0, sizeof hD);
        probe<<<1, 128>>>(A, B, D, var);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
        double err = 0;
        for (int i = 0; i < 128 * 64; i++) err = fmax(err, fabs(hD[i] - ref[i]));
        printf("var %d (A %s, swapA %d, swapB %d): max err %g  [%s]  D[0]=%g ref %g D[65]=%g ref %g\n", var, (var & 1) ? "K-major" : "MN-major",
               (var >> 1) & 1, (var >> 2) & 1, err, cudaGetErrorString(e), hD[0], ref[0], hD[65], ref[65]);
        if (e != cudaSuccess) break;
    }
    return 0;
}
