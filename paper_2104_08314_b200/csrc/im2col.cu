// im2col.cu -- dense comparison baseline: im2col lowering + GEMM.
//
// Lowering: L[n][c*R*S + l*S + m][y*Ow + x] = xp[n][c][y*sh + l][x*sw + m]
// (SI Eq. 6 elements per image), written coalesced along the output position.
// GEMM: y[n] (K x P) = W (K x CRS) * L[n] (CRS x P), P = Oh*Ow, FP32.
#include "common.cuh"

namespace spc {

__global__ void im2col_kernel(Geom g, const float* __restrict__ x, float* __restrict__ L) {
    const long long P = (long long)g.Oh * g.Ow;
    const long long RS = (long long)g.R * g.S;
    const long long total = (long long)g.N * g.C * RS * P;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long p = i % P;
        const long long row = i / P;           // n*CRS + crs
        const long long crs = row % (g.C * RS);
        const int n = (int)(row / (g.C * RS));
        const int c = (int)(crs / RS);
        const int l = (int)((crs % RS) / g.S), m = (int)(crs % g.S);
        const int oy = (int)(p / g.Ow), ox = (int)(p % g.Ow);
        const int h = oy * g.sh + l - g.pt, w = ox * g.sw + m - g.pl;
        float v = 0.f;
        if (h >= 0 && h < g.H && w >= 0 && w < g.W) v = __ldg(x + (((long long)n * g.C + c) * g.H + h) * g.W + w);
        L[i] = v;
    }
}

cudaError_t launch_im2col(const Geom& g, const float* x, float* L, cudaStream_t st) {
    long long total = (long long)g.N * g.C * g.R * g.S * g.Oh * g.Ow;
    long long nb = (total + 255) / 256; int blocks = (int)(nb < 148 * 16 ? nb : 148 * 16);
    im2col_kernel<<<blocks, 256, 0, st>>>(g, x, L);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- SGEMM
// C[z] (M x N) = A (M x Kd) * B[z] (Kd x N), all row-major, FP32 FFMA.
// 128 x 128 CTA tile, BK = 8, 256 threads with 8 x 8 register tiles,
// double-buffered shared memory, guarded edges.
constexpr int BM = 128, BN = 128, BK = 8;

__global__ void __launch_bounds__(256) sgemm_kernel(int M, int N, int Kd, const float* __restrict__ A,
                                                    const float* __restrict__ B, long long strideB,
                                                    float* __restrict__ C, long long strideC, int relu) {
    __shared__ __align__(16) float As[2][BK][BM];
    __shared__ __align__(16) float Bs[2][BK][BN];
    const int tid = threadIdx.x;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    B += blockIdx.z * strideB;
    C += blockIdx.z * strideC;
    // load mapping: A tile 128 x 8 -> thread loads 4 elements of row (tid>>1), cols (tid&1)*4..
    const int ar = tid >> 1, ac = (tid & 1) * 4;
    // B tile 8 x 128 -> thread loads row (tid>>5), cols (tid&31)*4..
    const int br = tid >> 5, bc = (tid & 31) * 4;
    float ra[4], rb[4];
    auto load_tile = [&](int k0) {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int gm = m0 + ar, gk = k0 + ac + i;
            ra[i] = (gm < M && gk < Kd) ? __ldg(A + (long long)gm * Kd + gk) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int gk = k0 + br, gn = n0 + bc + i;
            rb[i] = (gk < Kd && gn < N) ? __ldg(B + (long long)gk * N + gn) : 0.f;
        }
    };
    auto store_tile = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 4; i++) As[buf][ac + i][ar] = ra[i];
        *reinterpret_cast<float4*>(&Bs[buf][br][bc]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
    };
    const int tr = (tid >> 4) * 4, tc = (tid & 15) * 4;   // two 4x4 quadrants at +64
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[i][j] = 0.f;
    load_tile(0);
    store_tile(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < Kd; k0 += BK) {
        const bool more = k0 + BK < Kd;
        if (more) load_tile(k0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; kk++) {
            float a[8], b[8];
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][tr]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][tr + 64]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tc]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tc + 64]);
            a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w; a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
            b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w; b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 8; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (more) {
            store_tile(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int gm = m0 + tr + (i < 4 ? i : 60 + i);
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int gn = n0 + tc + (j < 4 ? j : 60 + j);
            if (gn >= N) continue;
            float v = acc[i][j];
            if (relu) v = fmaxf(v, 0.f);
            C[(long long)gm * N + gn] = v;
        }
    }
}

cudaError_t launch_gemm(const Geom& g, const float* w, const float* L, float* y, int relu, cudaStream_t st) {
    const int M = g.K, N = g.Oh * g.Ow, Kd = g.C * g.R * g.S;
    dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, g.N);
    sgemm_kernel<<<grid, 256, 0, st>>>(M, N, Kd, w, L, (long long)Kd * N, y, (long long)M * N, relu);
    return cudaGetLastError();
}

}  // namespace spc
