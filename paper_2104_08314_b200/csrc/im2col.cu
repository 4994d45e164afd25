// im2col.cu -- dense comparison baseline: im2col lowering + GEMM.
//
// Lowering: L[n][c*R*S + l*S + m][y*Ow + x] = xp[n][c][y*sh + l][x*sw + m]
// (SI Eq. 6 elements per image), written coalesced along the output position.
// GEMM: y[n] (K x P) = W (K x CRS) * L[n] (CRS x P), P = Oh*Ow, FP32.
#include <algorithm>
#include <cstdlib>
#include <cublas_v2.h>
#include <mutex>

#include "common.cuh"

namespace spc {

static int g_gemm = SPC_GEMM_AUTO;   // im2col GEMM engine (spc_set_im2col_gemm)

// The engine a layer actually runs: AUTO picks the tcgen05 kernel for layers of >= 2^28
// MACs, or >= 2^26 MACs spread over >= 20 output tiles (128 positions x 64 / 128 channels)
// or with long tiles (C*R*S >= 2048) -- measured (lowering + GEMM, graph, L2 flushed):
// cfg2 (1.2e8 MACs, 25 tiles) 26.7 vs 28.7 us for cuBLAS FP32, cfg3 s2 (2.3e8, 8 tiles,
// CRS 2304) 61 vs 68, cfg3 61 vs 98; Inception 1x3 @8 (2.3e8 MACs, 12 tiles, CRS 1152)
// 41 vs 39, cfg1 (4.5e5 MACs) 16 vs 12.
static int effective_engine(const Geom& g) {
    if (g_gemm != SPC_GEMM_AUTO) return g_gemm;
    const double macs = (double)g.N * g.Oh * g.Ow * g.K * g.C * g.R * g.S;
    const long long mt = ((long long)g.N * g.Oh * g.Ow + 127) / 128, bn = g.K <= 64 ? 64 : 128;
    const long long tiles = mt * ((g.K + bn - 1) / bn);
    const bool mid = macs >= 67108864.0 && (tiles >= 20 || g.C * g.R * g.S >= 2048);
    return (macs >= 268435456.0 || mid) ? SPC_GEMM_TC_3XTF32 : SPC_GEMM_CUBLAS_FP32;
}

// Block (32, 8): threadIdx.x strides 32 consecutive output positions of a lowered row
// (coalesced 128-byte stores), threadIdx.y picks one of 8 rows; rows = (n, c, l, m).
__global__ void __launch_bounds__(256) im2col_kernel(Geom g, const float* __restrict__ x, float* __restrict__ L) {
    const int RS = g.R * g.S;
    const long long rows = (long long)g.N * g.C * RS;
    const int P = g.Oh * g.Ow;
    const int p = blockIdx.x * 32 + threadIdx.x;
    const int oy = p / g.Ow, ox = p - oy * g.Ow;
    for (long long row = (long long)blockIdx.y * 8 + threadIdx.y; row < rows; row += (long long)gridDim.y * 8) {
        const long long nc = row / RS;
        const int rs = (int)(row - nc * RS);
        const int l = rs / g.S, m = rs - l * g.S;
        const int h = oy * g.sh + l - g.pt, w = ox * g.sw + m - g.pl;
        if (p < P)
            L[row * P + p] = (h >= 0 && h < g.H && w >= 0 && w < g.W) ? __ldg(x + (nc * g.H + h) * g.W + w) : 0.f;
    }
}

// Large Oh*Ow: one block row per lowered row, threads stride its positions.
__global__ void __launch_bounds__(256) im2col_row_kernel(Geom g, const float* __restrict__ x, float* __restrict__ L) {
    const int RS = g.R * g.S;
    const long long row = blockIdx.y + (long long)blockIdx.z * gridDim.y;   // n*CRS + crs
    const long long nc = row / RS;
    const int rs = (int)(row - nc * RS);
    const int l = rs / g.S, m = rs - l * g.S;
    const int P = g.Oh * g.Ow;
    const float* xc = x + nc * g.H * (long long)g.W;
    float* Lr = L + row * P;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
        const int oy = p / g.Ow, ox = p - oy * g.Ow;
        const int h = oy * g.sh + l - g.pt, w = ox * g.sw + m - g.pl;
        Lr[p] = (h >= 0 && h < g.H && w >= 0 && w < g.W) ? __ldg(xc + h * g.W + w) : 0.f;
    }
}

// K-major lowering for the tensor-core engine: A[m][crs] with m = n*P + p (one GEMM row per
// image position, all images in one GEMM).  A block owns 32 positions x kTcCB input channels:
// warps read x with lanes along the positions (coalesced; tap offsets by increment, no
// divisions) into a column-major smem tile, then write each position's C*R*S slice with
// lanes along CRS (coalesced 128-byte rows).  The tile is [CB*R*S][33] so both phases are
// bank-conflict free.
constexpr int kTcCB = 64;
template <int R_, int S_>   // compile-time taps (all loads of a channel in flight), or 0, 0: runtime
__global__ void __launch_bounds__(256) im2col_t_kernel(Geom g, const float* __restrict__ x, float* __restrict__ A,
                                                       int cb) {
    extern __shared__ float tile[];               // [cb * RS][33]
    const int R = R_ ? R_ : g.R, S = S_ ? S_ : g.S;
    const int P = g.Oh * g.Ow, RS = R * S, CRS = g.C * RS;
    const long long M = (long long)g.N * P;
    const long long m0 = (long long)blockIdx.x * 32;
    const int c0 = blockIdx.y * cb;
    const int nc = min(cb, g.C - c0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    {
        const long long m = m0 + lane;
        const bool mok = m < M;
        const int n = mok ? (int)(m / P) : 0, p = mok ? (int)(m - (long long)n * P) : 0;
        const int oy = p / g.Ow, ox = p - oy * g.Ow;
        const int h0 = oy * g.sh - g.pt, w0 = ox * g.sw - g.pl;
#pragma unroll 4
        for (int ci = warp; ci < nc; ci += 8) {
            const float* xc = x + ((long long)n * g.C + c0 + ci) * g.H * g.W;
            float* tc = tile + ci * RS * 33 + lane;
            if constexpr (R_ > 0) {
                float v[R_ * S_];
#pragma unroll
                for (int l = 0; l < R_; l++) {
                    const int h = h0 + l;
                    const bool hok = mok && h >= 0 && h < g.H;
#pragma unroll
                    for (int mm = 0; mm < S_; mm++) {
                        const int w = w0 + mm;
                        v[l * S_ + mm] = (hok && w >= 0 && w < g.W) ? __ldg(xc + h * g.W + w) : 0.f;
                    }
                }
#pragma unroll
                for (int t = 0; t < R_ * S_; t++) tc[t * 33] = v[t];
            } else {
                int t = 0;
                for (int l = 0; l < R; l++) {
                    const int h = h0 + l;
                    const bool hok = mok && h >= 0 && h < g.H;
                    for (int mm = 0; mm < S; mm++, t++) {
                        const int w = w0 + mm;
                        tc[t * 33] = (hok && w >= 0 && w < g.W) ? __ldg(xc + h * g.W + w) : 0.f;
                    }
                }
            }
        }
    }
    __syncthreads();
    const int row = nc * RS;
    for (int pp = warp; pp < 32; pp += 8) {
        const long long m = m0 + pp;
        if (m >= M) break;
        float* dst = A + m * CRS + (long long)c0 * RS;
        for (int col = lane; col < row; col += 32) dst[col] = tile[col * 33 + pp];
    }
}

// The tensor-core engine runs when TMA can address the operands (CRS % 4 == 0: 16-byte row
// pitches); other shapes fall back to cuBLAS FP32 with the standard lowering.
bool tc_layout(const Geom& g) { return effective_engine(g) == SPC_GEMM_TC_3XTF32 && (g.C * g.R * g.S) % 4 == 0; }

cudaError_t launch_im2col(const Geom& g, const float* x, float* L, cudaStream_t st) {
    if (tc_layout(g)) {
        const long long M = (long long)g.N * g.Oh * g.Ow;
        const int RS = g.R * g.S;
        // channels per block: longer contiguous row segments per position write faster
        // (batch-256 cfg5-L0: 32 -> 496 us, 64 -> 467 us; 128 is slower: 1 block/SM)
        // (larger taps: 5x5 @35 is faster with 12 channels, 42 KB, than with 25, 82 KB)
        const int cb = (RS <= 9) ? std::min(kTcCB, 640 / RS) : std::max(1, std::min(32, 320 / RS));
        const size_t smem = (size_t)cb * RS * 33 * sizeof(float);
        auto kern = (g.R == 3 && g.S == 3) ? im2col_t_kernel<3, 3>
                  : (g.R == 1 && g.S == 7) ? im2col_t_kernel<1, 7>
                  : (g.R == 7 && g.S == 1) ? im2col_t_kernel<7, 1> : im2col_t_kernel<0, 0>;
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
        }
        kern<<<dim3((unsigned)((M + 31) / 32), (g.C + cb - 1) / cb), 256, smem, st>>>(g, x, L, cb);
        return cudaGetLastError();
    }
    const long long rows = (long long)g.N * g.C * g.R * g.S;
    const int P = g.Oh * g.Ow;
    if (P >= 512) {
        long long rz = 1;
        while ((rows + rz - 1) / rz > 65535 || rows % rz) rz++;
        const int bx = std::min(8, (P + 255) / 256);
        im2col_row_kernel<<<dim3(bx, (unsigned)(rows / rz), (unsigned)rz), 256, 0, st>>>(g, x, L);
        return cudaGetLastError();
    }
    const long long ry = std::min<long long>((rows + 7) / 8, 65535);
    im2col_kernel<<<dim3((P + 31) / 32, (unsigned)ry), dim3(32, 8), 0, st>>>(g, x, L);
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

__global__ void relu_kernel(float* y, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = fmaxf(y[i], 0.f);
}


int gemm_engine() { return g_gemm; }
int gemm_engine_for(const Geom& g) {
    const int e = effective_engine(g);
    return (e == SPC_GEMM_TC_3XTF32 && (g.C * g.R * g.S) % 4 != 0) ? SPC_GEMM_CUBLAS_FP32 : e;
}
void set_gemm_engine(int e) { g_gemm = e; }

// one cuBLAS handle per device, created on first use (cuBLAS calls are stream-ordered
// and capturable in CUDA graphs; the handle is only re-bound to the caller's stream)
static cublasHandle_t cublas_handle(int dev) {
    static std::mutex mu;
    static cublasHandle_t h[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!h[dev] && cublasCreate(&h[dev]) != CUBLAS_STATUS_SUCCESS) h[dev] = nullptr;
    return h[dev];
}

// y[n] (K x P, row-major) = W (K x CRS) * L[n] (CRS x P).  Column-major view for cuBLAS:
// y^T (P x K, ld P) = L^T (P x CRS, ld P) * W^T (CRS x K, ld CRS), batched over n (W stride 0).
static cudaError_t cublas_gemm(const Geom& g, const float* w, const float* L, float* y, int relu, cudaStream_t st,
                               int engine) {
    int dev = 0;
    cudaGetDevice(&dev);
    cublasHandle_t h = cublas_handle(dev);
    if (!h) return cudaErrorNotSupported;
    if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
    const int P = g.Oh * g.Ow, K = g.K, CRS = g.C * g.R * g.S;
    const float one = 1.f, zero = 0.f;
    cublasComputeType_t ct = CUBLAS_COMPUTE_32F;
    if (engine == SPC_GEMM_CUBLAS_BF16X9) ct = CUBLAS_COMPUTE_32F_EMULATED_16BFX9;
    if (engine == SPC_GEMM_CUBLAS_TF32) ct = CUBLAS_COMPUTE_32F_FAST_TF32;
    cublasStatus_t s = cublasGemmStridedBatchedEx(
        h, CUBLAS_OP_N, CUBLAS_OP_N, P, K, CRS, &one, L, CUDA_R_32F, P, (long long)CRS * P, w, CUDA_R_32F, CRS, 0,
        &zero, y, CUDA_R_32F, P, (long long)K * P, g.N, ct, CUBLAS_GEMM_DEFAULT);
    // the cuBLAS loaded in the process may predate an engine (BF16x9 needs cuBLAS >= 12.9;
    // PyTorch bundles 12.8): report it as unsupported rather than as a CUDA fault
    if (s == CUBLAS_STATUS_INVALID_VALUE || s == CUBLAS_STATUS_NOT_SUPPORTED) return cudaErrorNotSupported;
    if (s != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
    if (relu) {
        const long long n = (long long)g.N * K * P;
        relu_kernel<<<(int)std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, st>>>(y, n);
    }
    return cudaGetLastError();
}

cudaError_t launch_gemm(const Geom& g, const float* w, const float* L, float* y, int relu, cudaStream_t st,
                        float* extra, size_t extra_bytes) {
    const int eng = effective_engine(g);
    if (eng == SPC_GEMM_TC_3XTF32) {
        const size_t need = (size_t)4 * g.K * g.C * g.R * g.S;   // the weights' lo half
        if (tc_layout(g)) return launch_tc_gemm(g, w, L, y, relu, st, extra_bytes >= need ? extra : nullptr);
        return cublas_gemm(g, w, L, y, relu, st, SPC_GEMM_CUBLAS_FP32);
    }
    if (eng != SPC_GEMM_SIMT) return cublas_gemm(g, w, L, y, relu, st, eng);
    const int M = g.K, N = g.Oh * g.Ow, Kd = g.C * g.R * g.S;
    dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, g.N);
    sgemm_kernel<<<grid, 256, 0, st>>>(M, N, Kd, w, L, (long long)Kd * N, y, (long long)M * N, relu);
    return cudaGetLastError();
}

}  // namespace spc
