// tcgemm.cu -- dense baseline GEMM on the 5th-generation tensor cores (tcgen05, sm_100a):
// fp32 accuracy from three TF32 products (3xTF32), accumulators in TMEM.
//
// The im2col baseline computes y[n] (K x P) = W (K x CRS) * L[n]
// (CRS x P).  Here the GEMM is laid out as D (P x K) = L^T (P x CRS) * W^T (CRS x K):
//   * MMA M = 128 output positions (TMEM lane = position), N = BN output channels
//     (TMEM column), K-step 8 (kind::tf32);
//   * A = L^T tile and B = W^T tile, both K-major (CRS contiguous) in the canonical
//     no-swizzle UMMA layout (8-row x 16-byte core matrices); A is transposed while it is
//     staged (thread = position, coalesced loads along positions);
//   * every fp32 operand x is split into hi = x with the 13 low mantissa bits cleared
//     (exactly representable in tf32) and lo = x - hi (exact); D += Ahi*Bhi + Ahi*Blo +
//     Alo*Bhi, whose dropped term Alo*Blo is ~2^-22 relative -- inside the 1e-4 fp32
//     tolerance of north_star, unlike a single TF32 product;
//   * 128 threads stage the hi/lo tiles through registers (the split needs ALU work, so
//     no TMA here) into canonical no-swizzle UMMA layouts, two stages; one elected thread
//     issues the 6 MMAs of a stage and commits them to the stage's mbarrier; the epilogue
//     reads TMEM with tcgen05.ld (lane = position) and stores y coalesced along positions.
#include <algorithm>

#include "common.cuh"

namespace spc {
namespace {

constexpr int TM = 128;      // MMA M (positions)
constexpr int TBK = 16;      // CRS elements per stage
constexpr int TTHREADS = 128;

__device__ __forceinline__ uint64_t umma_desc(unsigned saddr, unsigned lbo, unsigned sbo) {
    // SmemDescriptor (sm_100): start [0,14), LBO [16,30), SBO [32,46) in 16-byte units,
    // version 1 at [46,48), base offset 0, layout SWIZZLE_NONE (0) at [61,64)
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// round to the nearest tf32 (cvt.rna): hi = rn(x), lo = rn(x - hi); x - hi is exact in fp32
__device__ __forceinline__ float tf32_rn(float x) {
    unsigned r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ float tf32_hi(float x) { return tf32_rn(x); }

template <int BN>
__global__ void __launch_bounds__(TTHREADS) tc_gemm_kernel(int P, int K, int CRS, int nimg,
                                                           const float* __restrict__ L,
                                                           const float* __restrict__ W, float* __restrict__ y,
                                                           int relu) {
    constexpr int A_BYTES = TM * TBK * 4;           // one of hi / lo
    constexpr int B_BYTES = BN * TBK * 4;
    constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
    constexpr unsigned A_LBO = (TM / 8) * 128;      // between 4-element K chunks (K-major)
    constexpr unsigned A_SBO = 128;                 // between 8-position groups
    constexpr unsigned B_LBO = (BN / 8) * 128;      // between 4-element K chunks (K-major)
    constexpr unsigned B_SBO = 128;                 // between 8-row output-channel groups
    // instruction descriptor: D f32, A/B tf32, both K-major, N = BN, M = 128
    constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) |
                               ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar[2];
    __shared__ unsigned tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5;
    // GEMM rows m = (image, position) pairs of all images (the weights are shared), so a
    // tile may straddle two images; thread tid owns row m0 + tid
    const long long m0 = (long long)blockIdx.x * TM, NP = (long long)nimg * P;
    const int n0 = blockIdx.y * BN;
    const long long mrow = m0 + tid;
    const int img_t = (int)(mrow / P), p_t = (int)(mrow - (long long)img_t * P);
    const bool row_ok = mrow < NP;
    const float* Lrow = L + (size_t)(row_ok ? img_t : 0) * CRS * P + p_t;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(&tmem_base_s)), "r"((unsigned)(BN < 32 ? 32 : BN)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_base_s;
    const unsigned sbase = smem_u32(smem);
    const bool vecB = (CRS % 4) == 0;

    const int nk = (CRS + TBK - 1) / TBK;
    for (int it = 0; it < nk; it++) {
        const int s = it & 1, k0 = it * TBK;
        // ---- global -> registers: thread tid owns GEMM row m0+tid (16 loads, coalesced along
        //      positions), plus BN/32 float4 of B
        float ra[TBK];
        float4 rb[BN / 32];
#pragma unroll
        for (int kk = 0; kk < TBK; kk++)
            ra[kk] = (row_ok && k0 + kk < CRS) ? __ldg(Lrow + (size_t)(k0 + kk) * P) : 0.f;
#pragma unroll
        for (int j = 0; j < BN / 32; j++) {
            const int i = tid + TTHREADS * j;
            const int n = (i & 7) + 8 * (i >> 5), q = (i >> 3) & 3;
            const int kout = n0 + n, crs = k0 + 4 * q;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (kout < K) {
                const float* src = W + (size_t)kout * CRS + crs;
                if (vecB && crs + 3 < CRS) {
                    v = __ldg(reinterpret_cast<const float4*>(src));
                } else {
                    if (crs < CRS) v.x = __ldg(src);
                    if (crs + 1 < CRS) v.y = __ldg(src + 1);
                    if (crs + 2 < CRS) v.z = __ldg(src + 2);
                    if (crs + 3 < CRS) v.w = __ldg(src + 3);
                }
            }
            rb[j] = v;
        }
        // ---- stage s is free once the MMAs issued two iterations ago have completed
        if (it >= 2) mbar_wait(&bar[s], ((it >> 1) - 1) & 1);
        unsigned char* st = smem + s * STAGE;
        float* Ahi = reinterpret_cast<float*>(st);
        float* Alo = reinterpret_cast<float*>(st + A_BYTES);
        float* Bhi = reinterpret_cast<float*>(st + 2 * A_BYTES);
        float* Blo = reinterpret_cast<float*>(st + 2 * A_BYTES + B_BYTES);
#pragma unroll
        for (int q = 0; q < TBK / 4; q++) {      // K-major: 4 consecutive CRS of one position = 16 B
            const int off = (q * A_LBO + (tid >> 3) * A_SBO + (tid & 7) * 16) >> 2;
            const float4 v = make_float4(ra[4 * q], ra[4 * q + 1], ra[4 * q + 2], ra[4 * q + 3]);
            const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
            *reinterpret_cast<float4*>(Ahi + off) = h;
            *reinterpret_cast<float4*>(Alo + off) =
                make_float4(tf32_rn(v.x - h.x), tf32_rn(v.y - h.y), tf32_rn(v.z - h.z), tf32_rn(v.w - h.w));
        }
#pragma unroll
        for (int j = 0; j < BN / 32; j++) {
            const int i = tid + TTHREADS * j;
            const int n = (i & 7) + 8 * (i >> 5), q = (i >> 3) & 3;
            const int off = (q * B_LBO + (n >> 3) * B_SBO + (n & 7) * 16) >> 2;
            const float4 v = rb[j];
            const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
            *reinterpret_cast<float4*>(Bhi + off) = h;
            *reinterpret_cast<float4*>(Blo + off) =
                make_float4(tf32_rn(v.x - h.x), tf32_rn(v.y - h.y), tf32_rn(v.z - h.z), tf32_rn(v.w - h.w));
        }
        fence_proxy_async();     // generic-proxy smem writes -> visible to the tensor core (async proxy)
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const unsigned sa = sbase + s * STAGE;
#pragma unroll
            for (int ks = 0; ks < TBK / 8; ks++) {
                const uint64_t ahi = umma_desc(sa + 2 * ks * A_LBO, A_LBO, A_SBO);
                const uint64_t alo = umma_desc(sa + A_BYTES + 2 * ks * A_LBO, A_LBO, A_SBO);
                const uint64_t bhi = umma_desc(sa + 2 * A_BYTES + 2 * ks * B_LBO, B_LBO, B_SBO);
                const uint64_t blo = umma_desc(sa + 2 * A_BYTES + B_BYTES + 2 * ks * B_LBO, B_LBO, B_SBO);
                const uint64_t da[3] = {ahi, ahi, alo}, db[3] = {bhi, blo, bhi};
#pragma unroll
                for (int t = 0; t < 3; t++) {
                    const unsigned acc = (it > 0 || ks > 0 || t > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                        ::"r"(tmem), "l"(da[t]), "l"(db[t]), "r"(IDESC), "r"(acc) : "memory");
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         ::"r"(smem_u32(&bar[s])) : "memory");
        }
    }
    // ---- all MMAs done (the last commit covers every earlier MMA of this thread)
    if (nk > 0) mbar_wait(&bar[(nk - 1) & 1], ((nk - 1) >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // ---- epilogue: warp w reads TMEM lanes 32w..32w+31 (rows), 16 columns at a time;
    //      row tid = (img_t, p_t), so stores are coalesced along positions
    float* yrow = y + (size_t)(row_ok ? img_t : 0) * K * P + p_t;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        const unsigned taddr = tmem + ((unsigned)(warp * 32) << 16) + (unsigned)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row_ok) {
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const int kout = n0 + c0 + j;
                if (kout < K) {
                    const float v = __uint_as_float(r[j]);
                    yrow[(size_t)kout * P] = relu ? fmaxf(v, 0.f) : v;
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
                     ::"r"(tmem), "r"((unsigned)(BN < 32 ? 32 : BN)) : "memory");
}

template <int BN>
cudaError_t run_tc(int P, int K, int CRS, int nimg, const float* L, const float* W, float* y, int relu,
                   cudaStream_t st) {
    constexpr int STAGE = 2 * TM * TBK * 4 + 2 * BN * TBK * 4;
    const size_t smem = 2 * STAGE + 1024;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const long long mt = ((long long)nimg * P + TM - 1) / TM;
    dim3 grid((unsigned)mt, (K + BN - 1) / BN, 1);
    tc_gemm_kernel<BN><<<grid, TTHREADS, smem, st>>>(P, K, CRS, nimg, L, W, y, relu);
    return cudaGetLastError();
}

}  // namespace

// y[n] (K x P) = W (K x CRS) * L[n] (CRS x P), fp32 via 3xTF32 on tcgen05.
cudaError_t launch_tc_gemm(const Geom& g, const float* w, const float* L, float* y, int relu, cudaStream_t st) {
    const int P = g.Oh * g.Ow, K = g.K, CRS = g.C * g.R * g.S;
    // the widest N tile that still gives ~one CTA per SM (wider tiles reuse A more)
    const long long mt = ((long long)g.N * P + TM - 1) / TM;
    if (K <= 64 || mt * ((K + 127) / 128) < 148) return run_tc<64>(P, K, CRS, g.N, L, w, y, relu, st);
    if (K <= 128 || mt * ((K + 255) / 256) < 148) return run_tc<128>(P, K, CRS, g.N, L, w, y, relu, st);
    return run_tc<256>(P, K, CRS, g.N, L, w, y, relu, st);
}

}  // namespace spc
