// tcgemm.cu -- dense baseline GEMM on the 5th-generation tensor cores (tcgen05, sm_100a):
// fp32 accuracy from three TF32 products (3xTF32), accumulators in TMEM.
//
// The im2col baseline computes y[n] (K x P) = W (K x CRS) * L[n]
// (CRS x P).  Here the GEMM is D (M x K) = A (M x CRS) * W^T with M = N*P rows
// (image, output position) -- all images in one GEMM, the weights are shared:
//   * A is the lowered matrix written K-major ([M][CRS], CRS contiguous) by
//     im2col_t_kernel; B is the caller's KCRS weight tensor, already K-major;
//   * TMA (2D tensor maps, box = 32 CRS (128 B) x rows, 128-byte swizzle) lands a stage's
//     K slice in the UMMA K-major SWIZZLE_128B layout (one TMA per operand per stage);
//   * every fp32 operand x is split into hi = x with the 13 low mantissa
//     bits cleared (exactly representable in tf32) and lo = x - hi (exact); kind::tf32
//     reads only the top 19 bits of a 32-bit operand, so the raw x is passed as hi and only
//     lo is materialised -- for A by the split warps, which move each landed A tile (raw =
//     hi, and lo) from shared memory into TMEM (tcgen05.st; the MMAs take A from TMEM, so
//     they read only B from shared memory: the ring is shared-memory-bandwidth-bound), for
//     B (the weights) once per call into the workspace tail when the caller provides it
//     (split_b_kernel), else in shared memory by the split warps:
//     D += Ahi*Bhi + Ahi*Blo + Alo*Bhi; the dropped Alo*Blo is ~2^-22 relative -- inside
//     the 1e-4 fp32 tolerance of north_star, unlike a single TF32 product;
//   * warp-specialised pipeline over NST stages (mbarriers): warp 0 issues the TMA loads,
//     warps 2-5 (thread = A row = TMEM lane) write hi / lo of every landed A tile to TMEM, warp 1 issues
//     the 12 MMAs of a stage (M = 128, N = BN, K = 8 each) and commits them to the stage's
//     "empty" barrier;
//   * accuracy: the tensor core's fp32 accumulation over all of CRS (x3 products) left
//     ~2e-5 absolute error on near-zero outputs at CRS = 4608, so every KCH stages (256 CRS)
//     accumulate into one of two TMEM buffers, and warps 6-13 drain each finished chunk
//     (tcgen05.ld, lane = row, two warps per lane quarter) into fp32 register sums with
//     round-to-nearest adds, then store y coalesced along positions (optional ReLU).
#include <algorithm>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>

#include "common.cuh"

namespace spc {
namespace {

constexpr int TM = 128;       // MMA M (rows = image positions)
constexpr int TBK = 32;       // CRS elements per stage
constexpr int NCONV = 128;    // converter threads (warps 2-5)
constexpr int NDRAIN = 256;   // drain / epilogue threads (warps 6-13)
constexpr int TTHREADS = 64 + NCONV + NDRAIN;   // + warp 0 TMA, warp 1 MMA
constexpr int KCH = 8;        // stages (8 x 32 CRS) per TMEM accumulation chunk
#ifndef SPC_TC_NST64
#define SPC_TC_NST64 4
#endif
#ifndef SPC_TC_NST128
#define SPC_TC_NST128 4
#endif

// SmemDescriptor (sm_100) of a K-major operand tile in the 128-byte swizzle layout that TMA
// writes (rows of 128 B = 32 fp32, 16-byte chunks XOR-ed with row % 8 inside each 1024-byte
// group of 8 rows): start [0,14) and SBO [32,46) in 16-byte units (SBO = 1024 B between
// 8-row groups; LBO unused for swizzled K-major, 1), version 1 at [46,48), base offset 0
// (1024-byte aligned tiles), layout SWIZZLE_128B (2) at [61,64).  A K-step of 8 tf32 inside
// the 128-byte row advances the start address by 32 B (the hardware applies the XOR).
__device__ __forceinline__ uint64_t umma_desc_sw128(unsigned saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}

// 32 consecutive TMEM columns of this thread's lane (32x32b shape, one register per column)
__device__ __forceinline__ void tmem_st32(unsigned taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
          "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
          "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// lo = x - hi (exact in fp32), hi = x with the 13 low mantissa bits cleared (a tf32 value).
// hi itself is never written: kind::tf32 reads only the top 19 bits of each 32-bit operand,
// so the raw x already is hi to the tensor core (measured: outputs bit-identical to staging
// explicitly truncated copies, and 5-8 % faster on the K >= 128 layers: one smem write pass
// fewer per stage).
__device__ __forceinline__ float4 lo_of(const float4 v) {
    const unsigned M = 0xFFFFE000u;
    return make_float4(v.x - __uint_as_float(__float_as_uint(v.x) & M), v.y - __uint_as_float(__float_as_uint(v.y) & M),
                       v.z - __uint_as_float(__float_as_uint(v.z) & M), v.w - __uint_as_float(__float_as_uint(v.w) & M));
}

template <int BN, int NST, bool BPRE>   // BPRE: B's lo half arrives precomputed (its own tensor map)
__global__ void __launch_bounds__(TTHREADS, 1) tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                                                              const __grid_constant__ CUtensorMap mapB,
                                                              const __grid_constant__ CUtensorMap mapBlo,
                                                              int P, int K, int CRS, long long M,
                                                              float* __restrict__ y, int relu) {
    constexpr int A_BYTES = TM * TBK * 4;            // raw A tile (its hi / lo go to TMEM)
    constexpr int B_BYTES = BN * TBK * 4;
    constexpr int BOFF = A_BYTES;                    // B (hi, lo) after A
    constexpr int STAGE = BOFF + 2 * B_BYTES;
    constexpr int HALF = BN / 2;                     // columns per drain warp
    // instruction descriptor: D f32, A/B tf32, both K-major, N = BN, M = 128
    constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) |
                               ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

    // A (raw = hi, and lo) of every stage lives in TMEM next to the two accumulator buffers:
    // stage s at columns 2*BN + 64 s (hi) and + 32 (lo); the MMAs read only B from smem
    constexpr unsigned TCOLS = 512;
    static_assert(2 * BN + 64 * NST <= 512, "TMEM: accumulators + A stages");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte aligned stage base (TMA destinations need 128 B; the allocation has +1 KB)
    unsigned char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    __shared__ __align__(8) unsigned long long full[NST], conv[NST], empty[NST], accf[2], acce[2];
    __shared__ unsigned tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // persistent: CTA b takes tiles b, b + gridDim.x, ... (tile = n-tile major over m-tiles);
    // the stage ring and the two TMEM chunk buffers run on across tiles (flat counters)
    const long long mtiles = (M + TM - 1) / TM;
    const long long ntile_total = mtiles * ((K + BN - 1) / BN);
    const int nk = (CRS + TBK - 1) / TBK;
    const int nch = (nk + KCH - 1) / KCH;           // accumulation chunks per tile
    auto tile_m0 = [&](long long t) { return (t % mtiles) * TM; };
    auto tile_n0 = [&](long long t) { return (int)(t / mtiles) * BN; };

    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(&tmem_base_s)), "r"(TCOLS) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int s = 0; s < NST; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], NCONV);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&accf[b], 1);
            mbar_init(&acce[b], NDRAIN);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
        if (BPRE) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapBlo) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_base_s;

    if (warp == 0) {
        // ---- TMA producer: raw A (rows m0..) and B (output channels n0..) tiles of a stage
        if (lane == 0) {
            long long g = 0;   // stage counter across tiles
            for (long long t = blockIdx.x; t < ntile_total; t += gridDim.x) {
                const int m0 = (int)tile_m0(t), n0 = tile_n0(t);
                for (int kb = 0; kb < nk; kb++, g++) {
                    const int s = (int)(g % NST);
                    if (g >= NST) mbar_wait(&empty[s], (unsigned)(((g / NST) - 1) & 1));
                    unsigned char* st = smem + s * STAGE;
                    mbar_expect_tx(&full[s], A_BYTES + (BPRE ? 2 : 1) * B_BYTES);
                    tma_load_2d(st, &mapA, kb * TBK, m0, &full[s]);
                    tma_load_2d(st + BOFF, &mapB, kb * TBK, n0, &full[s]);
                    if (BPRE) tma_load_2d(st + BOFF + B_BYTES, &mapBlo, kb * TBK, n0, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer: 4 K-steps x 3 products per stage, committed to the stage's empty
        //      barrier; chunk j of KCH stages accumulates into TMEM buffer j & 1 and is
        //      committed to accf[j & 1] for the drain warps
        if (lane == 0) {
            const unsigned sbase = smem_u32(smem);
            long long g = 0, jg = 0;   // stage and chunk counters across tiles
            for (long long t = blockIdx.x; t < ntile_total; t += gridDim.x)
            for (int kb = 0; kb < nk; kb++, g++) {
                const int s = (int)(g % NST), b = (int)(jg & 1);
                const bool first = (kb % KCH) == 0, last = (kb % KCH) == KCH - 1 || kb == nk - 1;
                if (first && jg >= 2) mbar_wait(&acce[b], (unsigned)(((jg >> 1) - 1) & 1));
                mbar_wait(&conv[s], (unsigned)((g / NST) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned sa = sbase + s * STAGE;
                const unsigned dt = tmem + (unsigned)(b * BN);
#pragma unroll
                for (int ks = 0; ks < TBK / 8; ks++) {
                    const unsigned ahi = tmem + (unsigned)(2 * BN + 64 * s + 8 * ks), alo = ahi + 32;
                    const uint64_t bhi = umma_desc_sw128(sa + BOFF + 32 * ks);
                    const uint64_t blo = umma_desc_sw128(sa + BOFF + B_BYTES + 32 * ks);
                    const unsigned ta[3] = {ahi, ahi, alo};
                    const uint64_t db[3] = {bhi, blo, bhi};
#pragma unroll
                    for (int t = 0; t < 3; t++) {
                        const unsigned acc = (!first || ks > 0 || t > 0) ? 1u : 0u;
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                            ::"r"(dt), "r"(ta[t]), "l"(db[t]), "r"(IDESC), "r"(acc) : "memory");
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             ::"r"(smem_u32(&empty[s])) : "memory");
                if (last) {
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                 ::"r"(smem_u32(&accf[b])) : "memory");
                    jg++;
                }
            }
        }
    } else if (warp < 2 + NCONV / 32) {
        // ---- converter warps: the lo half of every landed stage (the raw values serve as hi)
        const int ct = tid - 64;
        const long long gtot = ((ntile_total - blockIdx.x + gridDim.x - 1) / gridDim.x) * nk;
        for (long long g = 0; g < gtot; g++) {
            const int s = (int)(g % NST);
            mbar_wait(&full[s], (unsigned)((g / NST) & 1));
            unsigned char* st = smem + s * STAGE;
            float4* bb = reinterpret_cast<float4*>(st + BOFF);
            float4* blo = reinterpret_cast<float4*>(st + BOFF + B_BYTES);
            {   // thread = A row m (its warp's TMEM lane quarter): the row's 32 CRS values from the
                // SW128 tile (16-byte chunk j of row m sits at chunk j ^ (m & 7)) -> TMEM hi, lo
                const int m = 32 * (warp & 3) + lane;
                const unsigned char* row = st + m * 128;
                uint32_t h[32], l[32];
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const float4 v = *reinterpret_cast<const float4*>(row + ((j ^ (m & 7)) << 4));
                    const float4 lv = lo_of(v);
                    h[4 * j] = __float_as_uint(v.x); h[4 * j + 1] = __float_as_uint(v.y);
                    h[4 * j + 2] = __float_as_uint(v.z); h[4 * j + 3] = __float_as_uint(v.w);
                    l[4 * j] = __float_as_uint(lv.x); l[4 * j + 1] = __float_as_uint(lv.y);
                    l[4 * j + 2] = __float_as_uint(lv.z); l[4 * j + 3] = __float_as_uint(lv.w);
                }
                const unsigned ta = tmem + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)(2 * BN + 64 * s);
                tmem_st32(ta, h);
                tmem_st32(ta + 32, l);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            }
#pragma unroll
            for (int i = ct; i < (BPRE ? 0 : B_BYTES / 16); i += NCONV) blo[i] = lo_of(bb[i]);
            fence_proxy_async();       // generic smem writes -> visible to the tensor core
            mbar_arrive(&conv[s]);
        }
    } else {
        // ---- drain warps: sum the chunk accumulators in fp32 registers (round-to-nearest adds
        //      over a few chunks instead of one tensor-core accumulation over all of CRS),
        //      then store y; two warps per TMEM lane quarter, half the columns each
        const int dw = warp - 2 - NCONV / 32;          // 0..7
        const int q = warp & 3, half = dw >> 2;        // a warp may access TMEM lanes 32 (warp % 4) ..
        long long jg = 0;
        for (long long t = blockIdx.x; t < ntile_total; t += gridDim.x) {
        const long long m0 = tile_m0(t);
        const int n0 = tile_n0(t);
        float sum[HALF];
#pragma unroll
        for (int i = 0; i < HALF; i++) sum[i] = 0.f;
        for (int j = 0; j < nch; j++, jg++) {
            const int b = (int)(jg & 1);
            mbar_wait(&accf[b], (unsigned)((jg >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int c0 = 0; c0 < HALF; c0 += 16) {
                uint32_t r[16];
                const unsigned taddr = tmem + ((unsigned)(32 * q) << 16) + (unsigned)(b * BN + half * HALF + c0);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 16; i++) sum[c0 + i] += __uint_as_float(r[i]);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&acce[b]);
        }
        const long long m = m0 + 32 * q + lane;
        if (m < M) {
            const int img = (int)(m / P), p = (int)(m - (long long)img * P);
            float* yrow = y + (size_t)img * K * P + p;
#pragma unroll
            for (int i = 0; i < HALF; i++) {
                const int kout = n0 + half * HALF + i;
                if (kout < K) yrow[(size_t)kout * P] = relu ? fmaxf(sum[i], 0.f) : sum[i];
            }
        }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS) : "memory");
}

int sm_count_tc() { return device_sm_count(); }

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2D fp32 tensor map of a row-major [rows][cols] matrix, box = 32 columns (128 B) x box_rows
// rows, 128-byte swizzle (the UMMA K-major SWIZZLE_128B layout)
bool make_map(CUtensorMap* map, const float* base, long long rows, int cols, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    const cuuint32_t box[2] = {TBK, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// lo = x - hi (hi = x with the 13 low mantissa bits cleared) over the K x CRS weights, once
// per call, so the GEMM's split warps only handle A; the raw weights serve as B hi
__global__ void __launch_bounds__(256) split_b_kernel(const float* __restrict__ w, float* __restrict__ lo,
                                                      long long n) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
        const float v = w[i];
        lo[i] = v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    }
}

template <int BN, int NST>
cudaError_t run_tc(int P, int K, int CRS, int nimg, const float* A, const float* W, float* bsplit, float* y,
                   int relu, cudaStream_t st) {
    constexpr int STAGE = TM * TBK * 4 + 2 * BN * TBK * 4;
    const size_t smem = (size_t)NST * STAGE + 1024;
    static std::atomic<size_t> attr[2][kMaxDevices];
    const bool pre = bsplit != nullptr;
    {
        cudaError_t e = ensure_smem_attr(pre ? (const void*)tc_gemm_kernel<BN, NST, true> : (const void*)tc_gemm_kernel<BN, NST, false>,
                                         smem, attr[pre]);
        if (e != cudaSuccess) return e;
    }
    const long long M = (long long)nimg * P;
    CUtensorMap ma, mb, mblo;
    if (!make_map(&ma, A, M, CRS, TM)) return cudaErrorNotSupported;
    if (pre) {
        const long long n = (long long)K * CRS;
        float* lo = bsplit;
        split_b_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 8), 256, 0, st>>>(W, lo, n);
        if (!make_map(&mb, W, K, CRS, BN) || !make_map(&mblo, lo, K, CRS, BN)) return cudaErrorNotSupported;
    } else {
        if (!make_map(&mb, W, K, CRS, BN)) return cudaErrorNotSupported;
        mblo = mb;
    }
    // persistent grid: one CTA per SM (the kernel's shared memory allows one)
    const long long tiles = ((M + TM - 1) / TM) * ((K + BN - 1) / BN);
    dim3 grid((unsigned)std::min<long long>(tiles, sm_count_tc()), 1, 1);
    if (pre)
        tc_gemm_kernel<BN, NST, true><<<grid, TTHREADS, smem, st>>>(ma, mb, mblo, P, K, CRS, M, y, relu);
    else
        tc_gemm_kernel<BN, NST, false><<<grid, TTHREADS, smem, st>>>(ma, mb, mblo, P, K, CRS, M, y, relu);
    return cudaGetLastError();
}

}  // namespace

// TMA needs 16-byte aligned bases and row pitches (CRS % 4 == 0).
bool tc_gemm_supported(const Geom& g, const float* w) {
    const int CRS = g.C * g.R * g.S;
    return CRS % 4 == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0 && encode_fn() != nullptr;
}

// y[n] (K x P) = W (K x CRS) * L[n] (CRS x P), fp32 via 3xTF32 on tcgen05; A = the lowered
// matrix in the K-major layout [N*P][CRS] (im2col_t_kernel).
cudaError_t launch_tc_gemm(const Geom& g, const float* w, const float* A, float* y, int relu, cudaStream_t st,
                           float* bsplit) {
    const int P = g.Oh * g.Ow, K = g.K, CRS = g.C * g.R * g.S;
    if (!tc_gemm_supported(g, w) || (reinterpret_cast<uintptr_t>(A) & 15)) return cudaErrorNotSupported;
    if (reinterpret_cast<uintptr_t>(bsplit) & 15) bsplit = nullptr;
    // N tile: 128 unless the grid would leave SMs idle with it
    const long long mt = ((long long)g.N * P + TM - 1) / TM;
    if (K <= 64 || mt * ((K + 127) / 128) < 148) return run_tc<64, SPC_TC_NST64>(P, K, CRS, g.N, A, w, bsplit, y, relu, st);
    return run_tc<128, SPC_TC_NST128>(P, K, CRS, g.N, A, w, bsplit, y, relu, st);
}

}  // namespace spc
