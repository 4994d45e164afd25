// cscc.cu -- the paper's comparison method, CSCC (fan2019cscc), on the GPU (sm_100a).
//
// What it computes:
//  * encoding = SI Alg. 5, which the paper calls its simplification of the
//    CSCC encoder "designed for any value of K_w and s_w": every output column s
//    owns the K_w-wide submatrix of padded columns [s*s_w, s*s_w + K_w) (the lowered matrix LM
//    of SI Eq. 17); its NZEs are stored row-major inside the submatrix with
//    IN = (w - s*s_w) + h*K_w, and ptr = [0, c_0 .. c_{O_w-1}] holds channel-cumulative counts
//    (O_w + 1 entries per channel, no NPC: Eq. 17 charges every channel O_w + 1).  Padded frame
//    (reading A30).  Channels n-major then c, side tables as for CPO (reading A19).
//  * convolution = SI Alg. 6: each NZE of submatrix s adds, for every
//    kernel row l, v * W[k, c, l, index % K_w] to output (index/K_w - l, s); a vertical stride
//    keeps the rows on the grid (reading A15).
//
// B200 design (a baseline: simple, correct, one launch per phase):
//  * encode: (1) one CTA per channel plane counts the NZEs of every (submatrix, row) pair from
//    the plane staged in shared memory; (2) one CTA scans the per-plane totals into the side
//    tables; (3) one CTA per plane writes ptr / DA / IN (thread per (submatrix, row): its
//    offset is the plane offset + the submatrix prefix + the row prefix).
//  * conv: CTA = (image, 4 output columns, 64 output channels); warp = one output column s,
//    lanes = 2 output channels each; the warp walks submatrix s of every channel (NZEs
//    broadcast by shuffles) and accumulates [O_h][64] in its own shared-memory slice.
#include <algorithm>

#include "common.cuh"

namespace spc {
namespace {

constexpr int kCsThreads = 256;

struct CsArgs {
    Geom g;
    const float* __restrict__ x;
    int32_t* ptr; float* da; int32_t* in;
    int64_t* cpo_off; int64_t* cnz_off; int64_t* cin_off;
    int64_t* lengths;
    int64_t cap_ptr, cap_da, cap_in;
};

__device__ __forceinline__ float plane_at(const float* pl, const Geom& g, int h, int w) {
    const int hh = h - g.pt, ww = w - g.pl;
    return (hh < 0 || hh >= g.H || ww < 0 || ww >= g.W) ? 0.0f : pl[hh * g.W + ww];
}

// cnt[s * Hp + h] = NZEs of row h of submatrix s (threads over (s, h) pairs)
__device__ void count_rows(const Geom& g, const float* pl, int* cnt) {
    for (int it = threadIdx.x; it < g.Ow * g.Hp; it += blockDim.x) {
        const int s = it / g.Hp, h = it % g.Hp;
        int c = 0;
        for (int m = 0; m < g.S; m++) c += plane_at(pl, g, h, s * g.sw + m) != 0.0f;
        cnt[it] = c;
    }
}

__device__ void stage_plane(const Geom& g, const float* __restrict__ src, float* dst) {
    const int HW = g.H * g.W;
    for (int i = threadIdx.x; i < HW; i += blockDim.x) dst[i] = __ldg(src + i);
}

// (1) per-plane LM non-zero count -> cnz_off[plane] (scanned in place by (2))
__global__ void __launch_bounds__(kCsThreads) cscc_count_kernel(CsArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geom& g = a.g;
    float* pl = reinterpret_cast<float*>(smem);
    int* cnt = reinterpret_cast<int*>(pl + g.H * g.W);
    __shared__ int s_red[kCsThreads / 32];
    pdl_wait();
    const long long plane = blockIdx.x;
    stage_plane(g, a.x + plane * g.H * g.W, pl);
    __syncthreads();
    count_rows(g, pl, cnt);
    __syncthreads();
    int t = 0;
    for (int i = threadIdx.x; i < g.Ow * g.Hp; i += blockDim.x) t += cnt[i];
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < kCsThreads / 32; w++) tot += s_red[w];
        a.cnz_off[plane] = tot;
    }
}

// (2) one CTA: exclusive scan of the per-plane counts -> side tables and lengths
__global__ void __launch_bounds__(1024) cscc_scan_kernel(CsArgs a) {
    const Geom& g = a.g;
    __shared__ long long s_w[32];
    const long long NC = g.NC;
    const int T = blockDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long per = (NC + T - 1) / T;
    const long long b0 = threadIdx.x * per, b1 = min(NC, b0 + per);
    long long sum = 0;
    for (long long i = b0; i < b1; i++) sum += a.cnz_off[i];
    long long inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        long long v = (lane < T / 32) ? s_w[lane] : 0, vi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, vi, o);
            if (lane >= o) vi += t;
        }
        if (lane < T / 32) s_w[lane] = vi - v;   // exclusive per-warp base
    }
    __syncthreads();
    long long run = s_w[warp] + inc - sum;
    for (long long i = b0; i < b1; i++) {
        const long long c = a.cnz_off[i];
        a.cnz_off[i] = run;
        a.cin_off[i] = run;
        a.cpo_off[i] = i * (g.Ow + 1);
        run += c;
    }
    if (threadIdx.x == T - 1) {
        const long long tp = NC * (g.Ow + 1);
        a.cnz_off[NC] = run;
        a.cin_off[NC] = run;
        a.cpo_off[NC] = tp;
        a.lengths[0] = tp;
        a.lengths[1] = run;
        a.lengths[2] = run;
        a.lengths[3] = (tp > a.cap_ptr || run > a.cap_da || run > a.cap_in) ? 1 : 0;
    }
}

// (3) per plane: ptr [0, c_0 .. c_{Ow-1}], then DA / IN of every (submatrix, row) pair
__global__ void __launch_bounds__(kCsThreads) cscc_write_kernel(CsArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geom& g = a.g;
    float* pl = reinterpret_cast<float*>(smem);
    int* cnt = reinterpret_cast<int*>(pl + g.H * g.W);      // [Ow][Hp] row counts -> row prefixes
    int* part = cnt + g.Ow * g.Hp;                          // [Ow + 1] submatrix prefixes
    const long long plane = blockIdx.x;
    if (a.lengths[3]) return;                               // capacities too small: nothing written
    stage_plane(g, a.x + plane * g.H * g.W, pl);
    __syncthreads();
    count_rows(g, pl, cnt);
    __syncthreads();
    // row prefix inside each submatrix (warp per submatrix), submatrix totals
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = warp; s < g.Ow; s += kCsThreads / 32) {
        int run = 0;
        for (int h0 = 0; h0 < g.Hp; h0 += 32) {
            const int h = h0 + lane;
            const int v = (h < g.Hp) ? cnt[s * g.Hp + h] : 0;
            int tot;
            const int ex = warp_exclusive_scan(v, &tot);
            if (h < g.Hp) cnt[s * g.Hp + h] = run + ex;
            run += tot;
        }
        if (lane == 0) part[s + 1] = run;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        part[0] = 0;
        for (int s = 1; s <= g.Ow; s++) part[s] += part[s - 1];   // channel-cumulative (Alg. 5)
    }
    __syncthreads();
    const long long P = a.cpo_off[plane], Z = a.cnz_off[plane];
    for (int s = threadIdx.x; s <= g.Ow; s += kCsThreads) a.ptr[P + s] = part[s];
    for (int it = threadIdx.x; it < g.Ow * g.Hp; it += blockDim.x) {
        const int s = it / g.Hp, h = it % g.Hp;
        long long o = Z + part[s] + cnt[it];
        for (int m = 0; m < g.S; m++) {
            const float v = plane_at(pl, g, h, s * g.sw + m);
            if (v != 0.0f) {
                a.da[o] = v;
                a.in[o] = m + h * g.S;
                o++;
            }
        }
    }
}

// ---- convolution (SI Alg. 6)
constexpr int kCcCols = 4, kCcKB = 64;

struct CcArgs {
    Geom g;
    const int32_t* __restrict__ ptr;
    const float* __restrict__ da;
    const int32_t* __restrict__ in;
    const int64_t* __restrict__ cpo_off;
    const int64_t* __restrict__ cnz_off;
    const float* __restrict__ wp;   // [C][R][S][K]
    float* y;
    int relu;
    const unsigned long long* status;
};

__global__ void __launch_bounds__(32 * kCcCols) cscc_conv_kernel(CcArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geom& g = a.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * kCcCols + warp;              // this warp's output column
    const int kbase = blockIdx.y * kCcKB;
    const int n = blockIdx.z;
    float2* acc = reinterpret_cast<float2*>(smem) + (size_t)warp * g.Oh * 32;   // [Oh][32 lanes]
    for (int i = lane; i < g.Oh * 32; i += 32) acc[i] = make_float2(0.f, 0.f);
    pdl_wait();
    const bool bad = *reinterpret_cast<volatile const unsigned long long*>(a.status) != 0ull;
    const int k0 = kbase + 2 * lane;
    const bool k0ok = k0 < g.K, k1ok = k0 + 1 < g.K;
    if (s < g.Ow && !bad) {
        for (int c = 0; c < g.C; c++) {
            const long long nc = (long long)n * g.C + c;
            const long long P = a.cpo_off[nc], Z = a.cnz_off[nc];
            const int lo = a.ptr[P + s], hi = a.ptr[P + 1 + s];
            const float* wc = a.wp + (size_t)c * g.R * g.S * g.K;
            for (int b = lo; b < hi; b += 32) {
                const int i = b + lane;
                const float v = (i < hi) ? __ldg(a.da + Z + i) : 0.f;
                const int e = (i < hi) ? __ldg(a.in + Z + i) : 0;
                const int cntb = min(32, hi - b);
                for (int j = 0; j < cntb; j++) {
                    const float vj = __shfl_sync(0xffffffffu, v, j);
                    const int ej = __shfl_sync(0xffffffffu, e, j);
                    const int h = ej / g.S, m = ej % g.S;
                    for (int l = 0; l < g.R; l++) {
                        const int y1 = h - l;
                        if (y1 < 0 || y1 >= g.Oh1 || (y1 % g.sh) != 0) continue;
                        const int yy = y1 / g.sh;
                        if (yy >= g.Oh) continue;
                        const float* wt = wc + (size_t)(l * g.S + m) * g.K;
                        const float w0 = k0ok ? __ldg(wt + k0) : 0.f, w1 = k1ok ? __ldg(wt + k0 + 1) : 0.f;
                        float2 cur = acc[yy * 32 + lane];
                        cur.x = fmaf(vj, w0, cur.x);
                        cur.y = fmaf(vj, w1, cur.y);
                        acc[yy * 32 + lane] = cur;
                    }
                }
            }
        }
    }
    __syncwarp();
    if (s >= g.Ow) return;
    float* yb = a.y + (size_t)n * g.K * g.Oh * g.Ow;
    for (int yy = 0; yy < g.Oh; yy++) {
        float2 v = acc[yy * 32 + lane];
        if (a.relu) { v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); }
        if (k0ok) yb[((size_t)k0 * g.Oh + yy) * g.Ow + s] = v.x;
        if (k1ok) yb[((size_t)(k0 + 1) * g.Oh + yy) * g.Ow + s] = v.y;
    }
}

}  // namespace

size_t cscc_smem_bytes(const Geom& g) {
    return (size_t)g.H * g.W * 4 + (size_t)g.Ow * g.Hp * 4 + (size_t)(g.Ow + 1) * 4 + 16;
}

cudaError_t launch_cscc_encode(const Geom& g, const float* x, spc_encoding* e, cudaStream_t st) {
    CsArgs a;
    a.g = g; a.x = x;
    a.ptr = e->ptr; a.da = e->da; a.in = e->in;
    a.cpo_off = e->chan_ptr_off; a.cnz_off = e->chan_nz_off; a.cin_off = e->chan_in_off;
    a.lengths = e->lengths;
    a.cap_ptr = e->ptr_cap; a.cap_da = e->da_cap; a.cap_in = e->in_cap;
    const size_t smem = cscc_smem_bytes(g);
    static std::atomic<size_t> attr_c[kMaxDevices], attr_w[kMaxDevices];
    cudaError_t err = ensure_smem_attr((const void*)cscc_count_kernel, smem, attr_c);
    if (err == cudaSuccess) err = ensure_smem_attr((const void*)cscc_write_kernel, smem, attr_w);
    if (err != cudaSuccess) return err;
    cscc_count_kernel<<<(unsigned)g.NC, kCsThreads, smem, st>>>(a);
    cscc_scan_kernel<<<1, 1024, 0, st>>>(a);
    cscc_write_kernel<<<(unsigned)g.NC, kCsThreads, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_cscc_conv(const Geom& g, const spc_encoding* e, const float* w_packed, float* y, int relu,
                             cudaStream_t st) {
    CcArgs a;
    a.g = g;
    a.ptr = e->ptr; a.da = e->da; a.in = e->in;
    a.cpo_off = e->chan_ptr_off; a.cnz_off = e->chan_nz_off;
    a.wp = w_packed; a.y = y; a.relu = relu;
    a.status = reinterpret_cast<const unsigned long long*>(e->lengths + 3);
    const size_t smem = (size_t)kCcCols * g.Oh * 32 * sizeof(float2);
    static std::atomic<size_t> attr[kMaxDevices];
    cudaError_t err = ensure_smem_attr((const void*)cscc_conv_kernel, smem, attr);
    if (err != cudaSuccess) return err;
    dim3 grid((g.Ow + kCcCols - 1) / kCcCols, (g.K + kCcKB - 1) / kCcKB, g.N);
    cscc_conv_kernel<<<grid, 32 * kCcCols, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace spc
