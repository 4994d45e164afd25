// stride_aware.cu -- the stride-aware CPO layout (reading A32) on the
// GPU (sm_100a): encoder and the convolution over it.
//
// Layout (SI Eq. 2's ceil(K_w/s_w) types; made concrete in DESIGN.md A32):
// partition s (0 <= s < O_w) covers padded columns [s*s_w, s*s_w + K_w); a column's coverage
// cov(w) is the number of partitions covering it, its owner the first of them, its local column
// L = w - owner*s_w and its type t = cov - 1.  Per channel: [NPC] when no covered column holds
// an NZE; otherwise, for every type present in the geometry (ascending), [t+1, c_0 .. c_{O_w-1}]
// with block-relative cumulative counts through partition s's owned type-t columns (-1: owns
// none) or [t+1, NPF]; DA / IN column by column (ascending), rows ascending, IN = L + h*K_w.
// Compared with the stride-agnostic encoding (reading A15) a stride-2 layer stores O_w instead
// of O_w1 ~ 2*O_w partitions per block (about half the ptr entries).
//
// B200 design (three launches like the CSCC encoder):
//  (1) counts per covered column -> per-plane ptr length and NZE count; (2) one CTA scans them
//  into the side tables; (3) per plane the blocks are laid out (columns of a type in ascending
//  order), ptr written, and one lane per column writes its DA / IN.  One WARP per plane in (1)
//  and (3) (8 planes per CTA), so layers with many small planes fill the GPU.
// Convolution: CTA = (image, 4 output columns, 64 output channels); warp = output column x;
// for every type t it walks the owners s in [x-t, x] (the partitions whose type-t columns x
// covers), tap m = L + (s-x)*s_w, into its own [O_h][64] shared-memory accumulator slice.
#include <algorithm>

#include "common.cuh"

namespace spc {
namespace {

constexpr int kSaThreads = 256;
constexpr int kSaMaxTypes = 8;

struct SaArgs {
    Geom g;
    const float* __restrict__ x;
    int32_t* ptr; float* da; int32_t* in;
    int64_t* cpo_off; int64_t* cnz_off; int64_t* cin_off;
    int64_t* lengths;
    int64_t cap_ptr, cap_da, cap_in;
};

// coverage / owner of padded column w at stride s_w (reading A32)
__device__ __forceinline__ int sa_cov(const Geom& g, int w) {
    const int hi = min(g.Ow - 1, w / g.sw);
    const int lo = max(0, (w - g.S + 1 + g.sw - 1) / g.sw);   // ceil((w-S+1)/sw) for w-S+1 >= 0
    const int lo2 = (w - g.S + 1 <= 0) ? 0 : lo;
    return max(0, hi - lo2 + 1);
}
__device__ __forceinline__ int sa_owner(const Geom& g, int w) {
    return (w - g.S + 1 <= 0) ? 0 : (w - g.S + 1 + g.sw - 1) / g.sw;
}
__device__ __forceinline__ int sa_ntypes(const Geom& g) { return (g.S + g.sw - 1) / g.sw; }

__device__ __forceinline__ float plane_at(const float* pl, const Geom& g, int h, int w) {
    const int hh = h - g.pt, ww = w - g.pl;
    return (hh < 0 || hh >= g.H || ww < 0 || ww >= g.W) ? 0.0f : pl[hh * g.W + ww];
}

// One WARP per channel plane (8 planes per CTA): the plane staged in the warp's shared slice,
// per-column counts (lanes over columns), per-type totals and the plane's ptr length.
constexpr int kSaWarps = kSaThreads / 32;

struct SaWarpSmem {
    float* pl; int* cnt; int* coff;
};
__device__ __forceinline__ SaWarpSmem sa_warp_smem(const Geom& g, unsigned char* smem, int warp) {
    const size_t per = align_up((size_t)g.H * g.W * 4 + (size_t)2 * g.Wp * 4, 16);
    SaWarpSmem m;
    m.pl = reinterpret_cast<float*>(smem + per * warp);
    m.cnt = reinterpret_cast<int*>(m.pl + g.H * g.W);
    m.coff = m.cnt + g.Wp;
    return m;
}

__device__ void warp_stage_counts(const Geom& g, const float* __restrict__ x, long long plane, SaWarpSmem m,
                                  int lane) {
    const int HW = g.H * g.W;
    const float* src = x + plane * HW;
    for (int i = lane; i < HW; i += 32) m.pl[i] = __ldg(src + i);
    __syncwarp();
    for (int w = lane; w < g.Wp; w += 32) {
        int c = 0;
        if (sa_cov(g, w) > 0)
            for (int h = g.pt; h < g.pt + g.H; h++) c += plane_at(m.pl, g, h, w) != 0.0f;
        m.cnt[w] = c;
    }
    __syncwarp();
}

// per-type totals (every lane computes the same values from the shared counts)
__device__ unsigned type_totals(const Geom& g, const int* cnt, int* tot) {
    unsigned present = 0;
    for (int t = 0; t < kSaMaxTypes; t++) tot[t] = 0;
    for (int w = 0; w < g.Wp; w++) {
        const int cv = sa_cov(g, w);
        if (cv == 0) continue;
        present |= 1u << (cv - 1);
#pragma unroll
        for (int t = 0; t < kSaMaxTypes; t++)
            if (t == cv - 1) tot[t] += cnt[w];
    }
    return present;
}

__global__ void __launch_bounds__(kSaThreads) sa_count_kernel(SaArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geom& g = a.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long plane = (long long)blockIdx.x * kSaWarps + warp;
    pdl_wait();
    if (plane >= g.NC) return;
    const SaWarpSmem m = sa_warp_smem(g, smem, warp);
    warp_stage_counts(g, a.x, plane, m, lane);
    if (lane == 0) {
        int tot[kSaMaxTypes];
        const unsigned present = type_totals(g, m.cnt, tot);
        int nnz = 0, plen = 0;
        for (int t = 0; t < sa_ntypes(g); t++) {
            if (!((present >> t) & 1u)) continue;
            nnz += tot[t];
            plen += tot[t] ? (1 + g.Ow) : 2;
        }
        a.cpo_off[plane] = nnz ? plen : 1;   // NPC: one entry
        a.cnz_off[plane] = nnz;
    }
}

// one CTA: exclusive scans of the per-plane ptr lengths and NZE counts
__global__ void __launch_bounds__(1024) sa_scan_kernel(SaArgs a) {
    __shared__ long long s_w[2][32];
    const long long NC = a.g.NC;
    const int T = blockDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long per = (NC + T - 1) / T;
    const long long b0 = threadIdx.x * per, b1 = min(NC, b0 + per);
    long long sp = 0, sz = 0;
    for (long long i = b0; i < b1; i++) { sp += a.cpo_off[i]; sz += a.cnz_off[i]; }
    long long ip = sp, iz = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long tp = __shfl_up_sync(0xffffffffu, ip, o), tz = __shfl_up_sync(0xffffffffu, iz, o);
        if (lane >= o) { ip += tp; iz += tz; }
    }
    if (lane == 31) { s_w[0][warp] = ip; s_w[1][warp] = iz; }
    __syncthreads();
    if (warp == 0) {
        for (int q = 0; q < 2; q++) {
            long long v = (lane < T / 32) ? s_w[q][lane] : 0, vi = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long t = __shfl_up_sync(0xffffffffu, vi, o);
                if (lane >= o) vi += t;
            }
            if (lane < T / 32) s_w[q][lane] = vi - v;
        }
    }
    __syncthreads();
    long long rp = s_w[0][warp] + ip - sp, rz = s_w[1][warp] + iz - sz;
    for (long long i = b0; i < b1; i++) {
        const long long cp = a.cpo_off[i], cz = a.cnz_off[i];
        a.cpo_off[i] = rp; a.cnz_off[i] = rz; a.cin_off[i] = rz;
        rp += cp; rz += cz;
    }
    if (threadIdx.x == T - 1) {
        a.cpo_off[NC] = rp; a.cnz_off[NC] = rz; a.cin_off[NC] = rz;
        a.lengths[0] = rp; a.lengths[1] = rz; a.lengths[2] = rz;
        a.lengths[3] = (rp > a.cap_ptr || rz > a.cap_da || rz > a.cap_in) ? 1 : 0;
    }
}

__global__ void __launch_bounds__(kSaThreads) sa_write_kernel(SaArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geom& g = a.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long plane = (long long)blockIdx.x * kSaWarps + warp;
    if (a.lengths[3] || plane >= g.NC) return;
    const SaWarpSmem m = sa_warp_smem(g, smem, warp);
    warp_stage_counts(g, a.x, plane, m, lane);
    const long long P = a.cpo_off[plane], Z = a.cnz_off[plane];
    const int nnz = (int)(a.cnz_off[plane + 1] - Z);
    if (nnz == 0) {
        if (lane == 0) a.ptr[P] = SPC_NPC;
        return;
    }
    int tot[kSaMaxTypes];
    const unsigned present = type_totals(g, m.cnt, tot);
    // block layout (every lane walks the same few types): ptr position and DA base of each
    int pos = 0, run = 0;
    for (int t = 0; t < sa_ntypes(g); t++) {
        if (!((present >> t) & 1u)) continue;
        if (lane == 0) a.ptr[P + pos] = t + 1;
        if (tot[t] == 0) {
            if (lane == 0) a.ptr[P + pos + 1] = SPC_NPF;
            pos += 2;
            continue;
        }
        // the block's columns ascending: DA offsets (lane 0 writes them for the warp)
        if (lane == 0) {
            int r = run;
            for (int w = 0; w < g.Wp; w++)
                if (sa_cov(g, w) == t + 1) { m.coff[w] = r; r += m.cnt[w]; }
        }
        __syncwarp();
        // partition s's count = cumulative through its last owned type-t column
        for (int s2 = lane; s2 < g.Ow; s2 += 32) {
            int last = -1;
            for (int L = 0; L < g.S; L++) {
                const int w = s2 * g.sw + L;
                if (w < g.Wp && sa_cov(g, w) == t + 1 && sa_owner(g, w) == s2) last = w;
            }
            a.ptr[P + pos + 1 + s2] = (last < 0) ? -1 : m.coff[last] + m.cnt[last] - run;
        }
        run += tot[t];
        pos += 1 + g.Ow;
        __syncwarp();
    }
    // DA / IN: lanes over covered columns, rows ascending (from the staged plane)
    for (int w = lane; w < g.Wp; w += 32) {
        if (sa_cov(g, w) == 0 || m.cnt[w] == 0) continue;
        const int L = w - sa_owner(g, w) * g.sw;
        long long o = Z + m.coff[w];
        for (int h = g.pt; h < g.pt + g.H; h++) {
            const float v = plane_at(m.pl, g, h, w);
            if (v != 0.0f) {
                a.da[o] = v;
                a.in[o] = L + h * g.S;
                o++;
            }
        }
    }
}

// ---- convolution over the stride-aware layout
constexpr int kScCols = 4, kScKB = 64;

struct ScArgs {
    Geom g;
    const int32_t* __restrict__ ptr;
    const float* __restrict__ da;
    const int32_t* __restrict__ in;
    const int64_t* __restrict__ cpo_off;
    const int64_t* __restrict__ cnz_off;
    const float* __restrict__ wp;
    float* y;
    int relu;
    const unsigned long long* status;
};

__global__ void __launch_bounds__(32 * kScCols) sa_conv_kernel(ScArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geom& g = a.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int xo = blockIdx.x * kScCols + warp;
    const int kbase = blockIdx.y * kScKB;
    const int n = blockIdx.z;
    float2* acc = reinterpret_cast<float2*>(smem) + (size_t)warp * g.Oh * 32;
    for (int i = lane; i < g.Oh * 32; i += 32) acc[i] = make_float2(0.f, 0.f);
    pdl_wait();
    const bool bad = *reinterpret_cast<volatile const unsigned long long*>(a.status) != 0ull;
    const int k0 = kbase + 2 * lane;
    const bool k0ok = k0 < g.K, k1ok = k0 + 1 < g.K;
    // present types of the geometry (every lane computes the same mask)
    unsigned present = 0;
    for (int w = 0; w < g.Wp; w++) {
        const int cv = sa_cov(g, w);
        if (cv) present |= 1u << (cv - 1);
    }
    if (xo < g.Ow && !bad) {
        for (int c = 0; c < g.C; c++) {
            const long long nc = (long long)n * g.C + c;
            const long long P = a.cpo_off[nc], Z = a.cnz_off[nc];
            if (a.ptr[P] == SPC_NPC) continue;
            const float* wc = a.wp + (size_t)c * g.R * g.S * g.K;
            int q = 0, zb = 0;                                 // ptr cursor, block's DA base
            for (int t = 0; t < sa_ntypes(g); t++) {
                if (!((present >> t) & 1u)) continue;
                const int32_t* blk = a.ptr + P + q;
                if (blk[1] == SPC_NPF) { q += 2; continue; }
                const int32_t* cs = blk + 1;
                // owners s in [xo - t, xo] feed output column xo
                for (int s = max(0, xo - t); s <= xo; s++) {
                    if (cs[s] < 0) continue;
                    int lo = 0;
                    for (int s2 = s - 1; s2 >= 0; s2--)
                        if (cs[s2] >= 0) { lo = cs[s2]; break; }
                    const int hi = cs[s];
                    for (int b = lo; b < hi; b += 32) {
                        const int i = b + lane;
                        const float v = (i < hi) ? __ldg(a.da + Z + zb + i) : 0.f;
                        const int e = (i < hi) ? __ldg(a.in + Z + zb + i) : 0;
                        const int nb = min(32, hi - b);
                        for (int j = 0; j < nb; j++) {
                            const float vj = __shfl_sync(0xffffffffu, v, j);
                            const int ej = __shfl_sync(0xffffffffu, e, j);
                            const int h = ej / g.S, m = ej % g.S + (s - xo) * g.sw;   // tap column
                            if (m < 0 || m >= g.S) continue;
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
                int last = 0;                                    // block total = last non-negative count
                for (int s2 = g.Ow - 1; s2 >= 0; s2--)
                    if (cs[s2] >= 0) { last = cs[s2]; break; }
                zb += last;
                q += 1 + g.Ow;
            }
        }
    }
    __syncwarp();
    if (xo >= g.Ow) return;
    float* yb = a.y + (size_t)n * g.K * g.Oh * g.Ow;
    for (int yy = 0; yy < g.Oh; yy++) {
        float2 v = acc[yy * 32 + lane];
        if (a.relu) { v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); }
        if (k0ok) yb[((size_t)k0 * g.Oh + yy) * g.Ow + xo] = v.x;
        if (k1ok) yb[((size_t)(k0 + 1) * g.Oh + yy) * g.Ow + xo] = v.y;
    }
}

}  // namespace

size_t sa_smem_bytes(const Geom& g) {   // one warp's slice (the API's one-CTA limit)
    return align_up((size_t)g.H * g.W * 4 + (size_t)2 * g.Wp * 4, 16);
}

int sa_types(const Geom& g) { return (g.S + g.sw - 1) / g.sw; }

cudaError_t launch_sa_encode(const Geom& g, const float* x, spc_encoding* e, cudaStream_t st) {
    SaArgs a;
    a.g = g; a.x = x;
    a.ptr = e->ptr; a.da = e->da; a.in = e->in;
    a.cpo_off = e->chan_ptr_off; a.cnz_off = e->chan_nz_off; a.cin_off = e->chan_in_off;
    a.lengths = e->lengths;
    a.cap_ptr = e->ptr_cap; a.cap_da = e->da_cap; a.cap_in = e->in_cap;
    const size_t smem = sa_smem_bytes(g) * kSaWarps;
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    static std::atomic<size_t> attr_c[kMaxDevices], attr_w[kMaxDevices];
    cudaError_t err = ensure_smem_attr((const void*)sa_count_kernel, smem, attr_c);
    if (err == cudaSuccess) err = ensure_smem_attr((const void*)sa_write_kernel, smem, attr_w);
    if (err != cudaSuccess) return err;
    const unsigned blocks = (unsigned)((g.NC + kSaWarps - 1) / kSaWarps);
    sa_count_kernel<<<blocks, kSaThreads, smem, st>>>(a);
    sa_scan_kernel<<<1, 1024, 0, st>>>(a);
    sa_write_kernel<<<blocks, kSaThreads, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_sa_conv(const Geom& g, const spc_encoding* e, const float* w_packed, float* y, int relu,
                           cudaStream_t st) {
    ScArgs a;
    a.g = g;
    a.ptr = e->ptr; a.da = e->da; a.in = e->in;
    a.cpo_off = e->chan_ptr_off; a.cnz_off = e->chan_nz_off;
    a.wp = w_packed; a.y = y; a.relu = relu;
    a.status = reinterpret_cast<const unsigned long long*>(e->lengths + 3);
    const size_t smem = (size_t)kScCols * g.Oh * 32 * sizeof(float2);
    static std::atomic<size_t> attr[kMaxDevices];
    cudaError_t err = ensure_smem_attr((const void*)sa_conv_kernel, smem, attr);
    if (err != cudaSuccess) return err;
    dim3 grid((g.Ow + kScCols - 1) / kScCols, (g.K + kScKB - 1) / kScKB, g.N);
    sa_conv_kernel<<<grid, 32 * kScCols, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace spc
