// fused_encode.cu -- NEXT-1: the convolution's output emitted already CPO-encoded for the next
// layer ("after activation map compression, CPO/CPS performs convolution": in a
// chain of sparse layers the compression of layer i+1's input belongs to layer i).
//
// The conv kernels (strip / warp-specialised / generic) take an optional `omask`: in their
// epilogue every output element that is non-zero after the (fused) ReLU sets its row bit in a
// 64-bit mask per output column (n, k, x) -- the encoder's "column masks" pass (Alg. 1's G()
// scan for NZEs) done by the kernel that produced the values, so the dense map is
// never re-scanned.  These three launches then turn the masks into the next layer's canonical
// CPO streams (DESIGN.md Appendix A: NOP iff pad_left = 0, blocks t = max(1, pad_left) .. S-1
// with NPF / -1 rules, DA / IN column by column in stream order, IN = L + h*S):
//  (1) per plane: column counts (popc of the masks shifted into the next layer's padded frame),
//      NZE total and ptr length (SI Eq. 3 with the plane's NPF flags);
//  (2) one CTA: exclusive scans -> the side tables and lengths;
//  (3) per plane: ptr blocks, then one thread per column gathers its NZE values from y at the
//      mask bits (only the NZEs are read) and writes DA / IN; the masks are re-zeroed for the
//      next launch.
// The streams are bit-identical to encoding y with cpo_encode (tests/test_gpu_fused.py).
#include <algorithm>

#include "common.cuh"

namespace spc {
namespace {

constexpr int kFeThreads = 128;

struct FeArgs {
    Geom g;                          // the NEXT layer's geometry (input = this conv's output)
    const float* __restrict__ y;     // dense output of the conv, N*C*H*W of the next layer
    unsigned long long* omask;       // [N*C*W] row masks of y (unpadded rows), zeroed here after use
    int32_t* ptr; float* da; int32_t* in;
    int64_t* cpo_off; int64_t* cnz_off; int64_t* cin_off;
    int64_t* lengths;
    int64_t cap_ptr, cap_da, cap_in;
};

// padded column w of the next layer's frame: mask of padded rows
__device__ __forceinline__ unsigned long long col_mask(const FeArgs& a, long long plane, int w) {
    const Geom& g = a.g;
    const int c = w - g.pl;
    if (c < 0 || c >= g.W) return 0ull;
    return a.omask[plane * g.W + c] << g.pt;
}

// canonical stream order of padded columns (NOP pair, type pairs, overlapK_w run; identity for S = 1)
__device__ __forceinline__ int fe_col_at(const Geom& g, int pos) {
    if (g.S == 1) return pos;
    const int edge = 2 * (g.S - 1);
    if (pos < edge) {
        const int t = pos >> 1;
        return (pos & 1) ? (g.Wp - 1 - t) : t;
    }
    return g.S - 1 + (pos - edge);
}

__device__ __forceinline__ int fe_local(const Geom& g, int w) { return (w >= g.S - 1) ? (g.S - 1) : w; }

// ptr length and DA count below the overlapK_w block of a plane with column counts cnt
__device__ int fe_plane_len(const Geom& g, const int* cnt, int nnz, int* lower_out) {
    if (nnz == 0) { *lower_out = 0; return 1; }          // NPC
    if (g.S == 1) { *lower_out = 0; return 1 + g.Ow1; }
    int plen = (g.pl == 0) ? 3 : 0, lower = (g.pl == 0) ? cnt[0] + cnt[g.Wp - 1] : 0;
    for (int t = max(1, g.pl); t <= g.S - 2; t++) {
        const int bn = cnt[t] + cnt[g.Wp - 1 - t];
        lower += bn;
        plen += bn ? (1 + g.Ow1) : 2;
    }
    plen += (nnz - lower) ? (1 + g.Ow1) : 2;
    *lower_out = lower;
    return plen;
}

__global__ void __launch_bounds__(kFeThreads) fe_count_kernel(FeArgs a) {
    __shared__ int cnt[256];
    const Geom& g = a.g;
    const long long plane = blockIdx.x;
    pdl_wait();
    for (int w = threadIdx.x; w < g.Wp; w += blockDim.x) cnt[w] = __popcll(col_mask(a, plane, w));
    __syncthreads();
    if (threadIdx.x == 0) {
        int nnz = 0, lower;
        for (int w = 0; w < g.Wp; w++) nnz += cnt[w];
        a.cpo_off[plane] = fe_plane_len(g, cnt, nnz, &lower);
        a.cnz_off[plane] = nnz;
    }
}

__global__ void __launch_bounds__(1024) fe_scan_kernel(FeArgs a) {
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

__global__ void __launch_bounds__(kFeThreads) fe_write_kernel(FeArgs a) {
    __shared__ int cnt[256], dab[256];
    __shared__ unsigned long long msk[256];
    const Geom& g = a.g;
    const long long plane = blockIdx.x;
    const bool ok = a.lengths[3] == 0;
    for (int w = threadIdx.x; w < g.Wp; w += blockDim.x) {
        msk[w] = col_mask(a, plane, w);
        cnt[w] = __popcll(msk[w]);
    }
    __syncthreads();
    const long long P = a.cpo_off[plane], Z = a.cnz_off[plane];
    const int nnz = (int)(a.cnz_off[plane + 1] - Z);
    if (ok && threadIdx.x == 0) {
        // stream-order DA offsets of the columns, then the ptr segment (Alg. 1 lines 9-37)
        int run = 0;
        for (int q = 0; q < g.Wp; q++) {
            const int w = fe_col_at(g, q);
            dab[w] = run;
            run += cnt[w];
        }
        int32_t* pp = a.ptr + P;
        if (nnz == 0) {
            pp[0] = SPC_NPC;
        } else if (g.S == 1) {
            pp[0] = 0;
            for (int s = 0; s < g.Ow1; s++) pp[1 + s] = dab[s] + cnt[s];
        } else {
            int q = 0, lower;
            fe_plane_len(g, cnt, nnz, &lower);
            if (g.pl == 0) { pp[0] = 0; pp[1] = cnt[0]; pp[2] = cnt[0] + cnt[g.Wp - 1]; q = 3; }
            for (int t = max(1, g.pl); t <= g.S - 2; t++) {
                const int bn = cnt[t] + cnt[g.Wp - 1 - t];
                pp[q] = t + 1;
                if (bn == 0) { pp[q + 1] = SPC_NPF; q += 2; continue; }
                for (int s = 0; s < g.Ow1; s++) pp[q + 1 + s] = (s == 0) ? cnt[t] : (s == g.Ow1 - 1 - t ? bn : -1);
                q += 1 + g.Ow1;
            }
            pp[q] = g.S;
            if (nnz - lower == 0) {
                pp[q + 1] = SPC_NPF;
            } else {
                const int base = dab[g.S - 1];
                for (int s = 0; s < g.Ow1; s++)
                    pp[q + 1 + s] = (s <= g.Ow1 - g.S) ? (dab[s + g.S - 1] + cnt[s + g.S - 1] - base) : -1;
            }
        }
    }
    __syncthreads();
    // DA / IN: one thread per padded column, its NZE rows ascending (values gathered from y)
    if (ok) {
        const float* yp = a.y + plane * g.H * g.W;
        for (int w = threadIdx.x; w < g.Wp; w += blockDim.x) {
            unsigned long long m = msk[w];
            long long o = Z + dab[w];
            const int L = (g.S == 1) ? 0 : fe_local(g, w);
            while (m) {
                const int h = __ffsll((long long)m) - 1;
                m &= m - 1;
                a.da[o] = yp[(h - g.pt) * g.W + (w - g.pl)];
                a.in[o] = L + h * g.S;
                o++;
            }
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < g.W; c += blockDim.x) a.omask[plane * g.W + c] = 0ull;   // for the next launch
}

}  // namespace

cudaError_t launch_encode_from_masks(const Geom& gn, const float* y, unsigned long long* omask, spc_encoding* e,
                                     cudaStream_t st) {
    FeArgs a;
    a.g = gn; a.y = y; a.omask = omask;
    a.ptr = e->ptr; a.da = e->da; a.in = e->in;
    a.cpo_off = e->chan_ptr_off; a.cnz_off = e->chan_nz_off; a.cin_off = e->chan_in_off;
    a.lengths = e->lengths;
    a.cap_ptr = e->ptr_cap; a.cap_da = e->da_cap; a.cap_in = e->in_cap;
    fe_count_kernel<<<(unsigned)gn.NC, kFeThreads, 0, st>>>(a);
    fe_scan_kernel<<<1, 1024, 0, st>>>(a);
    fe_write_kernel<<<(unsigned)gn.NC, kFeThreads, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace spc
