// fused_encode.cu -- NEXT-1: the convolution's output emitted already CPO-encoded for the next
// layer ("after activation map compression, CPO/CPS performs convolution": in a
// chain of sparse layers the compression of layer i+1's input belongs to layer i).
//
// The conv kernels (strip / warp-specialised / generic) take an optional `omask`: in their
// epilogue every output element that is non-zero after the (fused) ReLU sets its row bit in a
// 64-bit mask per output column (n, k, x) -- the encoder's "column masks" pass (Alg. 1's G()
// scan for NZEs) done by the kernel that produced the values, so the dense map is
// never re-scanned.  One launch then turns the masks into the next layer's canonical
// CPO streams (DESIGN.md Appendix A: NOP iff pad_left = 0, blocks t = max(1, pad_left) .. S-1
// with NPF / -1 rules, DA / IN column by column in stream order, IN = L + h*S):
//  a CTA per tile of planes: column counts (popc of the masks shifted into the next layer's
//  padded frame), NZE totals and ptr lengths (SI Eq. 3 with the plane's NPF flags), a scan
//  over the tile, the cross-tile prefix (epoch-tagged aggregates, as the stand-alone encoder),
//  then ptr blocks and one thread per NZE (column, row) gathering its value from y (only the
//  NZEs are read) for DA / IN; the masks are re-zeroed for the next launch.
// The streams are bit-identical to encoding y with cpo_encode (tests/test_gpu_fused.py).
#include <algorithm>

#include "common.cuh"

namespace spc {
namespace {

constexpr int kFeThreads = 512;

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

constexpr int kFeTagShift = 40;
constexpr unsigned long long kFeValMask = (1ull << kFeTagShift) - 1;

__device__ __forceinline__ unsigned long long fe_ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fe_st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct FeState {
    unsigned epoch;
    unsigned pad[63];
};

// One launch (cooperative: every tile's CTA is resident, so the cross-tile prefix cannot
// deadlock).  A CTA owns a tile of P consecutive planes: column counts from the masks, the
// stream-order column offsets and ptr length of every plane, a scan over the tile, then its
// aggregate is published (epoch-tagged words, never reset) and the aggregates of all preceding
// tiles are summed (one L2 round trip, as in the stand-alone encoder); then ptr, DA / IN (one
// thread per NZE, values gathered from y) and the side tables are written and the masks
// re-zeroed.  The last tile writes the lengths and advances the epoch.
__global__ void __launch_bounds__(kFeThreads) fe_encode_kernel(FeArgs a, FeState* st, unsigned long long* agg, int P,
                                                                int ntiles) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ long long s_pre[2], s_red[kFeThreads / 32][2], s_tot[2];
    __shared__ unsigned s_epoch;
    const Geom& g = a.g;
    const int Wp = g.Wp, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long* msk = reinterpret_cast<unsigned long long*>(smem);     // [P][Wp]
    int* cnt = reinterpret_cast<int*>(msk + (size_t)P * Wp);                   // [P][Wp]
    int* dab = cnt + (size_t)P * Wp;                                           // [P][Wp]
    int* pinfo = dab + (size_t)P * Wp;                                         // [P][4]: plen, nnz, lower
    long long* poff = reinterpret_cast<long long*>(pinfo + 4 * P + 4);         // [P][2] tile-relative
    const int tile = blockIdx.x;
    const long long p0 = (long long)tile * P;
    const int np = (int)min((long long)P, g.NC - p0);
    pdl_wait();
    if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile unsigned*>(&st->epoch);
    for (int it = threadIdx.x; it < np * Wp; it += blockDim.x) {
        const int p = it / Wp, w = it % Wp;
        const unsigned long long m = col_mask(a, p0 + p, w);
        msk[it] = m;
        cnt[it] = __popcll(m);
    }
    __syncthreads();
    for (int p = threadIdx.x; p < np; p += blockDim.x) {
        const int* c = cnt + p * Wp;
        int run = 0;
        for (int q = 0; q < Wp; q++) {
            const int w = fe_col_at(g, q);
            dab[p * Wp + w] = run;
            run += c[w];
        }
        int lower;
        pinfo[4 * p] = fe_plane_len(g, c, run, &lower);
        pinfo[4 * p + 1] = run;
        pinfo[4 * p + 2] = lower;
    }
    __syncthreads();
    if (warp == 0) {   // scan over the tile's planes
        long long r0 = 0, r1 = 0;
        for (int b = 0; b < np; b += 32) {
            const int p = b + lane;
            long long v0 = 0, v1 = 0, t0, t1;
            if (p < np) { v0 = pinfo[4 * p]; v1 = pinfo[4 * p + 1]; }
            const long long x0 = warp_exclusive_scan(v0, &t0), x1 = warp_exclusive_scan(v1, &t1);
            if (p < np) { poff[2 * p] = r0 + x0; poff[2 * p + 1] = r1 + x1; }
            r0 += t0; r1 += t1;
        }
        if (lane == 0) { s_tot[0] = r0; s_tot[1] = r1; }
    }
    __syncthreads();
    const unsigned long long tag = (unsigned long long)((s_epoch + 1u) & 0xFFFFFFu);
    if (threadIdx.x == 0) {
        fe_st_relaxed(agg + 2ll * tile, (tag << kFeTagShift) | (unsigned long long)s_tot[0]);
        fe_st_relaxed(agg + 2ll * tile + 1, (tag << kFeTagShift) | (unsigned long long)s_tot[1]);
    }
    {   // prefix = sum over every preceding tile (all resident: cooperative launch)
        long long q0 = 0, q1 = 0;
        for (long long i = threadIdx.x; i < 2ll * tile; i += blockDim.x) {
            unsigned long long v;
            long long spin = 0;
            while (((v = fe_ld_relaxed(agg + i)) >> kFeTagShift) != tag)
                if (++spin > (1ll << 24)) break;   // bounded (co-resident grid: unreachable)
            const long long val = (long long)(v & kFeValMask);
            if (i & 1) q1 += val; else q0 += val;
        }
        q0 = warp_sum(q0); q1 = warp_sum(q1);
        if (lane == 0) { s_red[warp][0] = q0; s_red[warp][1] = q1; }
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        long long v = 0;
        for (int w = 0; w < kFeThreads / 32; w++) v += s_red[w][threadIdx.x];
        s_pre[threadIdx.x] = v;
    }
    __syncthreads();
    const long long P0 = s_pre[0], Z0 = s_pre[1];
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        const long long t0 = P0 + s_tot[0], t1 = Z0 + s_tot[1];
        a.cpo_off[g.NC] = t0; a.cnz_off[g.NC] = t1; a.cin_off[g.NC] = t1;
        a.lengths[0] = t0; a.lengths[1] = t1; a.lengths[2] = t1;
        a.lengths[3] = (t0 > a.cap_ptr || t1 > a.cap_da || t1 > a.cap_in) ? 1 : 0;
        st->epoch = s_epoch + 1u;   // every tile has published, so every CTA has read the epoch
    }
    // ptr segments and side tables: thread per plane
    for (int p = threadIdx.x; p < np; p += blockDim.x) {
        const long long Pp = P0 + poff[2 * p], Zp = Z0 + poff[2 * p + 1];
        a.cpo_off[p0 + p] = Pp; a.cnz_off[p0 + p] = Zp; a.cin_off[p0 + p] = Zp;
        const int plen = pinfo[4 * p], nnz = pinfo[4 * p + 1], lower = pinfo[4 * p + 2];
        pinfo[4 * p + 3] = (Pp + plen <= a.cap_ptr && Zp + nnz <= a.cap_da && Zp + nnz <= a.cap_in) ? 1 : 0;
        if (!pinfo[4 * p + 3]) continue;
        const int* c = cnt + p * Wp;
        const int* db = dab + p * Wp;
        int32_t* pp = a.ptr + Pp;
        if (nnz == 0) {
            pp[0] = SPC_NPC;
        } else if (g.S == 1) {
            pp[0] = 0;
            for (int s2 = 0; s2 < g.Ow1; s2++) pp[1 + s2] = db[s2] + c[s2];
        } else {
            int q = 0;
            if (g.pl == 0) { pp[0] = 0; pp[1] = c[0]; pp[2] = c[0] + c[Wp - 1]; q = 3; }
            for (int t = max(1, g.pl); t <= g.S - 2; t++) {
                const int bn = c[t] + c[Wp - 1 - t];
                pp[q] = t + 1;
                if (bn == 0) { pp[q + 1] = SPC_NPF; q += 2; continue; }
                for (int s2 = 0; s2 < g.Ow1; s2++) pp[q + 1 + s2] = (s2 == 0) ? c[t] : (s2 == g.Ow1 - 1 - t ? bn : -1);
                q += 1 + g.Ow1;
            }
            pp[q] = g.S;
            if (nnz - lower == 0) {
                pp[q + 1] = SPC_NPF;
            } else {
                const int base = db[g.S - 1];
                for (int s2 = 0; s2 < g.Ow1; s2++)
                    pp[q + 1 + s2] = (s2 <= g.Ow1 - g.S) ? (db[s2 + g.S - 1] + c[s2 + g.S - 1] - base) : -1;
            }
        }
    }
    __syncthreads();
    // DA / IN: one thread per (plane, padded column, padded row) holding an NZE; the rank in its
    // column is the popc of the mask below the row; 4 pairs per thread in flight at once (the
    // gathers from y are the latency that bounds this kernel)
    {
        const int per_plane = Wp * g.Hp, total = np * per_plane;
        constexpr int U = 4;
        for (int base = threadIdx.x; base < total; base += U * blockDim.x) {
            long long o[U];
            float v[U];
            int e[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                o[u] = -1;
                const int it = base + u * blockDim.x;
                if (it >= total) continue;
                const int p = it / per_plane, r = it - p * per_plane, w = r / g.Hp, h = r - w * g.Hp;
                const unsigned long long m = msk[p * Wp + w];
                if (!((m >> h) & 1ull) || !pinfo[4 * p + 3]) continue;
                o[u] = Z0 + poff[2 * p + 1] + dab[p * Wp + w] + __popcll(m & ((1ull << h) - 1ull));
                v[u] = a.y[(p0 + p) * g.H * g.W + (long long)(h - g.pt) * g.W + (w - g.pl)];
                e[u] = ((g.S == 1) ? 0 : fe_local(g, w)) + h * g.S;
            }
#pragma unroll
            for (int u = 0; u < U; u++)
                if (o[u] >= 0) { a.da[o[u]] = v[u]; a.in[o[u]] = e[u]; }
        }
    }
    for (int it = threadIdx.x; it < np * g.W; it += blockDim.x) a.omask[p0 * g.W + it] = 0ull;   // next launch
}

}  // namespace

size_t fe_state_bytes(const Geom& gn) { return sizeof(FeState) + 16 * (size_t)gn.NC + 256; }

static size_t fe_smem(const Geom& gn, int P) {
    return (size_t)P * gn.Wp * (8 + 4 + 4) + (size_t)(4 * P + 4) * 4 + (size_t)P * 16 + 16;
}

cudaError_t launch_encode_from_masks(const Geom& gn, const float* y, unsigned long long* omask, spc_encoding* e,
                                     void* state, cudaStream_t st) {
    FeArgs a;
    a.g = gn; a.y = y; a.omask = omask;
    a.ptr = e->ptr; a.da = e->da; a.in = e->in;
    a.cpo_off = e->chan_ptr_off; a.cnz_off = e->chan_nz_off; a.cin_off = e->chan_in_off;
    a.lengths = e->lengths;
    a.cap_ptr = e->ptr_cap; a.cap_da = e->da_cap; a.cap_in = e->in_cap;
    FeState* fs = static_cast<FeState*>(state);
    unsigned long long* agg = reinterpret_cast<unsigned long long*>(fs + 1);
    // tile size: enough tiles for every SM (co-resident: cooperative launch), smem <= 48 KB
    const int sms = device_sm_count();
    int P = (int)std::max<long long>(1, (gn.NC + 2LL * sms - 1) / (2LL * sms));
    while (P > 1 && fe_smem(gn, P) > 48 * 1024) P--;
    const int ntiles = (int)((gn.NC + P - 1) / P);
    const size_t smem = fe_smem(gn, P);
    int occ = 0;
    cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fe_encode_kernel, kFeThreads, smem);
    if (err != cudaSuccess) return err;
    if ((long long)occ * sms < ntiles) return cudaErrorCooperativeLaunchTooLarge;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntiles);
    cfg.blockDim = dim3(kFeThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cooperative_launches() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fe_encode_kernel, a, fs, agg, P, ntiles);
}

}  // namespace spc
