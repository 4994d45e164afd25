// encode.cu -- single-pass CPO / CPS encoder for sm_100a.
//
// What it computes: the canonical CPO streams of Alg. 1 (
// SI Alg. 5 for K_w = 1) or the CPS streams of Alg. 3
// (PAPER.md:316-372), channels concatenated n-major then c (reading A19),
// plus the per-channel exclusive offsets (GPU side tables).
//
// How (B200 design, not the paper's serial loop):
//  * a tile = P consecutive channel planes (contiguous in NCHW) staged in
//    shared memory with coalesced 128-bit loads, many in flight per thread;
//    tiles are assigned statically to co-resident CTAs (grid <= resident
//    capacity, so no ticket atomic and no forward-progress hazard);
//  * per padded column a 32-bit row bitmask per 32-row word -> popc column
//    counts; NPF / NPC come from block / channel sums (Alg. 1 lines 31-37);
//    CPS set4 patterns are the 4-bit nibbles of the column masks (groups
//    anchored at padded row 0): popc decides {index, pattern} vs negated;
//  * stream offsets: a scan inside the tile, then every tile publishes its
//    aggregate once (epoch-tagged words, so nothing is ever reset) and sums
//    the aggregates of ALL its predecessors in parallel -- one L2 round trip,
//    no chained look-back;
//  * ptr / DA / IN are written once, DA/IN column by column with
//    ballot/popc compaction (warp per column).
//  * PDL: the kernel triggers its dependents at entry, so the convolution
//    that follows can stage its filter taps while the encoder runs.
#include <algorithm>

#include "common.cuh"

namespace spc {
namespace {

constexpr int kThreads = kEncWarps * 32;
constexpr int kTagShift = 40;
constexpr unsigned long long kValMask = (1ull << kTagShift) - 1;

struct EncArgs {
    Geom g;
    const float* __restrict__ x;
    int32_t* ptr; float* da; int32_t* in;
    int64_t* chan_ptr_off; int64_t* chan_nz_off; int64_t* chan_in_off;
    int64_t* lengths;
    int64_t cap_ptr, cap_da, cap_in;
    EncState* st;
    unsigned long long* agg;   // [3*ntiles] (tag << 40 | value)
    int ntiles;                // tiles of P planes
    int P;                     // planes per tile
};

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// padded column at position `pos` of the canonical stream order:
// NOP pair (0, Wp-1), then pairs (t, Wp-1-t) for t = 1..S-2, then the
// overlapK_w columns S-1..Wp-S ("first for NOP ... then overlap2,
// overlap3, etc., and overlapK_w"); identity for S = 1.
__device__ __forceinline__ int col_at(const Geom& g, int pos) {
    if (g.S == 1) return pos;
    const int edge = 2 * (g.S - 1);
    if (pos < edge) {
        const int t = pos >> 1;
        return (pos & 1) ? (g.Wp - 1 - t) : t;
    }
    return g.S - 1 + (pos - edge);
}

// local column index of padded column w inside its owner partition
// (owner(w) = max(0, w-S+1)).
__device__ __forceinline__ int local_of(const Geom& g, int w) { return (w >= g.S - 1) ? (g.S - 1) : w; }

__device__ __forceinline__ bool is_middle(const Geom& g, int w) {
    return g.S > 1 && w >= g.S - 1 && w <= g.Wp - g.S;
}

// shared-memory carve-up of one tile (host and device agree through this)
struct EncSmem {
    size_t planes, msk, cnt, incnt, dab, inb, pinfo, poff, total;
};
__host__ __device__ inline EncSmem enc_smem_layout(const Geom& g, int P) {
    EncSmem L;
    const size_t HW = (size_t)g.H * g.W, cols = (size_t)P * g.Wp;
    L.planes = 0;
    L.msk = align_up((P * HW + 8) * sizeof(float), 16);
    L.cnt = align_up(L.msk + cols * g.nwords * sizeof(unsigned), 16);
    L.incnt = L.cnt + cols * sizeof(int);
    L.dab = L.incnt + cols * sizeof(int);
    L.inb = L.dab + cols * sizeof(int);
    L.pinfo = align_up(L.inb + cols * sizeof(int), 16);            // [P][4]: plen, nnz, in_len, lower
    L.poff = align_up(L.pinfo + (size_t)P * 4 * sizeof(int), 16);   // [P][4] int64: ptr, da, in offsets, fits
    L.total = align_up(L.poff + (size_t)P * 4 * sizeof(long long), 16);
    return L;
}

template <bool CPS>
__global__ void __launch_bounds__(kThreads) encode_kernel(EncArgs a) {
    const Geom& g = a.g;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ long long s_red[kEncWarps][3];
    __shared__ long long s_tile_tot[3];
    __shared__ long long s_pre[3];
    __shared__ unsigned s_epoch;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int HW = g.H * g.W, Wp = g.Wp, NW = g.nwords;

    probe(0);
    pdl_wait();      // x may come from the kernel before us
    probe(1);
    pdl_trigger();   // the dependent convolution may launch and stage its taps
    if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile unsigned*>(&a.st->epoch);

    const EncSmem L = enc_smem_layout(g, a.P);
    float* planes = reinterpret_cast<float*>(smem_raw + L.planes);
    unsigned* msk = reinterpret_cast<unsigned*>(smem_raw + L.msk);   // [P][Wp][NW]
    int* cnt = reinterpret_cast<int*>(smem_raw + L.cnt);             // [P][Wp]
    int* incnt = reinterpret_cast<int*>(smem_raw + L.incnt);
    int* dab = reinterpret_cast<int*>(smem_raw + L.dab);
    int* inb = reinterpret_cast<int*>(smem_raw + L.inb);
    int* pinfo = reinterpret_cast<int*>(smem_raw + L.pinfo);
    long long* poff = reinterpret_cast<long long*>(smem_raw + L.poff);

    for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const long long plane0 = (long long)tile * a.P;
        const int np = (int)min((long long)a.P, g.NC - plane0);

        // ---- 1. stage the tile's planes: 128-bit loads from the 16-byte aligned
        //         element a0 <= e0 (x is 16-byte aligned), four in flight per thread
        const long long e0 = plane0 * HW, e1 = e0 + (long long)np * HW;
        const long long a0 = e0 & ~3ll;
        const int sh = (int)(e0 - a0);
        {
            const long long n4 = (e1 - a0) >> 2;
            const float4* s4 = reinterpret_cast<const float4*>(a.x + a0);
            float4* d4 = reinterpret_cast<float4*>(planes);
            for (long long i = threadIdx.x; i < n4; i += 4 * kThreads) {
                float4 v[4];
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (i + u * kThreads < n4) v[u] = __ldg(s4 + i + u * kThreads);
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (i + u * kThreads < n4) d4[i + u * kThreads] = v[u];
            }
            for (long long i = a0 + 4 * n4 + threadIdx.x; i < e1; i += kThreads) planes[i - a0] = __ldg(a.x + i);
        }
        __syncthreads();
        probe(2);
        const float* pl0 = planes + sh;

        // ---- 2. column bitmasks in the padded frame: item = (plane, word, column), column fastest
        for (int it = threadIdx.x; it < np * NW * Wp; it += kThreads) {
            const int w = it % Wp, pj = it / Wp, j = pj % NW, p = pj / NW;
            const int wu = w - g.pl;
            unsigned m = 0;
            if (wu >= 0 && wu < g.W) {
                const int h0 = 32 * j - g.pt;
                const int b0 = max(0, -h0), b1 = min(32, g.H - h0);
                const float* col = pl0 + (size_t)p * HW + wu;
#pragma unroll
                for (int b = 0; b < 32; b++)
                    if (b >= b0 && b < b1) m |= (unsigned)(col[(h0 + b) * g.W] != 0.0f) << b;
            }
            msk[(p * Wp + w) * NW + j] = m;
        }
        __syncthreads();

        probe(3);
        // ---- 3. per column: NZE count and IN entries (CPS set4 packing in overlapK_w)
        for (int it = threadIdx.x; it < np * Wp; it += kThreads) {
            const int w = it % Wp;
            int c = 0, e = 0;
            const bool mid = CPS && is_middle(g, w);
            for (int j = 0; j < NW; j++) {
                const unsigned m = msk[it * NW + j];
                c += __popc(m);
                if (mid) {
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const int k = __popc((m >> (4 * q)) & 0xFu);
                        e += k >= 3 ? 2 : k;   // {index, pattern} or k negated indices
                    }
                }
            }
            cnt[it] = c;
            incnt[it] = mid ? e : c;
        }
        __syncthreads();

        probe(4);
        // ---- 4. per plane (warp per plane): stream-order exclusive prefix over columns,
        //         plane totals and the ptr length (SI Eq. 3 with the actual NPF count)
        for (int p = warp; p < np; p += kEncWarps) {
            const int* wc = cnt + p * Wp;
            const int* wi = incnt + p * Wp;
            const int per = (Wp + 31) / 32;
            const int q0 = lane * per, q1 = min(q0 + per, Wp);
            int sd = 0, si = 0;
            for (int q = q0; q < q1; q++) {
                const int w = col_at(g, q);
                sd += wc[w];
                si += wi[w];
            }
            int td, ti;
            int ed = warp_exclusive_scan(sd, &td);
            int ei = warp_exclusive_scan(si, &ti);
            for (int q = q0; q < q1; q++) {
                const int w = col_at(g, q);
                dab[p * Wp + w] = ed;
                inb[p * Wp + w] = ei;
                ed += wc[w];
                ei += wi[w];
            }
            if (lane == 0) {
                int plen, lower = 0;
                if (td == 0) {
                    plen = 1;                                   // NPC
                } else if (g.S == 1) {
                    plen = 1 + g.Ow1;
                } else {
                    plen = (g.pl == 0) ? 3 : 0;                 // NOP block (reading A2)
                    for (int t = max(1, g.pl); t <= g.S - 2; t++) {
                        const int bn = wc[t] + wc[Wp - 1 - t];
                        lower += bn;
                        plen += bn ? (1 + g.Ow1) : 2;           // block or [tag, NPF] (reading A3)
                    }
                    if (g.pl == 0) lower += wc[0] + wc[Wp - 1];
                    plen += (td - lower) ? (1 + g.Ow1) : 2;
                }
                int* pi = pinfo + 4 * p;
                pi[0] = plen; pi[1] = td; pi[2] = ti; pi[3] = lower;
            }
        }
        __syncthreads();

        probe(5);
        // ---- 5. exclusive scan over the tile's planes (warp 0) -> tile aggregate
        if (warp == 0) {
            long long r0 = 0, r1 = 0, r2 = 0;
            for (int b = 0; b < np; b += 32) {
                const int p = b + lane;
                long long v0 = 0, v1 = 0, v2 = 0;
                if (p < np) { v0 = pinfo[4 * p]; v1 = pinfo[4 * p + 1]; v2 = pinfo[4 * p + 2]; }
                long long t0, t1, t2;
                const long long x0 = warp_exclusive_scan(v0, &t0);
                const long long x1 = warp_exclusive_scan(v1, &t1);
                const long long x2 = warp_exclusive_scan(v2, &t2);
                if (p < np) { poff[4 * p] = r0 + x0; poff[4 * p + 1] = r1 + x1; poff[4 * p + 2] = r2 + x2; }
                r0 += t0; r1 += t1; r2 += t2;
            }
            if (lane == 0) { s_tile_tot[0] = r0; s_tile_tot[1] = r1; s_tile_tot[2] = r2; }
        }
        __syncthreads();

        probe(6);
        // ---- 6. publish the tile aggregate; prefix = sum over ALL preceding tiles
        const unsigned long long tag = (unsigned long long)((s_epoch + 1u) & 0xFFFFFFu);
        if (threadIdx.x < 3)
            st_relaxed64(a.agg + 3ll * tile + threadIdx.x, (tag << kTagShift) | (unsigned long long)s_tile_tot[threadIdx.x]);
        {
            long long p0 = 0, p1 = 0, p2 = 0;
            for (long long i = threadIdx.x; i < 3ll * tile; i += kThreads) {
                unsigned long long v;
                long long spin = 0;
                while (((v = ld_relaxed64(a.agg + i)) >> kTagShift) != tag)
                    if (++spin > (1ll << 26)) __trap();   // bounded: never hang the GPU
                const long long val = (long long)(v & kValMask);
                const int s = (int)(i % 3);
                p0 += (s == 0) ? val : 0;
                p1 += (s == 1) ? val : 0;
                p2 += (s == 2) ? val : 0;
            }
            p0 = warp_sum(p0); p1 = warp_sum(p1); p2 = warp_sum(p2);
            if (lane == 0) { s_red[warp][0] = p0; s_red[warp][1] = p1; s_red[warp][2] = p2; }
        }
        __syncthreads();
        if (threadIdx.x < 3) {
            long long s = 0;
            for (int w = 0; w < kEncWarps; w++) s += s_red[w][threadIdx.x];
            s_pre[threadIdx.x] = s;
        }
        __syncthreads();
        probe(7);
        const long long P0 = s_pre[0], Z0 = s_pre[1], Q0 = s_pre[2];
        if (tile == a.ntiles - 1 && threadIdx.x == 0) {
            // every other tile has published, so every CTA has read the epoch
            const long long t0 = P0 + s_tile_tot[0], t1 = Z0 + s_tile_tot[1], t2 = Q0 + s_tile_tot[2];
            a.chan_ptr_off[g.NC] = t0;
            a.chan_nz_off[g.NC] = t1;
            a.chan_in_off[g.NC] = t2;
            a.lengths[0] = t0;
            a.lengths[1] = t1;
            a.lengths[2] = t2;
            a.lengths[3] = (t0 > a.cap_ptr || t1 > a.cap_da || t2 > a.cap_in) ? 1 : 0;
            a.st->epoch = s_epoch + 1u;
        }
        for (int p = threadIdx.x; p < np; p += kThreads) {
            const long long P = P0 + poff[4 * p], Z = Z0 + poff[4 * p + 1], Q = Q0 + poff[4 * p + 2];
            a.chan_ptr_off[plane0 + p] = P;
            a.chan_nz_off[plane0 + p] = Z;
            a.chan_in_off[plane0 + p] = Q;
            poff[4 * p] = P; poff[4 * p + 1] = Z; poff[4 * p + 2] = Q;
            poff[4 * p + 3] = (P + pinfo[4 * p] <= a.cap_ptr) && (Z + pinfo[4 * p + 1] <= a.cap_da) &&
                              (Q + pinfo[4 * p + 2] <= a.cap_in);
        }
        __syncthreads();

        probe(8);
        // ---- 7a. ptr segments (warp per plane; Alg. 1 lines 9-37, canonical layout)
        for (int p = warp; p < np; p += kEncWarps) {
            if (!poff[4 * p + 3]) continue;
            const int* wc = cnt + p * Wp;
            const int nnz = pinfo[4 * p + 1];
            int32_t* pp = a.ptr + poff[4 * p];
            if (nnz == 0) {
                if (lane == 0) pp[0] = SPC_NPC;
            } else if (g.S == 1) {
                if (lane == 0) pp[0] = 0;
                const int* wd = dab + p * Wp;
                for (int s = lane; s < g.Ow1; s += 32) pp[1 + s] = wd[s] + wc[s];
            } else {
                int q = 0;
                if (g.pl == 0) {
                    if (lane == 0) {
                        pp[0] = 0;
                        pp[1] = wc[0];
                        pp[2] = wc[0] + wc[Wp - 1];
                    }
                    q = 3;
                }
                for (int t = max(1, g.pl); t <= g.S - 2; t++) {
                    const int bn = wc[t] + wc[Wp - 1 - t];
                    if (bn == 0) {
                        if (lane == 0) { pp[q] = t + 1; pp[q + 1] = SPC_NPF; }
                        q += 2;
                    } else {
                        if (lane == 0) pp[q] = t + 1;
                        for (int s = lane; s < g.Ow1; s += 32)
                            pp[q + 1 + s] = (s == 0) ? wc[t] : (s == g.Ow1 - 1 - t ? bn : -1);
                        q += 1 + g.Ow1;
                    }
                }
                const int bn = nnz - pinfo[4 * p + 3];
                if (bn == 0) {
                    if (lane == 0) { pp[q] = g.S; pp[q + 1] = SPC_NPF; }
                } else {
                    if (lane == 0) pp[q] = g.S;
                    const int* wd = dab + p * Wp;
                    const int base = wd[g.S - 1];
                    for (int s = lane; s < g.Ow1; s += 32)
                        pp[q + 1 + s] = (s <= g.Ow1 - g.S) ? (wd[s + g.S - 1] + wc[s + g.S - 1] - base) : -1;
                }
            }
        }

        probe(9);
        // ---- 7b. DA / IN, column by column (G of Alg. 1), warp per (plane, column)
        for (int it = warp; it < np * Wp; it += kEncWarps) {
            if (cnt[it] == 0) continue;
            const int p = it / Wp, w = it % Wp;
            if (!poff[4 * p + 3]) continue;
            const int L = local_of(g, w);
            const int wu = w - g.pl;
            const float* pl = pl0 + (size_t)p * HW;
            float* dd = a.da + poff[4 * p + 1] + dab[it];
            int32_t* ii = a.in + poff[4 * p + 2] + inb[it];
            const bool mid = CPS && is_middle(g, w);
            int run = 0, irun = 0;
            for (int j = 0; j < NW; j++) {
                const unsigned m = msk[it * NW + j];
                if (m == 0) continue;
                const int h = 32 * j + lane;
                if ((m >> lane) & 1u) {
                    const int r = run + __popc(m & lanemask_lt());
                    dd[r] = pl[(h - g.pt) * g.W + wu];
                    if (!mid) ii[r] = L + h * g.S;
                }
                run += __popc(m);
                if (mid) {
                    // set4 packing: lanes 0..7 own the 8 nibbles of this word
                    int k = 0, e = 0;
                    unsigned nib = 0;
                    if (lane < 8) {
                        nib = (m >> (4 * lane)) & 0xFu;
                        k = __popc(nib);
                        e = k >= 3 ? 2 : k;
                    }
                    int te;
                    const int eo = warp_exclusive_scan(e, &te);
                    if (lane < 8 && k) {
                        const int row0 = 32 * j + 4 * lane;
                        int32_t* o = ii + irun + eo;
                        if (k >= 3) {
                            o[0] = L + (row0 + __ffs(nib) - 1) * g.S;  // first NZE index (A9)
                            o[1] = (int32_t)nib;                         // pattern, bit b = row b (A12)
                        } else {
                            int u = 0;
                            for (int b = 0; b < 4; b++)
                                if ((nib >> b) & 1u) o[u++] = -(L + (row0 + b) * g.S);
                        }
                    }
                    irun += te;
                }
            }
        }
        __syncthreads();   // the next tile reuses the shared memory
        probe(10);
    }
}

struct EncPlan {
    int P, ntiles, grid;
    size_t smem;
};

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Tile size: about one tile per resident CTA (2 per SM when the tile fits in
// ~100 KB of smem, else 1), capped by the shared-memory stage.
EncPlan plan_encode(const Geom& g) {
    EncPlan pl;
    const int sms = sm_count();
    const size_t b2 = 100 * 1024, b1 = 220 * 1024;
    long long P = (g.NC + 2 * sms - 1) / (2 * sms);
    if (enc_smem_layout(g, (int)P).total > b2) {
        P = (g.NC + sms - 1) / sms;
        while (P > 1 && enc_smem_layout(g, (int)P).total > b1) P--;
    }
    pl.P = (int)std::max(1ll, P);
    pl.ntiles = (int)((g.NC + pl.P - 1) / pl.P);
    pl.smem = enc_smem_layout(g, pl.P).total;
    pl.grid = pl.ntiles;
    return pl;
}

}  // namespace

size_t enc_smem_bytes(const Geom& g) { return plan_encode(g).smem; }

cudaError_t launch_encode(const Geom& g, bool cps, const float* x, spc_encoding* e, void* ws, cudaStream_t st) {
    WsLayout W = ws_layout(g);
    EncArgs a;
    a.g = g; a.x = x;
    a.ptr = e->ptr; a.da = e->da; a.in = e->in;
    a.chan_ptr_off = e->chan_ptr_off; a.chan_nz_off = e->chan_nz_off; a.chan_in_off = e->chan_in_off;
    a.lengths = e->lengths;
    a.cap_ptr = e->ptr_cap; a.cap_da = e->da_cap; a.cap_in = e->in_cap;
    unsigned char* base = static_cast<unsigned char*>(ws);
    a.st = reinterpret_cast<EncState*>(base + W.state);
    a.agg = reinterpret_cast<unsigned long long*>(base + W.agg);
    EncPlan pl = plan_encode(g);
    a.P = pl.P;
    a.ntiles = pl.ntiles;
    void (*kern)(EncArgs) = cps ? encode_kernel<true> : encode_kernel<false>;
    static size_t attr_bytes[2] = {0, 0};
    if (attr_bytes[cps] < pl.smem) {
        cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
        if (err != cudaSuccess) return err;
        attr_bytes[cps] = pl.smem;
    }
    // the cross-tile prefix needs every CTA resident: cap the grid at the
    // occupancy limit (CTAs then loop over tiles in increasing order)
    int occ = 0;
    cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, pl.smem);
    if (err != cudaSuccess) return err;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const int grid = std::min(pl.ntiles, occ * sm_count());
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace spc

#ifdef SPC_PROBES
SPC_PROBE_ACCESSOR(spc_debug_probes_enc)
#endif
