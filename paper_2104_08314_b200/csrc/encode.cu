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
constexpr unsigned kBulkChunk = 1u << 15;   // bytes per cp.async.bulk
constexpr int kTagShift = 40;
constexpr unsigned long long kValMask = (1ull << kTagShift) - 1;
constexpr int kTabIn = 1 << 16, kTabOk = 1 << 17;   // column-table flags (low 16 bits: local column)
constexpr long long kSpinLimit = 1ll << 24;         // polls before a cross-tile wait gives up

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
    // prefix wait: one round (all tiles resident): thread 0 waits on the round's counter, then
    // the aggregates are read once; several rounds: every thread spins on the tagged aggregates
    // it sums (its predecessors only), so later rounds' staging overlaps earlier stream writes
    // (measured: batch-256 cfg5-L3 493 -> 454 us; one round is faster with the counter)
    int multi_round;
};

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
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
    size_t planes, umask, msk, cnt, incnt, dab, inb, tab, pinfo, poff, sa_ord, sa_col, sa_last, total;
};
__host__ __device__ inline int sa_ntypes_of(const Geom& g) { return (g.S + g.sw - 1) / g.sw; }
__host__ __device__ inline EncSmem enc_smem_layout(const Geom& g, int P, bool sa = false) {
    EncSmem L;
    const size_t HW = (size_t)g.H * g.W, cols = (size_t)P * g.Wp;
    const size_t nrb = (g.H + 31) / 32;
    L.planes = 0;
    L.umask = align_up((P * HW + 8) * sizeof(float), 16);          // [P][W][nrb] unpadded column masks
    L.msk = align_up(L.umask + (size_t)P * g.W * nrb * sizeof(unsigned), 16);
    L.cnt = align_up(L.msk + cols * g.nwords * sizeof(unsigned), 16);
    L.incnt = L.cnt + cols * sizeof(int);
    L.dab = L.incnt + cols * sizeof(int);
    L.inb = L.dab + cols * sizeof(int);
    L.tab = align_up(L.inb + cols * sizeof(int), 16);              // [P][Wp] int4 column table
    L.pinfo = align_up(L.tab + cols * sizeof(int4), 16);           // [P][4]: plen, nnz, in_len, lower
    L.poff = align_up(L.pinfo + (size_t)P * 4 * sizeof(int), 16);   // [P][4] int64: ptr, da, in offsets, fits
    L.sa_ord = align_up(L.poff + (size_t)P * 4 * sizeof(long long), 16);   // stride-aware: [Wp] stream order
    L.sa_col = L.sa_ord + (sa ? (size_t)g.Wp * sizeof(int) : 0);            // [Wp] coverage | local column << 8
    L.sa_last = L.sa_col + (sa ? (size_t)g.Wp * sizeof(int) : 0);           // [types][O_w] last owned column
    L.total = align_up(L.sa_last + (sa ? (size_t)sa_ntypes_of(g) * g.Ow * sizeof(int) : 0), 16);
    return L;
}

// ---- stride-aware layout (reading A32, SI Eq. 2): partition s covers padded columns
// [s*s_w, s*s_w + K_w); coverage, owner (first covering partition), local column, type = cov - 1
__device__ __forceinline__ int sa_cov_e(const Geom& g, int w) {
    const int hi = min(g.Ow - 1, w / g.sw);
    const int lo = (w - g.S + 1 <= 0) ? 0 : (w - g.S + 1 + g.sw - 1) / g.sw;
    return max(0, hi - lo + 1);
}
__device__ __forceinline__ int sa_owner_e(const Geom& g, int w) {
    return (w - g.S + 1 <= 0) ? 0 : (w - g.S + 1 + g.sw - 1) / g.sw;
}
// ptr length of a stride-aware plane: per coverage type present in the geometry (ascending),
// a block [t+1, c_0 .. c_{O_w-1}] or [t+1, NPF]; NPC = one entry.  Columns w = l0, l0 + nl, ...
// of this thread; nl = 32: the warp's lanes split the columns (lane 0 gets the result)
__device__ __forceinline__ void sa_plane_lengths(const Geom& g, const int* wc, int td, unsigned types,
                                                 const int* sacol, int l0, int nl, int* pi) {
    int tot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int w = l0; w < g.Wp; w += nl) {
        const int cv = sacol[w] & 0xFF;
#pragma unroll
        for (int t = 0; t < 8; t++)
            if (t == cv - 1) tot[t] += wc[w];
    }
    if (nl == 32) {
#pragma unroll
        for (int t = 0; t < 8; t++)
            if ((types >> t) & 1u) tot[t] = warp_sum(tot[t]);
        if (l0 != 0) return;
    }
    int plen = 0;
#pragma unroll
    for (int t = 0; t < 8; t++)
        if ((types >> t) & 1u) plen += tot[t] ? (1 + g.Ow) : 2;
    pi[0] = td ? plen : 1;
    pi[1] = td;
    pi[2] = td;
    pi[3] = 0;
}

// ptr length (NPC | S=1 block | NOP + overlap blocks with NPF, SI Eq. 3), and the DA
// count below the overlapK_w block, of one plane with column counts wc and totals td, ti
__device__ __forceinline__ void plane_lengths(const Geom& g, const int* wc, int td, int ti, int* pi) {
    int plen, lower = 0;
    if (td == 0) {
        plen = 1;                                   // NPC
    } else if (g.S == 1) {
        plen = 1 + g.Ow1;
    } else {
        plen = (g.pl == 0) ? 3 : 0;                 // NOP block (reading A2)
        for (int t = max(1, g.pl); t <= g.S - 2; t++) {
            const int bn = wc[t] + wc[g.Wp - 1 - t];
            lower += bn;
            plen += bn ? (1 + g.Ow1) : 2;           // block or [tag, NPF] (reading A3)
        }
        if (g.pl == 0) lower += wc[0] + wc[g.Wp - 1];
        plen += (td - lower) ? (1 + g.Ow1) : 2;
    }
    pi[0] = plen; pi[1] = td; pi[2] = ti; pi[3] = lower;
}

template <bool CPS, bool SA>
__global__ void __launch_bounds__(kThreads, 2) encode_kernel(EncArgs a) {
    const Geom& g = a.g;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ long long s_red[kEncWarps][3];
    __shared__ long long s_tile_tot[3];
    __shared__ long long s_pre[3];
    __shared__ unsigned s_epoch;
    __shared__ int s_timeout;
    __shared__ __align__(8) unsigned long long s_bar[1];
    unsigned s_phase = 0;   // (per thread) parity of the staging barrier
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int HW = g.H * g.W, Wp = g.Wp, NW = g.nwords;

    probe(0);
    pdl_wait();      // x may come from the kernel before us
    probe(1);
    pdl_trigger();   // the dependent convolution may launch and stage its taps
    if (threadIdx.x == 0) {
        s_epoch = *reinterpret_cast<volatile unsigned*>(&a.st->epoch);
        s_timeout = 0;
        mbar_init(s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const EncSmem L = enc_smem_layout(g, a.P, SA);
    float* planes = reinterpret_cast<float*>(smem_raw + L.planes);
    unsigned* msk = reinterpret_cast<unsigned*>(smem_raw + L.msk);   // [P][Wp][NW]
    int* cnt = reinterpret_cast<int*>(smem_raw + L.cnt);             // [P][Wp]
    int* incnt = reinterpret_cast<int*>(smem_raw + L.incnt);
    int* dab = reinterpret_cast<int*>(smem_raw + L.dab);
    int* inb = reinterpret_cast<int*>(smem_raw + L.inb);
    unsigned* umask = reinterpret_cast<unsigned*>(smem_raw + L.umask);
    int4* tab = reinterpret_cast<int4*>(smem_raw + L.tab);
    const int NRB = (g.H + 31) / 32;
    int* pinfo = reinterpret_cast<int*>(smem_raw + L.pinfo);
    long long* poff = reinterpret_cast<long long*>(smem_raw + L.poff);
    int* sa_ord = reinterpret_cast<int*>(smem_raw + L.sa_ord);     // SA: padded column at stream position q
    int* sa_last = reinterpret_cast<int*>(smem_raw + L.sa_last);   // SA: [type][partition] last owned column
    int* sa_col = reinterpret_cast<int*>(smem_raw + L.sa_col);     // SA: coverage | local column << 8
    __shared__ unsigned s_types;                                   // SA: coverage types present (bit t = type t)
    if constexpr (SA) {
        // the layout's column order (types ascending, columns ascending inside a type; columns no
        // partition covers last -- they hold no stored NZE) and each partition's last owned column
        // of every type: geometry only, once per CTA
        if (threadIdx.x == 0) s_types = 0u;
        for (int w = threadIdx.x; w < Wp; w += kThreads) {
            const int cv = sa_cov_e(g, w);
            sa_col[w] = cv | ((w - sa_owner_e(g, w) * g.sw) << 8);
        }
        __syncthreads();
        for (int w = threadIdx.x; w < Wp; w += kThreads) {
            const int cv = sa_col[w] & 0xFF, key = cv ? cv : 1 << 20;
            int q = 0;
            for (int w2 = 0; w2 < Wp; w2++) {
                const int c2 = sa_col[w2] & 0xFF, k2 = c2 ? c2 : 1 << 20;
                q += (k2 < key) || (k2 == key && w2 < w);
            }
            sa_ord[q] = w;
            if (cv) atomicOr(&s_types, 1u << (cv - 1));
        }
        const int nt = sa_ntypes_of(g);
        for (int i = threadIdx.x; i < nt * g.Ow; i += kThreads) {
            const int t = i / g.Ow, s2 = i % g.Ow;
            int last = -1;
            for (int l = 0; l < g.S; l++) {
                const int w = s2 * g.sw + l;
                if (w < Wp && (sa_col[w] & 0xFF) == t + 1 && (sa_col[w] >> 8) == l) last = w;
            }
            sa_last[i] = last;
        }
        __syncthreads();
    }

    for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const long long plane0 = (long long)tile * a.P;
        const int np = (int)min((long long)a.P, g.NC - plane0);

        // ---- 1. stage the tile's planes with TMA bulk copies (one elected thread, the whole
        //         tile in flight) from the 16-byte aligned element a0 <= e0; the < 16-byte tail
        //         with plain loads (x is 16-byte aligned)
        const long long e0 = plane0 * HW, e1 = e0 + (long long)np * HW;
        const long long a0 = e0 & ~3ll;
        const int sh = (int)(e0 - a0);
        {
            const long long n4 = (e1 - a0) >> 2;        // whole 16-byte vectors
            if (threadIdx.x == 0) {
                const unsigned bytes = (unsigned)(n4 * 16);
                mbar_expect_tx(s_bar, bytes);
                const char* src = reinterpret_cast<const char*>(a.x + a0);
                char* dst = reinterpret_cast<char*>(planes);
                for (unsigned off = 0; off < bytes; off += kBulkChunk)
                    bulk_g2s(dst + off, src + off, min(kBulkChunk, bytes - off), s_bar);
            }
            for (long long i = a0 + 4 * n4 + threadIdx.x; i < e1; i += kThreads) planes[i - a0] = __ldg(a.x + i);
            mbar_wait(s_bar, s_phase);
            s_phase ^= 1u;
        }
        __syncthreads();
        probe(2);
        const float* pl0 = planes + sh;

        // ---- 2. unpadded column bitmasks by warp ballots + a 32x32 bit transpose:
        //         block = (plane group, 32-row block, 32-column block); for W <= 32 one
        //         warp covers G = 32/W planes (lane l -> plane l/W, column l%W)
        {
            const int G = (g.W <= 32) ? (32 / g.W) : 1;
            const int CBW = (g.W <= 32) ? g.W : 32;            // columns per lane group
            const int NCB = (g.W + 31) / 32;
            const int npg = (np + G - 1) / G;
            const int p_l = lane / CBW, c_l = lane % CBW;
            for (int blk = warp; blk < npg * NRB * NCB; blk += kEncWarps) {
                const int cb = blk % NCB, rb = (blk / NCB) % NRB, pg = blk / (NCB * NRB);
                const int p = pg * G + p_l, col = cb * 32 + c_l;
                const bool ok = (lane < G * CBW) && (p < np) && (col < g.W);
                const float* src = pl0 + (size_t)(ok ? p : 0) * HW + (ok ? col : 0);
                unsigned x = 0;
#pragma unroll
                for (int r0 = 0; r0 < 32; r0 += 8) {
                    float v[8];
#pragma unroll
                    for (int u = 0; u < 8; u++)      // unconditional (clamped) loads, all in flight
                        v[u] = src[min(rb * 32 + r0 + u, g.H - 1) * g.W];
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        const bool nz = ok && (rb * 32 + r0 + u < g.H) && (v[u] != 0.0f);
                        const unsigned b = __ballot_sync(0xffffffffu, nz);
                        x = (lane == r0 + u) ? b : x;
                    }
                }
                // lane r holds row r (bit l = lane-column l); transpose -> lane l holds column l
#pragma unroll
                for (int sft = 16; sft >= 1; sft >>= 1) {
                    const unsigned M = (sft == 16) ? 0x0000FFFFu : (sft == 8) ? 0x00FF00FFu
                                     : (sft == 4) ? 0x0F0F0F0Fu : (sft == 2) ? 0x33333333u : 0x55555555u;
                    const unsigned y = __shfl_xor_sync(0xffffffffu, x, sft);
                    x = (lane & sft) ? ((x & ~M) | ((y & ~M) >> sft)) : ((x & M) | ((y & M) << sft));
                }
                if (ok) umask[((size_t)p * g.W + col) * NRB + rb] = x;
            }
        }
        __syncthreads();
        probe(3);
        // ---- 3. padded masks (shift by pad_top), per-column NZE count and IN entries
        //         (CPS set4 packing in overlapK_w)
        for (int it = threadIdx.x; it < np * Wp; it += kThreads) {
            const int w = it % Wp, p = it / Wp;
            const int col = w - g.pl;
            const bool real = col >= 0 && col < g.W;
            const unsigned* u = umask + ((size_t)p * g.W + (real ? col : 0)) * NRB;
            int c = 0, e = 0;
            const bool mid = CPS && is_middle(g, w);
            const bool stored = !SA || (sa_col[w] & 0xFF) > 0;   // SA: columns no partition covers are not stored
            unsigned prev = 0;
            for (int j = 0; j < NW; j++) {
                const unsigned uj = (real && j < NRB) ? u[j] : 0u;
                const unsigned m = g.pt ? ((uj << g.pt) | (prev >> (32 - g.pt))) : uj;
                prev = uj;
                msk[it * NW + j] = m;
                c += stored ? __popc(m) : 0;
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
        // ---- 4. per plane: stream-order exclusive prefix over columns, plane totals and
        //         the ptr length (SI Eq. 3 with the actual NPF count); thread per plane for
        //         narrow planes, warp per plane otherwise
        // (thread per plane only when the tile has more planes than warps: a few planes of a
        //  narrow map are scanned faster by a warp each -- cfg3: 7 planes of Wp = 16)
        static_assert(kEncWarps >= 8, "");
#ifndef SPC_ENC_THREAD_SCAN
        if (Wp <= 24 && np > kEncWarps) {
#else
        if (Wp <= 24) {
#endif
            for (int p = threadIdx.x; p < np; p += kThreads) {
                const int* wc = cnt + p * Wp;
                const int* wi = incnt + p * Wp;
                int ed = 0, ei = 0;
                for (int q = 0; q < Wp; q++) {
                    const int w = SA ? sa_ord[q] : col_at(g, q);
                    dab[p * Wp + w] = ed;
                    inb[p * Wp + w] = ei;
                    ed += wc[w];
                    ei += wi[w];
                }
                if (SA) sa_plane_lengths(g, wc, ed, s_types, sa_col, 0, 1, pinfo + 4 * p);
                else plane_lengths(g, wc, ed, ei, pinfo + 4 * p);
            }
        } else {
            for (int p = warp; p < np; p += kEncWarps) {
                const int* wc = cnt + p * Wp;
                const int* wi = incnt + p * Wp;
                const int per = (Wp + 31) / 32;
                const int q0 = lane * per, q1 = min(q0 + per, Wp);
                int sd = 0, si = 0;
                for (int q = q0; q < q1; q++) {
                    const int w = SA ? sa_ord[q] : col_at(g, q);
                    sd += wc[w];
                    si += wi[w];
                }
                int td, ti;
                int ed = warp_exclusive_scan(sd, &td);
                int ei = warp_exclusive_scan(si, &ti);
                for (int q = q0; q < q1; q++) {
                    const int w = SA ? sa_ord[q] : col_at(g, q);
                    dab[p * Wp + w] = ed;
                    inb[p * Wp + w] = ei;
                    ed += wc[w];
                    ei += wi[w];
                }
                if (SA) sa_plane_lengths(g, wc, td, s_types, sa_col, lane, 32, pinfo + 4 * p);
                else if (lane == 0) plane_lengths(g, wc, td, ti, pinfo + 4 * p);
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
        // ---- 6. publish the tile aggregate (tagged words + a per-launch counter),
        //         wait for every tile of this round, prefix = sum over ALL preceding tiles
        const unsigned long long tag = (unsigned long long)((s_epoch + 1u) & 0xFFFFFFu);
        unsigned* counter = &a.st->count[s_epoch & 1u];
        if (threadIdx.x == 0) {
#pragma unroll
            for (int i = 0; i < 3; i++)
                st_relaxed64(a.agg + 3ll * tile + i, (tag << kTagShift) | (unsigned long long)s_tile_tot[i]);
            red_release_add(counter, 1u);
            if (!a.multi_round) {
                const unsigned target = (unsigned)min(a.ntiles, (tile / (int)gridDim.x + 1) * (int)gridDim.x);
                long long spin = 0;
                while (ld_acquire_u32(counter) < target) {
                    __nanosleep(32);
                    if (++spin > kSpinLimit) { s_timeout = 1; break; }   // bounded: never hang the GPU
                }
            }
        }
        __syncthreads();
        {
            long long p0 = 0, p1 = 0, p2 = 0;
            for (long long i = threadIdx.x; i < 3ll * tile; i += kThreads) {
                unsigned long long v;
                long long spin = 0;
                while (((v = ld_relaxed64(a.agg + i)) >> kTagShift) != tag) {
                    if (a.multi_round) __nanosleep(64);
                    if (++spin > kSpinLimit) { s_timeout = 1; break; }
                }
                const long long val = (long long)(v & kValMask);
                const int sidx = (int)(i % 3);
                p0 += (sidx == 0) ? val : 0;
                p1 += (sidx == 1) ? val : 0;
                p2 += (sidx == 2) ? val : 0;
            }
            p0 = warp_sum(p0); p1 = warp_sum(p1); p2 = warp_sum(p2);
            if (lane == 0) { s_red[warp][0] = p0; s_red[warp][1] = p1; s_red[warp][2] = p2; }
        }
        __syncthreads();
        if (s_timeout) {
            // a predecessor never published (cannot happen with a co-resident grid): report it in
            // the overflow word (bit 1, sticky) and leave; waiters on this tile time out as well
            if (threadIdx.x == 0) atomicOr(reinterpret_cast<unsigned long long*>(a.lengths + 3), 2ull);
            return;
        }
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
            // the whole word: bit 0 = capacity overflow of this launch (a launch that completes
            // here had every predecessor publish, so no wait of it timed out)
            a.lengths[3] = (t0 > a.cap_ptr || t1 > a.cap_da || t2 > a.cap_in) ? 1 : 0;
            a.st->count[(s_epoch + 1u) & 1u] = 0;   // the next launch's counter (unused in this one)
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
        // per-column table for the DA/IN pass: tile-relative DA / IN offsets of the column,
        // smem index of its padded row 0, local column L and flags (no divisions later)
        for (int it = threadIdx.x; it < np * Wp; it += kThreads) {
            const int p = it / Wp, w = it % Wp;
            const bool ok = poff[4 * p + 3] && cnt[it] > 0;
            const bool wr_in = !(CPS && is_middle(g, w));
            tab[it] = make_int4((int)(poff[4 * p + 1] - Z0) + dab[it], (int)(poff[4 * p + 2] - Q0) + inb[it],
                                p * HW + (w - g.pl) - g.pt * g.W,
                                (SA ? sa_col[w] >> 8 : local_of(g, w)) | (wr_in ? kTabIn : 0) |
                                    (ok ? kTabOk : 0));
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
            } else if (SA) {
                // stride-aware blocks (reading A32): per type present, [t+1, c_0 .. c_{O_w-1}] with
                // c_s = block-relative cumulative count through partition s's last owned type-t
                // column (-1: owns none), or [t+1, NPF]
                const int* wd = dab + p * Wp;
                int pos = 0, run = 0;
                for (int t = 0; t < sa_ntypes_of(g); t++) {
                    if (!((s_types >> t) & 1u)) continue;
                    long long tl = 0;
                    for (int w = lane; w < Wp; w += 32) tl += ((sa_col[w] & 0xFF) == t + 1) ? wc[w] : 0;
                    const int tt = (int)warp_sum(tl);
                    if (lane == 0) pp[pos] = t + 1;
                    if (tt == 0) {
                        if (lane == 0) pp[pos + 1] = SPC_NPF;
                        pos += 2;
                        continue;
                    }
                    for (int s2 = lane; s2 < g.Ow; s2 += 32) {
                        const int last = sa_last[t * g.Ow + s2];
                        pp[pos + 1 + s2] = (last < 0) ? -1 : wd[last] + wc[last] - run;
                    }
                    run += tt;
                    pos += 1 + g.Ow;
                }
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
        // ---- 7b. DA (and CPO-form IN): lanes = rows of a column word; the rank of an NZE
        //          is a popc of the mask below its lane (coalesced stores).  Short columns
        //          (one word, Hp <= 16) pack 32/Hp columns into a warp pass.
        {
            float* dT = a.da + Z0;
            int32_t* iT = a.in + Q0;
            const int nit = np * Wp;
            if (NW == 1 && g.Hp <= 16) {
                const int CPW = 32 / g.Hp;
                const int sub = lane / g.Hp, row = lane - sub * g.Hp;
                for (int it0 = warp * CPW; it0 < nit; it0 += kEncWarps * CPW) {
                    const int it = it0 + sub;
                    const unsigned m = (sub < CPW && it < nit) ? msk[it] : 0u;
                    if ((m >> row) & 1u) {
                        const int4 t = tab[it];
                        if (t.w & kTabOk) {
                            const int r = __popc(m & ((1u << row) - 1u));
                            dT[t.x + r] = pl0[t.z + row * g.W];
                            if (t.w & kTabIn) iT[t.y + r] = (t.w & 0xFFFF) + row * g.S;
                        }
                    }
                }
            } else if (NW <= 2 && (g.W & 7) == 4) {
                // W = 4 x odd (28, 12, 20, ...): lanes = 4 column items x 8 rows, so the plane
                // reads hit 32 distinct banks instead of 8 (4-way with lanes = 32 rows of one
                // column); each lane ranks its NZE in its own column (popc below its row) and the
                // stores form 4 short runs.  Measured: cfg5-L7 82 -> 71 us, batch-256 L4 203 ->
                // 176 us; at W = 56 (2-way here vs 8-way) it was slower (34 -> 37 us), so W = 8k
                // keeps the row-lane pass below.
                const int cu = lane >> 3, hr = lane & 7;
                for (int it0 = 4 * warp; it0 < nit; it0 += 4 * kEncWarps) {
                    const int it = it0 + cu;
                    const bool v = it < nit;
                    const int4 t = v ? tab[it] : make_int4(0, 0, 0, 0);
                    const unsigned m0 = v ? msk[it * NW] : 0u;
                    const unsigned m1 = (v && NW == 2) ? msk[it * NW + 1] : 0u;
                    if (!__any_sync(0xffffffffu, (t.w & kTabOk) != 0)) continue;
                    const bool ok = (t.w & kTabOk) != 0;
                    const int c0 = __popc(m0);
                    const int Lc = t.w & 0xFFFF;
                    const bool win = (t.w & kTabIn) != 0;
#pragma unroll
                    for (int rb = 0; rb < 64; rb += 8) {
                        const int h = rb + hr;                 // padded row
                        if (rb >= g.Hp) break;
                        const unsigned word = (h < 32) ? m0 : m1;
                        const bool b = ok && h < g.Hp && ((word >> (h & 31)) & 1u);
                        const int r = (h < 32) ? __popc(m0 & ((1u << h) - 1u))
                                               : c0 + __popc(m1 & ((1u << (h - 32)) - 1u));
                        const int hc = min(max(h, g.pt), g.pt + g.H - 1);   // clamped: unconditional load
                        const float val = pl0[t.z + hc * g.W];
                        if (b) {
                            dT[t.x + r] = val;
                            if (win) iT[t.y + r] = Lc + h * g.S;
                        }
                    }
                }
            } else if (NW <= 2) {
                // two column items per warp iteration: table and mask loads of both in flight
                for (int it0 = 2 * warp; it0 < nit; it0 += 2 * kEncWarps) {
                    int4 t[2];
                    unsigned m[2][2];
#pragma unroll
                    for (int u = 0; u < 2; u++) {
                        const bool v = it0 + u < nit;
                        t[u] = v ? tab[it0 + u] : make_int4(0, 0, 0, 0);
                        m[u][0] = v ? msk[(it0 + u) * NW] : 0u;
                        m[u][1] = (v && NW == 2) ? msk[(it0 + u) * NW + 1] : 0u;
                    }
#pragma unroll
                    for (int u = 0; u < 2; u++) {
                        if (!(t[u].w & kTabOk)) continue;
                        const int c0 = __popc(m[u][0]);
                        const bool b0 = (m[u][0] >> lane) & 1u, b1 = (m[u][1] >> lane) & 1u;
                        const int r0 = __popc(m[u][0] & lanemask_lt());
                        const int r1 = c0 + __popc(m[u][1] & lanemask_lt());
                        // unconditional loads at rows clamped into the real (unpadded) plane
                        const int hc0 = min(max(lane, g.pt), g.pt + g.H - 1);
                        const int hc1 = min(max(32 + lane, g.pt), g.pt + g.H - 1);
                        const float v0 = pl0[t[u].z + hc0 * g.W];
                        const float v1 = pl0[t[u].z + hc1 * g.W];
                        if (b0) dT[t[u].x + r0] = v0;
                        if (b1) dT[t[u].x + r1] = v1;
                        if (t[u].w & kTabIn) {
                            const int Lc = t[u].w & 0xFFFF;
                            if (b0) iT[t[u].y + r0] = Lc + lane * g.S;
                            if (b1) iT[t[u].y + r1] = Lc + (32 + lane) * g.S;
                        }
                    }
                }
            } else {
                for (int it = warp; it < nit; it += kEncWarps) {
                    const int4 t = tab[it];
                    if (!(t.w & kTabOk)) continue;
                    int base = 0;
                    for (int j = 0; j < NW; j++) {
                        const unsigned m = msk[it * NW + j];
                        if ((m >> lane) & 1u) {
                            const int r = base + __popc(m & lanemask_lt());
                            const int h = 32 * j + lane;
                            dT[t.x + r] = pl0[t.z + h * g.W];
                            if (t.w & kTabIn) iT[t.y + r] = (t.w & 0xFFFF) + h * g.S;
                        }
                        base += __popc(m);
                    }
                }
            }
        }
        // ---- 7c. CPS IN of the overlapK_w columns: lane per set4 group, G lanes per column
        //          (G = 8 / 16 / 32 by the padded height: short columns share a warp)
        if (CPS) {
            const int NG = 8 * NW;                          // set4 groups per padded column
            const int G = (NG <= 8) ? 8 : (NG <= 16) ? 16 : 32;
            const int CPW = 32 / G, sub = lane / G, sl = lane % G;
            for (int it0 = warp * CPW; it0 < np * Wp; it0 += kEncWarps * CPW) {
                const int it = it0 + sub;
                const int p = it / Wp, w = it % Wp;
                const bool act = it < np * Wp && is_middle(g, w) && cnt[it] != 0 && poff[4 * p + 3];
                const int L = act ? local_of(g, w) : 0;
                int32_t* ii = act ? a.in + poff[4 * p + 2] + inb[it] : nullptr;
                const unsigned* mw = msk + (act ? it : 0) * NW;
                int irun = 0;
                for (int g0 = 0; g0 < NG; g0 += G) {
                    const int grp = g0 + sl;                // rows 4*grp .. 4*grp+3
                    unsigned nib = 0;
                    if (act && grp < NG) nib = (mw[grp >> 3] >> (4 * (grp & 7))) & 0xFu;
                    const int k = __popc(nib);
                    const int e = k >= 3 ? 2 : k;
                    int inc = e;                            // scan inside the column's G lanes
                    for (int o = 1; o < G; o <<= 1) {
                        const int t = __shfl_up_sync(0xffffffffu, inc, o, G);
                        if (sl >= o) inc += t;
                    }
                    const int te = __shfl_sync(0xffffffffu, inc, G - 1, G);
                    if (k) {
                        const int row0 = 4 * grp;
                        int32_t* o = ii + irun + (inc - e);
                        if (k >= 3) {
                            o[0] = L + (row0 + __ffs(nib) - 1) * g.S;  // first NZE index (A9)
                            o[1] = (int32_t)nib;                         // pattern, bit b = row b (A12)
                        } else {
                            int u = 0;
                            for (int bb = 0; bb < 4; bb++)
                                if ((nib >> bb) & 1u) o[u++] = -(L + (row0 + bb) * g.S);
                        }
                    }
                    irun += te;
                }
            }
        }
        probe(10);
        fence_proxy_async();   // generic-proxy reads of this tile before the next bulk copy
        __syncthreads();       // the next tile reuses the shared memory
        probe(11);
    }
}

struct EncPlan {
    int P, ntiles, grid;
    size_t smem;
};

int sm_count() { return device_sm_count(); }

// Tile size: prefer 2 resident CTAs per SM (tiles within ~110 KB of smem), else 1; take
// the fewest rounds that largest tile allows, then the smallest P that still needs only
// that many rounds, so every round is (nearly) full.  Measured: cfg5-L7 (batch 32) 71 -> 50 us
// (a 51-plane tile at 1 CTA/SM had left a 13-tile second round), batch 256 L4 176 -> 147 us,
// L14 137 -> 102 us; one-round launches are unchanged (cfg2: P = 1, cfg5-L0: P = 7).
EncPlan plan_encode(const Geom& g, bool sa = false) {
    EncPlan pl;
    const int sms = sm_count();
    const size_t b2 = 110 * 1024, b1 = 220 * 1024;
    long long P = 0;
    for (int per_sm = 2; per_sm >= 1 && P == 0; per_sm--) {
        const size_t budget = (per_sm == 2) ? b2 : b1;
        long long pmax = 0;
        while (pmax < g.NC && enc_smem_layout(g, (int)(pmax + 1), sa).total <= budget) pmax++;
        if (pmax == 0) continue;
        const long long slots = (long long)per_sm * sms;
        const long long rounds = (g.NC + slots * pmax - 1) / (slots * pmax);
        P = (g.NC + slots * rounds - 1) / (slots * rounds);
    }
    static const int force_p = [] { const char* v = getenv("SPC_ENC_P"); return v ? atoi(v) : 0; }();
    if (force_p > 0 && enc_smem_layout(g, force_p, sa).total <= b1) P = force_p;   // development A/B
    pl.P = (int)std::max(1ll, P);
    pl.ntiles = (int)((g.NC + pl.P - 1) / pl.P);
    pl.smem = enc_smem_layout(g, pl.P, sa).total;
    pl.grid = pl.ntiles;
    return pl;
}

}  // namespace

size_t enc_smem_bytes(const Geom& g) { return plan_encode(g).smem; }

cudaError_t launch_encode(const Geom& g, bool cps, const float* x, spc_encoding* e, void* ws, cudaStream_t st,
                          bool sa) {
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
    EncPlan pl = plan_encode(g, sa);
    a.P = pl.P;
    a.ntiles = pl.ntiles;
    void (*kern)(EncArgs) = sa ? encode_kernel<false, true> : cps ? encode_kernel<true, false> : encode_kernel<false, false>;
    static std::atomic<size_t> attr_bytes[3][kMaxDevices];
    {
        cudaError_t err = ensure_smem_attr((const void*)kern, pl.smem, attr_bytes[sa ? 2 : cps ? 1 : 0]);
        if (err != cudaSuccess) return err;
    }
    // the cross-tile prefix needs every CTA resident: cap the grid at the
    // occupancy limit (CTAs then loop over tiles in increasing order) and launch cooperatively
    int occ = 0;
    cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, pl.smem);
    if (err != cudaSuccess) return err;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const int grid = std::min(pl.ntiles, occ * sm_count());
    a.multi_round = pl.ntiles > grid;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = st;
    // cooperative: the driver co-schedules every CTA of the grid (the cross-tile prefix waits
    // on other CTAs), even when kernels on other streams hold SMs
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cooperative_launches() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace spc

#ifdef SPC_PROBES
SPC_PROBE_ACCESSOR(spc_debug_probes_enc)
#endif
