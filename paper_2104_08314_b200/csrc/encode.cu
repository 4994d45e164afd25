// encode.cu -- single-pass CPO / CPS encoder for sm_100a.
//
// What it computes: the canonical CPO streams of Alg. 1 (
// SI Alg. 5 for K_w = 1) or the CPS streams of Alg. 3
// (PAPER.md:316-372), channels concatenated n-major then c (reading A19),
// plus the per-channel exclusive offsets (GPU side tables).
//
// How (B200 design, not the paper's serial loop):
//  * one CTA (8 warps) = G consecutive channel planes (contiguous in NCHW),
//    WPP = 8/G warps per plane; the planes are staged into shared memory with
//    coalesced 128-bit loads;
//  * per padded column a 32-bit row bitmask per 32-row word -> popc column
//    counts; NPF / NPC come from block / channel sums (Alg. 1 lines 31-37);
//  * CPS set4 patterns are the 4-bit nibbles of the column masks (groups
//    anchored at padded row 0): popc decides {index, pattern} vs negated;
//  * stream offsets: scans inside the CTA and a decoupled look-back across
//    CTAs (ticket-ordered), so the whole tensor is encoded in ONE launch that
//    reads x once and writes each stream once;
//  * DA/IN are written column by column with ballot/popc compaction, the
//    plane's warps splitting the columns.
#include "common.cuh"

namespace spc {
namespace {

constexpr int kFlagAgg = 1, kFlagInc = 2;
constexpr int kThreads = kEncWarps * 32;

struct EncArgs {
    Geom g;
    const float* __restrict__ x;
    int32_t* ptr; float* da; int32_t* in;
    int64_t* chan_ptr_off; int64_t* chan_nz_off; int64_t* chan_in_off;
    int64_t* lengths;
    int64_t cap_ptr, cap_da, cap_in;
    EncState* st; int* flags; long long* agg; long long* inc;
    int ntiles;
    int G;      // planes per CTA
    int WPP;    // warps per plane
};

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

// named barrier over the WPP warps of one plane (ids 1..8)
__device__ __forceinline__ void plane_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <bool CPS>
__global__ void __launch_bounds__(kThreads) encode_kernel(EncArgs a) {
    const Geom& g = a.g;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int HW = g.H * g.W, G = a.G, WPP = a.WPP;
    const int pi = warp / WPP;            // plane of this warp inside the CTA
    const int sub = warp % WPP;           // warp index inside the plane's group
    const int gt = sub * 32 + lane;       // thread index inside the group
    const int GT = WPP * 32;              // threads per group

    __shared__ int s_tile;
    __shared__ long long s_len[kEncWarps][3];
    __shared__ long long s_prefix[3];
    __shared__ int s_blk_lower[kEncWarps];
    float* planes = reinterpret_cast<float*>(smem_raw);                        // [G][H*W]
    size_t off = align_up((size_t)G * HW * sizeof(float), 16);
    unsigned* masks = reinterpret_cast<unsigned*>(smem_raw + off);             // [G][Wp*nwords]
    off += (size_t)G * g.Wp * g.nwords * sizeof(unsigned);
    int* cnt = reinterpret_cast<int*>(smem_raw + off);                         // [G][Wp]
    int* incnt = cnt + G * g.Wp;
    int* dabase = incnt + G * g.Wp;
    int* inbase = dabase + G * g.Wp;

    if (threadIdx.x == 0) s_tile = atomicAdd(&a.st->ticket, 1);
    __syncthreads();
    const int tile = s_tile;
    const long long plane0 = (long long)tile * G;
    const int nplanes = (int)min((long long)G, g.NC - plane0);

    // ---- 1. stage the CTA's contiguous planes (coalesced 128-bit loads)
    {
        const long long n_el = (long long)nplanes * HW;
        const float* src = a.x + plane0 * HW;
        const bool al = ((reinterpret_cast<uintptr_t>(src) & 15u) == 0);
        const long long n4 = al ? (n_el >> 2) : 0;
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(planes);
        for (long long i = threadIdx.x; i < n4; i += kThreads) d4[i] = __ldg(s4 + i);
        for (long long i = (n4 << 2) + threadIdx.x; i < n_el; i += kThreads) planes[i] = __ldg(src + i);
    }
    __syncthreads();

    const bool active = pi < nplanes;
    const float* pl = planes + (size_t)pi * HW;
    unsigned* msk = masks + (size_t)pi * g.Wp * g.nwords;
    int* wcnt = cnt + pi * g.Wp;
    int* wincnt = incnt + pi * g.Wp;
    int* wdab = dabase + pi * g.Wp;
    int* winb = inbase + pi * g.Wp;

    if (active) {
        // ---- 2. column bitmasks in the padded frame: item = (column, 32-row word)
        for (int it = gt; it < g.Wp * g.nwords; it += GT) {
            const int w = it / g.nwords, j = it % g.nwords;
            const int wu = w - g.pl;
            unsigned m = 0;
            if (wu >= 0 && wu < g.W) {
                const int h0 = 32 * j - g.pt;
                const int b0 = max(0, -h0), b1 = min(32, g.H - h0);
#pragma unroll 8
                for (int b = b0; b < b1; b++) m |= (unsigned)(pl[(h0 + b) * g.W + wu] != 0.0f) << b;
            }
            msk[it] = m;
        }
        plane_sync(1 + pi, GT);
        // ---- 3. per column: NZE count and IN entries (CPS set4 packing in overlapK_w)
        for (int w = gt; w < g.Wp; w += GT) {
            int c = 0, e = 0;
            const bool mid = CPS && is_middle(g, w);
            for (int j = 0; j < g.nwords; j++) {
                const unsigned m = msk[w * g.nwords + j];
                c += __popc(m);
                if (mid) {
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const int k = __popc((m >> (4 * q)) & 0xFu);
                        e += k >= 3 ? 2 : k;   // {index, pattern} or k negated indices
                    }
                }
            }
            wcnt[w] = c;
            wincnt[w] = mid ? e : c;
        }
        plane_sync(1 + pi, GT);
        // ---- 4. stream-order exclusive prefix (first warp of the group)
        if (sub == 0) {
            const int per = (g.Wp + 31) / 32;
            const int p0 = lane * per;
            int sd = 0, si = 0;
            for (int p = p0; p < min(p0 + per, g.Wp); p++) {
                const int w = col_at(g, p);
                sd += wcnt[w];
                si += wincnt[w];
            }
            int td, ti;
            int ed = warp_exclusive_scan(sd, &td);
            int ei = warp_exclusive_scan(si, &ti);
            for (int p = p0; p < min(p0 + per, g.Wp); p++) {
                const int w = col_at(g, p);
                wdab[w] = ed; winb[w] = ei;
                ed += wcnt[w]; ei += wincnt[w];
            }
            if (lane == 0) {
                // ptr length: NPC | S=1 block | NOP + overlap blocks with NPF (SI Eq. 3)
                long long plen;
                int lower = 0;
                if (td == 0) {
                    plen = 1;
                } else if (g.S == 1) {
                    plen = 1 + g.Ow1;
                } else {
                    plen = (g.pl == 0) ? 3 : 0;
                    for (int t = max(1, g.pl); t <= g.S - 2; t++) {
                        const int bn = wcnt[t] + wcnt[g.Wp - 1 - t];
                        lower += bn;
                        plen += bn ? (1 + g.Ow1) : 2;
                    }
                    if (g.pl == 0) lower += wcnt[0] + wcnt[g.Wp - 1];
                    plen += (td - lower) ? (1 + g.Ow1) : 2;
                }
                s_len[pi][0] = plen;
                s_len[pi][1] = td;
                s_len[pi][2] = ti;
                s_blk_lower[pi] = lower;
            }
        }
    } else if (sub == 0 && lane == 0) {
        s_len[pi][0] = s_len[pi][1] = s_len[pi][2] = 0;
    }
    __syncthreads();

    // ---- 5. decoupled look-back across tiles (warp 0)
    if (warp == 0) {
        long long aggv[3] = {0, 0, 0};
        for (int p = 0; p < G; p++)
            for (int i = 0; i < 3; i++) aggv[i] += s_len[p][i];
        long long pre[3] = {0, 0, 0};
        if (tile == 0) {
            if (lane == 0) {
                for (int i = 0; i < 3; i++) a.inc[i] = aggv[i];
                __threadfence();
                st_release(&a.flags[0], kFlagInc);
            }
        } else {
            if (lane == 0) {
                for (int i = 0; i < 3; i++) a.agg[3 * (long long)tile + i] = aggv[i];
                __threadfence();
                st_release(&a.flags[tile], kFlagAgg);
            }
            int j = tile - 1;  // nearest predecessor inspected by lane 0
            long long spin = 0;
            while (true) {
                const int idx = j - lane;
                const int f = (idx >= 0) ? ld_acquire(&a.flags[idx]) : kFlagInc;
                const unsigned incm = __ballot_sync(0xffffffffu, f == kFlagInc);
                const int first = incm ? (__ffs(incm) - 1) : 32;  // nearest tile with inclusive prefix
                const unsigned below = (first == 32) ? 0xffffffffu : ((1u << first) - 1u);
                if (__ballot_sync(0xffffffffu, f == 0) & below) {
                    if (++spin > (1ll << 22)) __trap();  // bounded spin: never hang the GPU
                    continue;
                }
                long long v[3] = {0, 0, 0};
                if (idx >= 0 && lane <= first) {
                    const long long* src = (lane == first) ? (a.inc + 3 * (long long)idx) : (a.agg + 3 * (long long)idx);
                    for (int i = 0; i < 3; i++) v[i] = __ldcg(src + i);
                }
                for (int i = 0; i < 3; i++) pre[i] += warp_sum(v[i]);
                if (first < 32) break;
                j -= 32;
            }
            if (lane == 0) {
                for (int i = 0; i < 3; i++) a.inc[3 * (long long)tile + i] = pre[i] + aggv[i];
                __threadfence();
                st_release(&a.flags[tile], kFlagInc);
            }
        }
        if (lane == 0) {
            for (int i = 0; i < 3; i++) s_prefix[i] = pre[i];
            if (tile == a.ntiles - 1) {
                long long tot[3];
                for (int i = 0; i < 3; i++) tot[i] = pre[i] + aggv[i];
                a.chan_ptr_off[g.NC] = tot[0];
                a.chan_nz_off[g.NC] = tot[1];
                a.chan_in_off[g.NC] = tot[2];
                a.lengths[0] = tot[0];
                a.lengths[1] = tot[1];
                a.lengths[2] = tot[2];
                a.lengths[3] = (tot[0] > a.cap_ptr || tot[1] > a.cap_da || tot[2] > a.cap_in) ? 1 : 0;
            }
        }
    }
    __syncthreads();

    // ---- 6. write this plane's channel segment
    if (active) {
        long long P = s_prefix[0], Z = s_prefix[1], Q = s_prefix[2];
        for (int i = 0; i < pi; i++) {
            P += s_len[i][0]; Z += s_len[i][1]; Q += s_len[i][2];
        }
        const long long my_ptr = s_len[pi][0], nnz = s_len[pi][1], my_in = s_len[pi][2];
        const long long nc = plane0 + pi;
        if (gt == 0) {
            a.chan_ptr_off[nc] = P;
            a.chan_nz_off[nc] = Z;
            a.chan_in_off[nc] = Q;
        }
        const bool fits = (P + my_ptr <= a.cap_ptr) && (Z + nnz <= a.cap_da) && (Q + my_in <= a.cap_in);
        if (fits) {
            int32_t* pp = a.ptr + P;
            if (nnz == 0) {
                if (gt == 0) pp[0] = SPC_NPC;
            } else if (g.S == 1) {
                if (gt == 0) pp[0] = 0;
                for (int s = gt; s < g.Ow1; s += GT) pp[1 + s] = wdab[s] + wcnt[s];
            } else {
                int q = 0;
                if (g.pl == 0) {
                    if (gt == 0) {
                        pp[0] = 0;
                        pp[1] = wcnt[0];
                        pp[2] = wcnt[0] + wcnt[g.Wp - 1];
                    }
                    q = 3;
                }
                for (int t = max(1, g.pl); t <= g.S - 2; t++) {
                    const int bn = wcnt[t] + wcnt[g.Wp - 1 - t];
                    if (bn == 0) {
                        if (gt == 0) { pp[q] = t + 1; pp[q + 1] = SPC_NPF; }
                        q += 2;
                    } else {
                        if (gt == 0) pp[q] = t + 1;
                        for (int s = gt; s < g.Ow1; s += GT)
                            pp[q + 1 + s] = (s == 0) ? wcnt[t] : (s == g.Ow1 - 1 - t ? bn : -1);
                        q += 1 + g.Ow1;
                    }
                }
                const int bn = (int)nnz - s_blk_lower[pi];
                if (bn == 0) {
                    if (gt == 0) { pp[q] = g.S; pp[q + 1] = SPC_NPF; }
                } else {
                    if (gt == 0) pp[q] = g.S;
                    const int base = wdab[g.S - 1];
                    for (int s = gt; s < g.Ow1; s += GT)
                        pp[q + 1 + s] = (s <= g.Ow1 - g.S) ? (wdab[s + g.S - 1] + wcnt[s + g.S - 1] - base) : -1;
                }
            }
            // DA / IN: column by column (G of Alg. 1), the group's warps split the columns
            float* dd = a.da + Z;
            int32_t* ii = a.in + Q;
            for (int w = sub; w < g.Wp; w += WPP) {
                if (wcnt[w] == 0) continue;
                const int L = local_of(g, w);
                const int wu = w - g.pl;
                const int db = wdab[w], ib = winb[w];
                const bool mid = CPS && is_middle(g, w);
                int run = 0, irun = 0;
                for (int j = 0; j < g.nwords; j++) {
                    const unsigned m = msk[w * g.nwords + j];
                    if (m == 0) continue;
                    const int h = 32 * j + lane;
                    if ((m >> lane) & 1u) {
                        const int r = run + __popc(m & lanemask_lt());
                        dd[db + r] = pl[(h - g.pt) * g.W + wu];
                        if (!mid) ii[ib + r] = L + h * g.S;
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
                            int32_t* o = ii + ib + irun + eo;
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
        }
    }

    // ---- 7. the last CTA to finish resets the look-back state for the next launch
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int prev = atomicAdd(&a.st->done, 1);
        s_tile = (prev == (int)gridDim.x - 1) ? -1 : 0;
    }
    __syncthreads();
    if (s_tile == -1) {
        for (int i = threadIdx.x; i < a.ntiles; i += kThreads) a.flags[i] = 0;
        if (threadIdx.x == 0) {
            a.st->ticket = 0;
            a.st->done = 0;
        }
    }
}

}  // namespace

// planes per CTA: small planes share a CTA, large planes get all 8 warps
int enc_planes_per_cta(const Geom& g) {
    const long long hw = (long long)g.H * g.W;
    if (hw >= 2048) return 1;
    if (hw >= 1024) return 2;
    if (hw >= 256) return 4;
    return 8;
}

size_t enc_smem_bytes(const Geom& g) {
    const int G = enc_planes_per_cta(g);
    size_t off = align_up((size_t)G * g.H * g.W * sizeof(float), 16);
    off += (size_t)G * g.Wp * g.nwords * sizeof(unsigned);
    off += (size_t)4 * G * g.Wp * sizeof(int);
    return off;
}

cudaError_t launch_encode(const Geom& g, bool cps, const float* x, spc_encoding* e, void* ws, cudaStream_t st) {
    WsLayout L = ws_layout(g);
    EncArgs a;
    a.g = g; a.x = x;
    a.ptr = e->ptr; a.da = e->da; a.in = e->in;
    a.chan_ptr_off = e->chan_ptr_off; a.chan_nz_off = e->chan_nz_off; a.chan_in_off = e->chan_in_off;
    a.lengths = e->lengths;
    a.cap_ptr = e->ptr_cap; a.cap_da = e->da_cap; a.cap_in = e->in_cap;
    unsigned char* base = static_cast<unsigned char*>(ws);
    a.st = reinterpret_cast<EncState*>(base + L.state);
    a.flags = reinterpret_cast<int*>(base + L.flags);
    a.agg = reinterpret_cast<long long*>(base + L.agg);
    a.inc = reinterpret_cast<long long*>(base + L.inc);
    a.G = enc_planes_per_cta(g);
    a.WPP = kEncWarps / a.G;
    a.ntiles = (int)((g.NC + a.G - 1) / a.G);
    size_t smem = enc_smem_bytes(g);
    static size_t attr_bytes[2] = {0, 0};
    if (attr_bytes[cps] < smem) {
        cudaError_t err = cps ? cudaFuncSetAttribute(encode_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                              : cudaFuncSetAttribute(encode_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err != cudaSuccess) return err;
        attr_bytes[cps] = smem;
    }
    if (cps) encode_kernel<true><<<a.ntiles, kThreads, smem, st>>>(a);
    else encode_kernel<false><<<a.ntiles, kThreads, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace spc
