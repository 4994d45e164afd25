// sparse_conv.cu -- SpMV-style convolution over the CPO / CPS encoding (sm_100a).
//
// What it computes (PAPER.md:236-309 Alg. 2 / convSpMv, :376-426 Alg. 4,
// SI Alg. 6): every NZE v at padded (h, w) of channel c adds v * W[k,c,l,m]
// to the output that sees it through kernel tap (l, m); with a stride the
// stride-1 outputs off the stride grid are dropped (reading A15).  Result =
// Eq. 1 up to fp32 reassociation.  NPC channels and NPF blocks are never read.
//
// B200 design (FP32 FFMA pipe, no tensor cores: the work is not a dense
// contraction):
//  * CTA = (image n, output tile TY x TX, group of 32*KPL output channels);
//    its WARPS warps split the input channels and are reduced through smem
//    at the end (deterministic, no atomics);
//  * lanes = output channels k.  A warp walks one channel at a time: it
//    parses the channel's ptr blocks (NOP / overlap2..K_w, skipping NPF),
//    reads the DA/IN ranges of the input columns under the tile, keeps the
//    NZEs whose rows fall in the tile window (ballot compaction into a smem
//    list of {value, window position}), then replays the list: a warp-uniform
//    jump table on the window position selects a static FFMA sequence into a
//    register-resident accumulator tile (acc[KPL][TY][TX] per lane) with the
//    channel's taps held in registers (w[KPL][R][S]);
//  * the GENERIC variant (any R, S, stride) runs the same pipeline with smem
//    accumulators and runtime tap loops.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "common.cuh"
#include "dispatch_gen.cuh"

namespace spc {

// ---------------------------------------------------------------- weights

__global__ void pack_weights_kernel(Geom g, const float* __restrict__ w, float* __restrict__ wp) {
    // KCRS -> [C][R][S][K]
    const long long total = (long long)g.K * g.C * g.R * g.S;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(i % g.K);
        const long long crs = i / g.K;
        wp[i] = w[(long long)k * g.C * g.R * g.S + crs];
    }
}

cudaError_t launch_pack_weights(const Geom& g, const float* w, float* wp, cudaStream_t st) {
    long long total = (long long)g.K * g.C * g.R * g.S;
    long long nb = (total + 255) / 256; int blocks = (int)(nb < 148 * 8 ? nb : 148 * 8);
    pack_weights_kernel<<<blocks, 256, 0, st>>>(g, w, wp);
    return cudaGetLastError();
}

// ------------------------------------------------------ channel ptr parse

constexpr int kMaxS = 8;

// Block directory of one channel, from its ptr segment `seg` (Alg. 2 lines
// 9-20).  pos[t]: position in seg of the first count of block t (NOP: a, a+b),
// -1 when the block is absent or NPF; da[t]: DA offset of block t inside the
// channel.  Works on a global or a shared-memory copy of the segment.
struct ChanDir {
    int npc;
    int pos[kMaxS];
    int da[kMaxS];
};

__device__ __forceinline__ void parse_channel_rel(const Geom& g, const int32_t* seg, ChanDir& d) {
#pragma unroll
    for (int t = 0; t < kMaxS; t++) { d.pos[t] = -1; d.da[t] = 0; }
    d.npc = (seg[0] == SPC_NPC);                 // skip channel
    if (d.npc) return;
    if (g.S == 1) {                              // SI Alg. 5: [0, c_0 .. c_{Ow-1}]
        d.pos[0] = 1;
        return;
    }
    int p = 0, dacur = 0;
    if (g.pl == 0) {                             // NOP [0, a, a+b]
        d.pos[0] = 1;
        dacur = seg[2];
        p = 3;
    }
#pragma unroll 1
    for (int t = max(1, g.pl); t <= g.S - 1; t++) {
        if (seg[p + 1] == SPC_NPF) {            // skip pointer
            p += 2;
            continue;
        }
        d.pos[t] = p + 1;
        d.da[t] = dacur;
        const int last = (t < g.S - 1) ? (g.Ow1 - 1 - t) : (g.Ow1 - g.S);
        dacur += seg[p + 1 + last];
        p += 1 + g.Ow1;
    }
}

__device__ __forceinline__ void parse_channel(const Geom& g, const int32_t* __restrict__ ptr, long long P,
                                              ChanDir& d) {
    parse_channel_rel(g, ptr + P, d);
}

// DA range [lo, hi) (channel-relative) of padded column w.
__device__ __forceinline__ void column_range_rel(const Geom& g, const int32_t* seg, const ChanDir& d, int w,
                                                 int& lo, int& hi) {
    lo = hi = 0;
    if (w < 0 || w >= g.Wp) return;
    if (g.S == 1) {                                           // channel-cumulative counts
        lo = (w == 0) ? 0 : seg[d.pos[0] + w - 1];
        hi = seg[d.pos[0] + w];
        return;
    }
    if (w >= g.S - 1 && w <= g.Wp - g.S) {                    // overlapK_w column of partition s
        const int t = g.S - 1, s = w - g.S + 1;
        if (d.pos[t] < 0) return;
        lo = d.da[t] + ((s == 0) ? 0 : seg[d.pos[t] + s - 1]);
        hi = d.da[t] + seg[d.pos[t] + s];
        return;
    }
    const bool left = w < g.S - 1;
    const int t = left ? w : (g.Wp - 1 - w);
    if (t < g.pl || d.pos[t] < 0) return;                    // pad column or NPF block
    if (t == 0) {                                             // NOP: col 0 then col Wp-1
        const int a = seg[d.pos[0]];
        if (left) { lo = 0; hi = a; }
        else { lo = a; hi = seg[d.pos[0] + 1]; }
        return;
    }
    const int c0 = seg[d.pos[t]];                             // left column owned by partition 0
    if (left) { lo = d.da[t]; hi = d.da[t] + c0; }
    else { lo = d.da[t] + c0; hi = d.da[t] + seg[d.pos[t] + g.Ow1 - 1 - t]; }
}

__device__ __forceinline__ void column_range(const Geom& g, const int32_t* __restrict__ seg, const ChanDir& d,
                                             int w, int& lo, int& hi) {
    column_range_rel(g, seg, d, w, lo, hi);
}

// -------------------------------------------------------- CPS expansion

// Alg. 4 index reconstruction for the overlapK_w block:
// negative entry -> singleton at -e; non-negative e -> first NZE at e, the
// next entry is the pattern P and the other NZEs follow at e + S*nextOffset.
// Warp-parallel: inside a maximal run of non-negative entries, indices and
// patterns alternate, so a lane knows its role from the distance to the last
// negative entry (carried across 32-entry chunks); per-entry NZE counts
// (1 / popc(P) / 0) are scanned to give each entry its DA position.
// Output: CPO-form indices at DA positions (in_cpo[chan_nz_off + r]).
__global__ void __launch_bounds__(256) cps_expand_kernel(Geom g, const int32_t* __restrict__ ptr,
                                                         const int32_t* __restrict__ in,
                                                         const int64_t* __restrict__ cpo_off,
                                                         const int64_t* __restrict__ cnz_off,
                                                         const int64_t* __restrict__ cin_off,
                                                         int32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long nc = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (nc >= g.NC) return;
    const long long Z = cnz_off[nc], Q = cin_off[nc];
    const int nnz = (int)(cnz_off[nc + 1] - Z), nin = (int)(cin_off[nc + 1] - Q);
    if (nnz == 0) return;
    int dmid = nnz;  // DA offset where the overlapK_w block starts
    if (g.S > 1) {
        ChanDir d;
        parse_channel(g, ptr, cpo_off[nc], d);
        dmid = (d.pos[g.S - 1] >= 0) ? d.da[g.S - 1] : nnz;
    }
    // 1:1 part (every block below overlapK_w; all of it for S = 1)
    for (int r = lane; r < dmid; r += 32) out[Z + r] = in[Q + r];
    if (dmid == nnz) return;
    const int S = g.S;
    int q = dmid, dpos = dmid;
    bool carry_pat = false;  // next entry is a pattern (its index ended the previous chunk)
    while (q < nin) {
        const int i = q + lane;
        const bool valid = i < nin;
        const int e = valid ? __ldg(in + Q + i) : -1;
        const unsigned neg = __ballot_sync(0xffffffffu, valid && e < 0);
        const unsigned before = neg & lanemask_lt();
        const int r = before ? (32 - __clz(before)) : 0;  // run start (lane after the last negative)
        const bool base_pat = (r == 0) ? carry_pat : false;
        const bool is_pat = valid && e >= 0 && (base_pat ^ (((lane - r) & 1) != 0));
        const bool is_idx = valid && e >= 0 && !is_pat;
        int nxt = __shfl_down_sync(0xffffffffu, e, 1);
        if (lane == 31 && is_idx) nxt = __ldg(in + Q + i + 1);  // pattern sits in the next chunk
        const int cnt = !valid ? 0 : (e < 0 ? 1 : (is_idx ? __popc(nxt & 0xF) : 0));
        int tot;
        const int ex = warp_exclusive_scan(cnt, &tot);
        const long long o = Z + dpos + ex;
        if (valid && e < 0) {
            out[o] = -e;
        } else if (is_idx) {
            const unsigned p = (unsigned)nxt & 0xFu;
            const int b0 = __ffs(p) - 1;
            int u = 0;
#pragma unroll
            for (int b = 0; b < 4; b++)
                if ((p >> b) & 1u) out[o + u++] = e + S * (b - b0);
        }
        const bool last_is_idx = __shfl_sync(0xffffffffu, is_idx, 31);
        carry_pat = last_is_idx;
        dpos += tot;
        q += 32;
    }
}

cudaError_t launch_cps_expand(const Geom& g, const spc_encoding* e, int32_t* in_cpo, cudaStream_t st) {
    const int wpb = 8;
    long long blocks = (g.NC + wpb - 1) / wpb;
    cps_expand_kernel<<<(unsigned)blocks, wpb * 32, 0, st>>>(g, e->ptr, e->in, e->chan_ptr_off, e->chan_nz_off,
                                                            e->chan_in_off, in_cpo);
    return cudaGetLastError();
}

// ------------------------------------------------------------ conv kernels

struct ConvArgs {
    Geom g;
    const int32_t* __restrict__ ptr;
    const float* __restrict__ da;
    const int32_t* __restrict__ in;      // CPO-form indices at DA positions
    const int64_t* __restrict__ cpo_off; // chan_ptr_off
    const int64_t* __restrict__ cnz_off; // chan_nz_off
    const float* __restrict__ wp;        // [C][R][S][K]
    float* __restrict__ y;
    int relu;
    int tiles_x;
    int cg;     // CTAs per cluster splitting the input channels
    int pmax;   // longest ptr segment of one channel
};

// Tile configuration of the register-tile kernel.
//   TY x TX outputs per CTA, KPL output channels per lane, KG k-groups of 32*KPL
//   channels and CS channel splits per CTA (WARPS = KG*CS), CH channels staged
//   per chunk.
template <int R_, int S_, int SH_, int SW_, int TY_, int TX_, int KPL_, int KG_, int CS_, int CH_, int MINB_ = 1>
struct TileCfg {
    static constexpr int MINB = MINB_;   // CTAs per SM the register budget targets
    static constexpr int R = R_, S = S_, SH = SH_, SW = SW_, TY = TY_, TX = TX_, KPL = KPL_;
    static constexpr int KG = KG_, CS = CS_, CH = CH_;
    static constexpr int WARPS = KG * CS, THREADS = 32 * WARPS;
    static constexpr int KB = 32 * KPL * KG;          // output channels per CTA
    static constexpr int RS = R * S;
    static constexpr int NACC = KPL * TY * TX;         // accumulators per lane
    static constexpr int WH = (TY - 1) * SH + R;       // input window rows
    static constexpr int WW = (TX - 1) * SW + S;       // input window cols
    static constexpr int NCASE = WH * WW;
    static_assert(WW <= 32, "window columns are mapped to lanes");
    static_assert(NCASE <= 256, "jump table size");
    static_assert(NACC % 32 == 0, "reduction pieces of 32 accumulators");
    using RP = Replay<R, S, SH, SW, TY, TX, KPL>;
    using Word = typename RP::Word;                     // f32x2 pair (k, k+32) or f32
    static constexpr int NP = RP::kPacked ? KPL / 2 : KPL;
};

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}

// Builds the list of NZEs of one channel that fall in the window
// [hy0, hy0+WH) x [wx0, wx0+WW) (padded coordinates) from global memory;
// returns its length (generic kernel).  lanes j < WW own window column wx0 + j.
__device__ __forceinline__ int build_list(const ConvArgs& a, const int32_t* seg, const ChanDir& d, long long Z,
                                          int hy0, int wx0,
                                          int WH, int WW, float2* list) {
    const Geom& g = a.g;
    const int lane = threadIdx.x & 31;
    int lo = 0, hi = 0;
    if (lane < WW) column_range(g, seg, d, wx0 + lane, lo, hi);
    int n = 0;
    unsigned nonempty = __ballot_sync(0xffffffffu, hi > lo);
    while (nonempty) {
        const int j = __ffs(nonempty) - 1;
        nonempty &= nonempty - 1;
        const int clo = __shfl_sync(0xffffffffu, lo, j);
        const int chi = __shfl_sync(0xffffffffu, hi, j);
        for (int b = clo; b < chi; b += 32) {
            const int i = b + lane;
            bool keep = false;
            int h = 0;
            if (i < chi) {
                h = __ldg(a.in + Z + i) / g.S;   // IN = L + h*S, L < S
                keep = (h >= hy0) && (h < hy0 + WH);
            }
            const unsigned km = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int pos = n + __popc(km & lanemask_lt());
                list[pos] = make_float2(__ldg(a.da + Z + i), __int_as_float((h - hy0) * WW + j));
            }
            n += __popc(km);
            if (__shfl_sync(0xffffffffu, h, 31) >= hy0 + WH && b + 32 < chi) break;
        }
    }
    __syncwarp();
    return n;
}

// Register-tile kernel.  Per chunk of CH input channels:
//  P0  stage the chunk's ptr segments (contiguous in the stream), DA offsets and
//      the taps W[c][l][m][kbase..kbase+KB) in shared memory (cp.async);
//  P1  one warp per channel: block directory from the staged ptr (NPC/NPF skip),
//      DA ranges of the window columns, then the window columns' NZEs with many
//      loads in flight; rows outside the tile window are dropped, the kept ones
//      compacted and given their window position -> smem list {v, v, case, 0}
//      closed by a sentinel;
//  P2  warp (kg, cs) replays the lists of channels cs, cs+CS, ... with the
//      generated brx.idx / FFMA2 loop into register accumulators.
// Epilogue: reduce the CS warps through smem (all warps), then the cg CTAs of
// the cluster through distributed shared memory; ReLU; coalesced NKHW store.
template <class T>
__global__ void __launch_bounds__(T::THREADS, T::MINB) sparse_conv_kernel(ConvArgs a) {
    namespace cgrp = cooperative_groups;
    const Geom& g = a.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kg = warp / T::CS, cs = warp % T::CS;
    const int n = blockIdx.z / a.cg;
    const int rank = (a.cg > 1) ? (int)cgrp::this_cluster().block_rank() : 0;
    const int kbase = blockIdx.y * T::KB;
    const int tyi = blockIdx.x / a.tiles_x, txi = blockIdx.x % a.tiles_x;
    const int oy0 = tyi * T::TY, ox0 = txi * T::TX;
    const int hy0 = oy0 * T::SH, wx0 = ox0 * T::SW;
    const int cper = (g.C + a.cg - 1) / a.cg;
    const int c_begin = rank * cper, c_end = min(g.C, c_begin + cper);
    constexpr int LCAP = T::NCASE + 1;   // list capacity per channel, + sentinel

    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* s_w = reinterpret_cast<float*>(smem_raw);                                  // [CH][RS][KB]
    float4* s_list = reinterpret_cast<float4*>(s_w + T::CH * T::RS * T::KB);          // [CH][LCAP]
    int* s_ptr = reinterpret_cast<int*>(s_list + T::CH * LCAP);                       // [CH * pmax]
    int* s_poff = s_ptr + T::CH * a.pmax;                                             // [CH]
    int* s_cnt = s_poff + T::CH;                                                      // [CH]
    int* s_scr = s_cnt + T::CH;                                                       // [WARPS][2][32]
    long long* s_z = reinterpret_cast<long long*>(s_scr + T::WARPS * 64 + 2);         // [CH] (8B aligned)
    s_z = reinterpret_cast<long long*>((reinterpret_cast<uintptr_t>(s_z) + 7) & ~uintptr_t(7));

    typename T::Word acc[T::NP][T::TY][T::TX];
#pragma unroll
    for (int p = 0; p < T::NP; p++)
#pragma unroll
        for (int yy = 0; yy < T::TY; yy++)
#pragma unroll
            for (int xx = 0; xx < T::TX; xx++) acc[p][yy][xx] = 0;
    const bool w16 = (g.K % 4) == 0;

    for (int c0 = c_begin; c0 < c_end; c0 += T::CH) {
        const int chn = min(T::CH, c_end - c0);
        const long long nc0 = (long long)n * g.C + c0;
        // ---- P0: stage ptr segments, DA offsets, taps (cp.async: all copies in flight at once)
        {
            const long long pbase = __ldg(a.cpo_off + nc0);
            const int plen = (int)(__ldg(a.cpo_off + nc0 + chn) - pbase);
            const int32_t* src = a.ptr + pbase;
            for (int i = threadIdx.x; i < plen; i += T::THREADS) cp_async4(s_ptr + i, src + i, 4);
            if (threadIdx.x < chn) {
                s_poff[threadIdx.x] = (int)(__ldg(a.cpo_off + nc0 + threadIdx.x) - pbase);
                s_z[threadIdx.x] = __ldg(a.cnz_off + nc0 + threadIdx.x);
            }
            const float* wsrc = a.wp + (long long)c0 * T::RS * g.K + kbase;   // row (j*RS+rs) at stride K
            const int rows = chn * T::RS;
            if (w16) {
                constexpr int VPR = T::KB / 4;                 // 16-byte vectors per row
                constexpr int RSTEP = T::THREADS / VPR;
                const int vq = threadIdx.x % VPR, r0 = threadIdx.x / VPR;
                const int kq = 4 * vq;
                const int nb = max(0, min(16, 4 * (g.K - (kbase + kq))));
                for (int r = r0; r < rows; r += RSTEP)
                    cp_async16(s_w + r * T::KB + kq, wsrc + (long long)r * g.K + (nb ? kq : 0), nb);
            } else {
                for (int i = threadIdx.x; i < rows * T::KB; i += T::THREADS) {
                    const int kk = i % T::KB, r = i / T::KB;
                    const bool ok = kbase + kk < g.K;
                    cp_async4(s_w + i, wsrc + (long long)r * g.K + (ok ? kk : 0), ok ? 4 : 0);
                }
            }
            cp_async_wait_all();
        }
        __syncthreads();
        // ---- P1: window NZE lists, one warp per channel
        for (int j = warp; j < chn; j += T::WARPS) {
            const int* seg = s_ptr + s_poff[j];
            float4* lst = s_list + j * LCAP;
            ChanDir d;
            parse_channel_rel(g, seg, d);
            int lo = 0, hi = 0;
            if (!d.npc && lane < T::WW) column_range_rel(g, seg, d, wx0 + lane, lo, hi);
            int tot;
            const int pre = warp_exclusive_scan(hi - lo, &tot);
            int* spre = s_scr + warp * 64;
            int* slo = spre + 32;
            spre[lane] = (lane < T::WW) ? pre : (1 << 30);
            slo[lane] = lo;
            const int lo0 = __shfl_sync(0xffffffffu, lo, 0);
            // contiguous when every window column starts where the flattened prefix says
            const bool contig = __all_sync(0xffffffffu, lane >= T::WW || hi == lo || lo == lo0 + pre);
            __syncwarp();
            const long long Z = s_z[j];
            int cnt = 0;
            // pass 1: load, keep rows of the tile window, compact {v, h, f}
            for (int f0 = 0; f0 < tot; f0 += 128) {
                int e[4], ff[4];
                float v[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int f = f0 + 32 * u + lane;
                    ff[u] = f;
                    e[u] = -1;
                    v[u] = 0.f;
                    if (f < tot) {
                        int idx = lo0 + f;
                        if (!contig) {
                            int jc = 0;
#pragma unroll
                            for (int step = 16; step > 0; step >>= 1)
                                if (jc + step < T::WW && spre[jc + step] <= f) jc += step;
                            idx = slo[jc] + (f - spre[jc]);
                        }
                        e[u] = __ldg(a.in + Z + idx);
                        v[u] = __ldg(a.da + Z + idx);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int h = e[u] / T::S;     // IN = L + h*S with L < S
                    const bool keep = e[u] >= 0 && h >= hy0 && h < hy0 + T::WH;
                    const unsigned km = __ballot_sync(0xffffffffu, keep);
                    if (keep)
                        lst[cnt + __popc(km & lanemask_lt())] =
                            make_float4(v[u], __int_as_float(h - hy0), __int_as_float(ff[u]), 0.f);
                    cnt += __popc(km);
                }
            }
            __syncwarp();
            // pass 2: window column of each kept NZE -> replay entry {v, v, case, 0}
            for (int i = lane; i < cnt; i += 32) {
                const float4 t = lst[i];
                const int f = __float_as_int(t.z);
                int jc = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1)
                    if (jc + step < T::WW && spre[jc + step] <= f) jc += step;
                lst[i] = make_float4(t.x, t.x, __int_as_float(__float_as_int(t.y) * T::WW + jc), 0.f);
            }
            if (lane == 0) {
                lst[cnt] = make_float4(0.f, 0.f, __int_as_float(T::RP::kSentinel), 0.f);
                s_cnt[j] = cnt;
            }
            __syncwarp();
        }
        __syncthreads();
        // ---- P2: FFMA replay (generated brx.idx jump table, FFMA2 bodies)
        for (int j = cs; j < chn; j += T::CS) {
            if (s_cnt[j] == 0) continue;
            typename T::Word w[T::NP][T::R][T::S];
#pragma unroll
            for (int p = 0; p < T::NP; p++)
#pragma unroll
                for (int l = 0; l < T::R; l++)
#pragma unroll
                    for (int m = 0; m < T::S; m++) {
                        const float* ws = s_w + (j * T::RS + l * T::S + m) * T::KB + lane;
                        if constexpr (T::RP::kPacked) {
                            const unsigned lo = __float_as_uint(ws[(kg * T::KPL + 2 * p) * 32]);
                            const unsigned hi = __float_as_uint(ws[(kg * T::KPL + 2 * p + 1) * 32]);
                            w[p][l][m] = (unsigned long long)lo | ((unsigned long long)hi << 32);
                        } else {
                            w[p][l][m] = ws[(kg * T::KPL + p) * 32];
                        }
                    }
            T::RP::run((unsigned)__cvta_generic_to_shared(s_list + j * LCAP), acc, w);
        }
        __syncthreads();
    }

    // ---- epilogue 1: unpack, reduce the CS channel splits (all warps), CTA partial -> part
    constexpr int TT = T::TY * T::TX, TP = TT + 1;
    constexpr int PIECE = 64 < T::NACC ? 64 : T::NACC;
    float* red = s_w;                                              // [CS][KG][PIECE][32]
    float* part = s_w + (T::CS > 1 ? T::CS * T::KG * PIECE * 32 : 0);   // [KG*KPL*32][TP]
    float accf[T::NACC];
#pragma unroll
    for (int p = 0; p < T::NP; p++)
#pragma unroll
        for (int t = 0; t < TT; t++) {
            if constexpr (T::RP::kPacked) {
                accf[(2 * p) * TT + t] = __uint_as_float((unsigned)(acc[p][t / T::TX][t % T::TX] & 0xffffffffull));
                accf[(2 * p + 1) * TT + t] = __uint_as_float((unsigned)(acc[p][t / T::TX][t % T::TX] >> 32));
            } else {
                accf[p * TT + t] = acc[p][t / T::TX][t % T::TX];
            }
        }
    // accf index i = kk*TT + t  ->  part[((kg*KPL + kk)*32 + lane)*TP + t]
    if constexpr (T::CS == 1) {
#pragma unroll
        for (int i = 0; i < T::NACC; i++) part[((kg * T::KPL + i / TT) * 32 + lane) * TP + i % TT] = accf[i];
    } else {
#pragma unroll
        for (int pc = 0; pc < T::NACC / PIECE; pc++) {
#pragma unroll
            for (int i = 0; i < PIECE; i++) red[((cs * T::KG + kg) * PIECE + i) * 32 + lane] = accf[pc * PIECE + i];
            __syncthreads();
            constexpr int PER = PIECE / T::CS;
            for (int i = cs * PER; i < (cs + 1) * PER; i++) {
                float sum = 0.f;
#pragma unroll
                for (int q = 0; q < T::CS; q++) sum += red[((q * T::KG + kg) * PIECE + i) * 32 + lane];
                const int gi = pc * PIECE + i;
                part[((kg * T::KPL + gi / TT) * 32 + lane) * TP + gi % TT] = sum;
            }
            __syncthreads();
        }
    }
    if (a.cg > 1) cgrp::this_cluster().sync(); else __syncthreads();
    // ---- epilogue 2: sum the cluster's partials (DSMEM), ReLU, store NKHW
    float* peers[8];
#pragma unroll
    for (int r = 0; r < 8; r++) peers[r] = (r < a.cg && r != rank) ? cgrp::this_cluster().map_shared_rank(part, r) : nullptr;
    const int total = T::KB * TT;
    const int per = (total + a.cg - 1) / a.cg;
    const int i0 = rank * per, i1 = min(total, i0 + per);
    for (int i = i0 + threadIdx.x; i < i1; i += T::THREADS) {
        const int t = i % TT, kl = i / TT;        // kl = (kg*KPL + kk)*32 + lane
        const int sidx = kl * TP + t;
        float sum = part[sidx];
#pragma unroll
        for (int r = 0; r < 8; r++)
            if (peers[r]) sum += peers[r][sidx];
        const int k = kbase + kl, oy = oy0 + t / T::TX, ox = ox0 + t % T::TX;
        if (k >= g.K || oy >= g.Oh || ox >= g.Ow) continue;
        if (a.relu) sum = fmaxf(sum, 0.f);
        a.y[(((long long)n * g.K + k) * g.Oh + oy) * g.Ow + ox] = sum;
    }
    if (a.cg > 1) cgrp::this_cluster().sync();
}

// Generic variant: any R, S, stride; TY x TX = 4 x 4 tile, accumulators in smem.
constexpr int kGenTY = 4, kGenTX = 4, kGenWarps = 4;

__global__ void __launch_bounds__(kGenWarps * 32) sparse_conv_generic_kernel(ConvArgs a, int WH, int WW) {
    const Geom& g = a.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = blockIdx.z;
    const int kbase = blockIdx.y * 32;
    const int tyi = blockIdx.x / a.tiles_x, txi = blockIdx.x % a.tiles_x;
    const int oy0 = tyi * kGenTY, ox0 = txi * kGenTX;
    const int hy0 = oy0 * g.sh, wx0 = ox0 * g.sw;
    const int NCASE = WH * WW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* accs = reinterpret_cast<float*>(smem_raw);                       // [WARPS][TY*TX][32]
    float2* list = reinterpret_cast<float2*>(accs + kGenWarps * kGenTY * kGenTX * 32) + warp * NCASE;
    float* acc = accs + warp * kGenTY * kGenTX * 32;
    for (int i = 0; i < kGenTY * kGenTX; i++) acc[i * 32 + lane] = 0.f;
    const int k = kbase + lane;
    for (int c = warp; c < g.C; c += kGenWarps) {
        const long long nc = (long long)n * g.C + c;
        ChanDir d;
        const int32_t* seg = a.ptr + a.cpo_off[nc];
        parse_channel_rel(g, seg, d);
        if (d.npc) continue;
        const long long Z = a.cnz_off[nc];
        const int cnt = build_list(a, seg, d, Z, hy0, wx0, WH, WW, list);
        for (int e = 0; e < cnt; e++) {
            const float2 it = list[e];
            const int cs = __float_as_int(it.y);
            const int hr = cs / WW, wr = cs % WW;
            for (int l = 0; l < g.R; l++) {
                const int y1 = hr - l;
                if (y1 < 0 || y1 % g.sh) continue;
                if (y1 / g.sh >= kGenTY) continue;
                for (int m = 0; m < g.S; m++) {
                    const int x1 = wr - m;
                    if (x1 < 0 || x1 % g.sw || x1 / g.sw >= kGenTX) continue;
                    const float wv = (k < g.K) ? __ldg(a.wp + (((long long)c * g.R + l) * g.S + m) * g.K + k) : 0.f;
                    float* p = acc + ((y1 / g.sh) * kGenTX + x1 / g.sw) * 32 + lane;
                    *p = fmaf(it.x, wv, *p);
                }
            }
        }
        __syncwarp();
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 32 * kGenTY * kGenTX; idx += kGenWarps * 32) {
        const int xx = idx % kGenTX, yy = (idx / kGenTX) % kGenTY, kl = idx / (kGenTX * kGenTY);
        const int kk = kbase + kl, oy = oy0 + yy, ox = ox0 + xx;
        if (kk >= g.K || oy >= g.Oh || ox >= g.Ow) continue;
        float s = 0.f;
        for (int wv = 0; wv < kGenWarps; wv++) s += accs[(wv * kGenTY * kGenTX + yy * kGenTX + xx) * 32 + kl];
        if (a.relu) s = fmaxf(s, 0.f);
        a.y[(((long long)n * g.K + kk) * g.Oh + oy) * g.Ow + ox] = s;
    }
}

template <class T>
static size_t tiled_smem(const ConvArgs& a) {
    const size_t main = (size_t)T::CH * T::RS * T::KB * 4 + (size_t)T::CH * (T::NCASE + 1) * 16 +
                        (size_t)T::CH * a.pmax * 4 + (size_t)2 * T::CH * 4 + (size_t)(T::WARPS * 64 + 2) * 4 + 16 +
                        (size_t)T::CH * 8;
    constexpr int PIECE = 64 < T::NACC ? 64 : T::NACC;
    const size_t red = (T::CS > 1 ? (size_t)T::CS * T::KG * PIECE * 32 * 4 : 0) +
                       (size_t)T::KB * (T::TY * T::TX + 1) * 4;
    return std::max(main, red);
}

template <class T>
static cudaError_t run_tiled(ConvArgs& a, int cg, cudaStream_t st) {
    const Geom& g = a.g;
    const int tx = (g.Ow + T::TX - 1) / T::TX, ty = (g.Oh + T::TY - 1) / T::TY;
    a.tiles_x = tx;
    a.cg = cg;
    const int kblocks = (g.K + T::KB - 1) / T::KB;
    const size_t smem = tiled_smem<T>(a);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    static bool attr_set = false;     // per instantiation
    static size_t attr_bytes = 0;
    if (!attr_set || attr_bytes < smem) {
        cudaError_t err = cudaFuncSetAttribute(sparse_conv_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)std::max(smem, attr_bytes));
        if (err != cudaSuccess) return err;
        attr_set = true;
        attr_bytes = std::max(smem, attr_bytes);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(tx * ty, kblocks, g.N * cg);
    cfg.blockDim = dim3(T::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = cg;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, sparse_conv_kernel<T>, a);
}

// Channel split across a cluster: the largest cg in {1,2,3,4,6,8} that keeps the
// grid within one wave of resident CTAs and at least 8 channels per CTA.
static int pick_cg(long long ctas, int C, int minb) {
    int best = 1;
    const int cands[] = {1, 2, 3, 4, 6, 8};
    for (int cg : cands)
        if (ctas * cg <= 148LL * minb && C >= 8 * cg) best = cg;
    return best;
}

// Development override: SPC_TUNE="<config>:<cg>" (cg 0 = automatic).
static const char* tune_cfg(int* cg) {
    static const char* env = getenv("SPC_TUNE");
    *cg = 0;
    if (!env) return nullptr;
    const char* colon = strchr(env, ':');
    if (colon) *cg = atoi(colon + 1);
    return env;
}

template <class T>
static cudaError_t run_auto(ConvArgs& a, int cg_override, cudaStream_t st) {
    const Geom& g = a.g;
    const long long ctas = (long long)((g.Oh + T::TY - 1) / T::TY) * ((g.Ow + T::TX - 1) / T::TX) *
                           ((g.K + T::KB - 1) / T::KB) * g.N;
    const int cg = cg_override > 0 ? cg_override : pick_cg(ctas, g.C, T::MINB);
    return run_tiled<T>(a, cg, st);
}

static bool tune_is(const char* t, const char* name) {
    return t && strncmp(t, name, strlen(name)) == 0 && (t[strlen(name)] == ':' || t[strlen(name)] == 0);
}

cudaError_t launch_sparse_conv(const Geom& g, const spc_encoding* e, const int32_t* in_override,
                               const float* w_packed, float* y, int relu, cudaStream_t st) {
    ConvArgs a;
    a.g = g;
    a.ptr = e->ptr;
    a.da = e->da;
    a.in = in_override ? in_override : e->in;
    a.cpo_off = e->chan_ptr_off;
    a.cnz_off = e->chan_nz_off;
    a.wp = w_packed;
    a.y = y;
    a.relu = relu;
    a.tiles_x = 1;
    a.cg = 1;
    a.pmax = (g.S == 1) ? (1 + g.Ow1) : (3 + (g.S - 1) * (1 + g.Ow1));
    int tcg = 0;
    const char* t = tune_cfg(&tcg);
    if (g.R == 3 && g.S == 3 && g.sh == 1 && g.sw == 1) {
        using A = TileCfg<3, 3, 1, 1, 8, 8, 2, 1, 8, 16, 1>;
        using B = TileCfg<3, 3, 1, 1, 4, 8, 2, 1, 8, 16, 2>;
        using C = TileCfg<3, 3, 1, 1, 4, 8, 2, 1, 4, 16, 3>;
        using D = TileCfg<3, 3, 1, 1, 4, 8, 4, 1, 8, 16, 1>;
        using E = TileCfg<3, 3, 1, 1, 4, 8, 4, 1, 4, 16, 2>;
        using F = TileCfg<3, 3, 1, 1, 8, 8, 1, 1, 8, 16, 1>;
        if (tune_is(t, "A")) return run_auto<A>(a, tcg, st);
        if (tune_is(t, "B")) return run_auto<B>(a, tcg, st);
        if (tune_is(t, "C")) return run_auto<C>(a, tcg, st);
        if (tune_is(t, "D")) return run_auto<D>(a, tcg, st);
        if (tune_is(t, "E")) return run_auto<E>(a, tcg, st);
        if (g.K <= 32) return run_auto<F>(a, tcg, st);
        if (g.K <= 64) return run_auto<B>(a, tcg, st);
        return run_auto<E>(a, tcg, st);
    }
    if (g.R == 3 && g.S == 3 && g.sh == 2 && g.sw == 2) {
        using A = TileCfg<3, 3, 2, 2, 4, 8, 2, 1, 8, 16, 2>;
        using B = TileCfg<3, 3, 2, 2, 4, 8, 4, 1, 8, 16, 1>;
        using C = TileCfg<3, 3, 2, 2, 4, 8, 4, 1, 4, 16, 2>;
        if (tune_is(t, "A")) return run_auto<A>(a, tcg, st);
        if (tune_is(t, "B")) return run_auto<B>(a, tcg, st);
        if (tune_is(t, "C")) return run_auto<C>(a, tcg, st);
        if (g.K <= 64) return run_auto<A>(a, tcg, st);
        return run_auto<C>(a, tcg, st);
    }
    if (g.R == 1 && g.S == 7 && g.sh == 1 && g.sw == 1) {
        using A = TileCfg<1, 7, 1, 1, 8, 8, 2, 1, 8, 16, 1>;
        return run_auto<A>(a, tcg, st);
    }
    if (g.R == 7 && g.S == 1 && g.sh == 1 && g.sw == 1) {
        using A = TileCfg<7, 1, 1, 1, 8, 8, 2, 1, 8, 16, 1>;
        return run_auto<A>(a, tcg, st);
    }
    // generic
    const int WH = (kGenTY - 1) * g.sh + g.R, WW = (kGenTX - 1) * g.sw + g.S;
    if (WW > 32) return cudaErrorInvalidValue;
    a.tiles_x = (g.Ow + kGenTX - 1) / kGenTX;
    const int ty = (g.Oh + kGenTY - 1) / kGenTY;
    size_t smem = (size_t)kGenWarps * kGenTY * kGenTX * 32 * sizeof(float) + (size_t)kGenWarps * WH * WW * sizeof(float2);
    cudaError_t err = cudaFuncSetAttribute(sparse_conv_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    dim3 grid(a.tiles_x * ty, (g.K + 31) / 32, g.N);
    sparse_conv_generic_kernel<<<grid, kGenWarps * 32, smem, st>>>(a, WH, WW);
    return cudaGetLastError();
}

}  // namespace spc
