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
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "common.cuh"

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

// Compile-time-S variant for the strip kernel: fully unrolled, so the
// directory stays in registers (a runtime-indexed ChanDir spills to local memory).
template <int S>
struct DirS {
    int npc;
    int pos[S];
    int da[S];
};

template <int S>
__device__ __forceinline__ void parse_dir(const Geom& g, const int32_t* seg, DirS<S>& d) {
#pragma unroll
    for (int t = 0; t < S; t++) { d.pos[t] = -1; d.da[t] = 0; }
    d.npc = (seg[0] == SPC_NPC);
    if (d.npc) return;
    if (S == 1) {                                // SI Alg. 5: [0, c_0 .. c_{Ow-1}]
        d.pos[0] = 1;
        return;
    }
    int p = 0, dacur = 0;
    if (g.pl == 0) {                             // NOP [0, a, a+b]
        d.pos[0] = 1;
        dacur = seg[2];
        p = 3;
    }
#pragma unroll
    for (int t = 1; t < S; t++) {
        if (t < g.pl) continue;                  // pad columns own no block
        if (seg[p + 1] == SPC_NPF) {            // skip pointer
            p += 2;
            continue;
        }
        d.pos[t] = p + 1;
        d.da[t] = dacur;
        const int last = (t < S - 1) ? (g.Ow1 - 1 - t) : (g.Ow1 - S);
        dacur += seg[p + 1 + last];
        p += 1 + g.Ow1;
    }
}

template <int S>
__device__ __forceinline__ int sel(const int (&arr)[S], int t) {
    int v = arr[0];
#pragma unroll
    for (int i = 1; i < S; i++)
        if (t == i) v = arr[i];
    return v;
}

// DA range [lo, hi) (channel-relative) of padded column w (compile-time S).
template <int S>
__device__ __forceinline__ void column_range_s(const Geom& g, const int32_t* seg, const DirS<S>& d, int w,
                                               int& lo, int& hi) {
    lo = hi = 0;
    if (w < 0 || w >= g.Wp) return;
    if (S == 1) {
        lo = (w == 0) ? 0 : seg[d.pos[0] + w - 1];
        hi = seg[d.pos[0] + w];
        return;
    }
    if (w >= S - 1 && w <= g.Wp - S) {                        // overlapK_w column of partition s
        const int s = w - S + 1;
        if (d.pos[S - 1] < 0) return;
        lo = d.da[S - 1] + ((s == 0) ? 0 : seg[d.pos[S - 1] + s - 1]);
        hi = d.da[S - 1] + seg[d.pos[S - 1] + s];
        return;
    }
    const bool left = w < S - 1;
    const int t = left ? w : (g.Wp - 1 - w);
    const int pos = sel(d.pos, t), dat = sel(d.da, t);
    if (t < g.pl || pos < 0) return;                          // pad column or NPF block
    if (t == 0) {                                             // NOP: col 0 then col Wp-1
        const int a = seg[pos];
        if (left) { lo = 0; hi = a; }
        else { lo = a; hi = seg[pos + 1]; }
        return;
    }
    const int c0 = seg[pos];                                  // left column owned by partition 0
    if (left) { lo = dat; hi = dat + c0; }
    else { lo = dat + c0; hi = dat + seg[pos + g.Ow1 - 1 - t]; }
}

// Stride-aware layout (reading A32, stride_aware.cu): partitions = output columns at stride
// s_w; coverage / owner of a padded column, block directory and column ranges.  Used when
// every (partition, type) owns at most one non-pad column (3x3 / stride 2 and the like; the
// host checks), so a partition's count range IS its column's range.
__device__ __forceinline__ int sa_cov_c(const Geom& g, int w) {
    const int hi = min(g.Ow - 1, w / g.sw);
    const int lo = (w - g.S + 1 <= 0) ? 0 : (w - g.S + 1 + g.sw - 1) / g.sw;
    return max(0, hi - lo + 1);
}
__device__ __forceinline__ int sa_owner_c(const Geom& g, int w) {
    return (w - g.S + 1 <= 0) ? 0 : (w - g.S + 1 + g.sw - 1) / g.sw;
}

template <int S>
__device__ __forceinline__ void parse_dir_sa(const Geom& g, const int32_t* seg, DirS<S>& d, unsigned types) {
#pragma unroll
    for (int t = 0; t < S; t++) { d.pos[t] = -1; d.da[t] = 0; }
    d.npc = (seg[0] == SPC_NPC);
    if (d.npc) return;
    int p = 0, dacur = 0;
#pragma unroll
    for (int t = 0; t < S; t++) {
        if (!((types >> t) & 1u)) continue;
        if (seg[p + 1] == SPC_NPF) { p += 2; continue; }
        d.pos[t] = p + 1;
        d.da[t] = dacur;
        int last = 0;
        for (int s2 = g.Ow - 1; s2 >= 0; s2--) {
            const int v = seg[p + 1 + s2];
            if (v >= 0) { last = v; break; }
        }
        dacur += last;
        p += 1 + g.Ow;
    }
}

template <int S>
__device__ __forceinline__ void column_range_sa(const Geom& g, const int32_t* seg, const DirS<S>& d, int w, int& lo,
                                                int& hi) {
    lo = hi = 0;
    if (w < g.pl || w >= g.pl + g.W) return;                  // pad columns hold no NZE
    const int cov = sa_cov_c(g, w);
    if (cov == 0) return;
    const int t = cov - 1, s = sa_owner_c(g, w);
    const int pos = sel(d.pos, t), dat = sel(d.da, t);
    if (pos < 0) return;                                       // NPF block
    const int c = seg[pos + s];
    if (c < 0) return;
    int prev = 0;
    for (int s2 = s - 1; s2 >= 0; s2--) {
        const int v = seg[pos + s2];
        if (v >= 0) { prev = v; break; }
    }
    lo = dat + prev;
    hi = dat + c;
}

// Stride-aware layout, general case: slot q of the window = (partition s = s_lo + q / T, type
// t = q % T) over the partitions whose owned columns can fall in [wx0, wx0 + WW); its DA range
// [lo, hi) and the window column of its partition's first column cb = s*s_w - wx0.  An NZE of the
// slot sits at window column cb + L (L = IN % K_w); those outside [0, WW) are skipped.
__device__ __forceinline__ int sa_slot_s_lo(const Geom& g, int wx0) {
    const int num = wx0 - g.S + 1;
    return num <= 0 ? 0 : (num + g.sw - 1) / g.sw;
}
__device__ __forceinline__ int sa_nslots(const Geom& g, int wx0, int WW) {
    const int T = (g.S + g.sw - 1) / g.sw;
    const int s_lo = sa_slot_s_lo(g, wx0), s_hi = min(g.Ow - 1, (wx0 + WW - 1) / g.sw);
    return max(0, s_hi - s_lo + 1) * T;
}
template <int S>
__device__ __forceinline__ void sa_slot_range(const Geom& g, const int32_t* seg, const DirS<S>& d, int wx0, int WW,
                                              int q, int& lo, int& hi, int& cb) {
    lo = hi = 0;
    cb = 0;
    const int T = (g.S + g.sw - 1) / g.sw;
    const int s = sa_slot_s_lo(g, wx0) + q / T, t = q % T;
    if (q >= sa_nslots(g, wx0, WW)) return;
    cb = s * g.sw - wx0;
    const int pos = sel(d.pos, t), dat = sel(d.da, t);
    if (pos < 0) return;
    const int c = seg[pos + s];
    if (c < 0) return;
    int prev = 0;
    for (int s2 = s - 1; s2 >= 0; s2--) {
        const int v = seg[pos + s2];
        if (v >= 0) { prev = v; break; }
    }
    lo = dat + prev;
    hi = dat + c;
}

// -------------------------------------------------------- CPS expansion

// Alg. 4 index reconstruction for the overlapK_w block:
// negative entry -> singleton at -e; non-negative e -> first NZE at e, the
// next entry is the pattern P and the other NZEs follow at e + S*nextOffset.
// Warp-parallel: inside a maximal run of non-negative entries, indices and
// patterns alternate, so a lane knows its role from the distance to the last
// negative entry (carried across 32-entry chunks); per-entry NZE counts
// (1 / popc(P) / 0) are scanned to give each entry its DA position.
// One CTA per channel: the block's entries are cut into 8 warp segments; a warp finds
// its starting role by looking back to the last negative entry before its segment,
// counts its NZEs (pass 1), takes its DA base from a scan over the warps' counts, and
// writes (pass 2, loads served by L1).
// Output: CPO-form indices at DA positions (in_cpo[chan_nz_off + r]).
template <bool WRITE>
__device__ __forceinline__ int cps_segment(const int32_t* __restrict__ in, long long Q, int q0, int q1, int nin,
                                           bool carry_pat, int S, int32_t* __restrict__ out, long long obase) {
    const int lane = threadIdx.x & 31;
    int dpos = 0;
    constexpr int B = 4;     // chunks of 32 entries whose loads are in flight together
    for (int q = q0; q < q1; q += 32 * B) {
        int eb[B];
#pragma unroll
        for (int b = 0; b < B; b++) {
            const int i = q + 32 * b + lane;
            eb[b] = (i < q1) ? __ldg(in + Q + i) : -1;
        }
        const int after = min(q + 32 * B, q1);                      // first entry after the batch
        const int tail = (after < nin) ? __ldg(in + Q + after) : -1;
#pragma unroll
        for (int b = 0; b < B; b++) {
            const int i = q + 32 * b + lane;
            const bool valid = i < q1;
            const int e = eb[b];
            const unsigned neg = __ballot_sync(0xffffffffu, valid && e < 0);
            const unsigned before = neg & lanemask_lt();
            const int r = before ? (32 - __clz(before)) : 0;  // run start (lane after the last negative)
            const bool base_pat = (r == 0) ? carry_pat : false;
            const bool is_pat = valid && e >= 0 && (base_pat ^ (((lane - r) & 1) != 0));
            const bool is_idx = valid && e >= 0 && !is_pat;
            int nxt = __shfl_down_sync(0xffffffffu, e, 1);
            // the successor of the last valid entry of the chunk: lane 0 of the next chunk,
            // or the entry after the batch (the next segment's first entry)
            const int first_next = __shfl_sync(0xffffffffu, (b + 1 < B) ? eb[(b + 1) % B] : tail, 0);
            const bool next_in_batch = (b + 1 < B) && (q + 32 * (b + 1) < q1);
            if (lane == 31) nxt = next_in_batch ? first_next : tail;
            if (valid && i + 1 == q1) nxt = tail;                    // last entry of the segment
            const int cnt = !valid ? 0 : (e < 0 ? 1 : (is_idx ? __popc(nxt & 0xF) : 0));
            int tot;
            const int ex = warp_exclusive_scan(cnt, &tot);
            if (WRITE) {
                const long long o = obase + dpos + ex;
                if (valid && e < 0) {
                    out[o] = -e;
                } else if (is_idx) {
                    const unsigned p = (unsigned)nxt & 0xFu;
                    const int b0 = __ffs(p) - 1;
                    int u = 0;
#pragma unroll
                    for (int bb = 0; bb < 4; bb++)
                        if ((p >> bb) & 1u) out[o + u++] = e + S * (bb - b0);
                }
            }
            carry_pat = __shfl_sync(0xffffffffu, is_idx, 31);
            dpos += tot;
            if (q + 32 * (b + 1) >= q1) break;
        }
    }
    return dpos;
}

__global__ void __launch_bounds__(256) cps_expand_kernel(Geom g, const int32_t* __restrict__ ptr,
                                                         const int32_t* __restrict__ in,
                                                         const int64_t* __restrict__ cpo_off,
                                                         const int64_t* __restrict__ cnz_off,
                                                         const int64_t* __restrict__ cin_off,
                                                         int32_t* __restrict__ out,
                                                         const unsigned long long* status) {
    __shared__ int s_cnt[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long nc = blockIdx.x;
    pdl_wait();
    pdl_trigger();
    if (*reinterpret_cast<volatile const unsigned long long*>(status) != 0ull) return;   // flagged encoding
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
    for (int r = threadIdx.x; r < dmid; r += blockDim.x) out[Z + r] = in[Q + r];
    if (dmid == nnz) return;
    // this warp's segment of the overlapK_w entries, and the role of its first entry: the
    // parity of its distance to the start of its run (after the last negative entry, or
    // the block start)
    const int per = (nin - dmid + 7) / 8;
    const int q0 = min(nin, dmid + warp * per), q1 = min(nin, q0 + per);
    int run_start = dmid;
    for (int p = q0; p > dmid;) {
        const int lo = max(dmid, p - 32);
        const int i = lo + lane;
        const int e = (i < p) ? __ldg(in + Q + i) : 0;
        const unsigned neg = __ballot_sync(0xffffffffu, i < p && e < 0);
        if (neg) { run_start = lo + (31 - __clz(neg)) + 1; break; }
        p = lo;
    }
    const bool carry = ((q0 - run_start) & 1) != 0;
    const int cnt = (q0 < q1) ? cps_segment<false>(in, Q, q0, q1, nin, carry, g.S, out, 0) : 0;
    if (lane == 0) s_cnt[warp] = cnt;
    __syncthreads();
    int base = dmid;
    for (int w = 0; w < warp; w++) base += s_cnt[w];
    if (q0 < q1) cps_segment<true>(in, Q, q0, q1, nin, carry, g.S, out, Z + base);
}

// Many small channels (14x14 / 7x7 planes, or batches of thousands of channels): one warp per
// channel, 8 channels per CTA -- the overlapK_w block of such a channel is a few dozen entries,
// so splitting it over 8 warps (above) only added a CTA barrier and a count pass per channel.
__global__ void __launch_bounds__(256) cps_expand_warp_kernel(Geom g, const int32_t* __restrict__ ptr,
                                                              const int32_t* __restrict__ in,
                                                              const int64_t* __restrict__ cpo_off,
                                                              const int64_t* __restrict__ cnz_off,
                                                              const int64_t* __restrict__ cin_off,
                                                              int32_t* __restrict__ out,
                                                              const unsigned long long* status) {
    const int lane = threadIdx.x & 31;
    const long long nc = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
    pdl_wait();
    pdl_trigger();
    if (nc >= g.NC) return;
    if (*reinterpret_cast<volatile const unsigned long long*>(status) != 0ull) return;   // flagged encoding
    const long long Z = cnz_off[nc], Q = cin_off[nc], P = cpo_off[nc];
    const int nnz = (int)(cnz_off[nc + 1] - Z), nin = (int)(cin_off[nc + 1] - Q), plen = (int)(cpo_off[nc + 1] - P);
    if (nnz == 0) return;
    const int e0 = (lane < nin) ? __ldg(in + Q + lane) : 0;   // in flight during the directory parse
    int dmid = nnz;
    if (g.S > 1 && plen <= 64) {
        // the channel's ptr segment in two registers per lane (one round trip), the block
        // directory walked by shuffles: DA start of the overlapK_w block (Alg. 1 layout)
        const int v0 = (lane < plen) ? __ldg(ptr + P + lane) : 0;
        const int v1 = (32 + lane < plen) ? __ldg(ptr + P + 32 + lane) : 0;
        auto seg = [&](int i) {
            const int a0 = __shfl_sync(0xffffffffu, v0, i & 31), a1 = __shfl_sync(0xffffffffu, v1, i & 31);
            return i < 32 ? a0 : a1;
        };
        int p = 0, dacur = 0;
        if (g.pl == 0) {                             // NOP [0, a, a+b]
            dacur = seg(2);
            p = 3;
        }
        for (int t = max(1, g.pl); t <= g.S - 2; t++) {
            if (seg(p + 1) == SPC_NPF) { p += 2; continue; }
            dacur += seg(p + 1 + (g.Ow1 - 1 - t));
            p += 1 + g.Ow1;
        }
        dmid = (seg(p + 1) == SPC_NPF) ? nnz : dacur;
    } else if (g.S > 1) {
        ChanDir d;
        parse_channel(g, ptr, P, d);
        dmid = (d.pos[g.S - 1] >= 0) ? d.da[g.S - 1] : nnz;
    }
    if (lane < dmid) out[Z + lane] = e0;
    for (int r = 32 + lane; r < dmid; r += 32) out[Z + r] = __ldg(in + Q + r);
    if (dmid < nnz) cps_segment<true>(in, Q, dmid, nin, nin, false, g.S, out, Z + dmid);
}

cudaError_t launch_cps_expand(const Geom& g, const spc_encoding* e, int32_t* in_cpo, cudaStream_t st) {
    static const int force = [] { const char* v = getenv("SPC_CPS_EXPAND"); return v ? atoi(v) : 0; }();
    const bool per_warp = force ? force == 1 : (g.H * g.W <= 1024 || g.NC >= 4096);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(per_warp ? (unsigned)((g.NC + 7) / 8)    // one warp per channel
                                : (unsigned)g.NC);              // one CTA (8 warp segments) per channel
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, per_warp ? cps_expand_warp_kernel : cps_expand_kernel, g, (const int32_t*)e->ptr,
                              (const int32_t*)e->in,
                              (const int64_t*)e->chan_ptr_off, (const int64_t*)e->chan_nz_off,
                              (const int64_t*)e->chan_in_off, in_cpo,
                              (const unsigned long long*)(e->lengths + 3));
}

// ------------------------------------------------------------ conv kernels

// Development phase switch (probe build only): 1 = stage/scatter only the first chunk of
// a segment (times the walk alone), 2 = skip the walk, 3 = stage the taps of the first
// chunk only, 4 = scatter the first chunk only.  Always 0 in the product library.
#ifdef SPC_PROBES
__constant__ int g_dev_phase_mode = 0;
__device__ __forceinline__ int dev_phase_mode() { return g_dev_phase_mode; }
#else
__device__ __forceinline__ constexpr int dev_phase_mode() { return 0; }
#endif

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
    int tiles_x;    // generic kernel: tiles per output row
    int cg;         // CTAs per cluster splitting the input channels
    int pmax;       // longest ptr segment of one channel
    int rt;         // strip kernel: row tiles per strip (warps per channel split)
    int csplit;     // strip kernel: channel splits inside the CTA
    float* scratch; // strip kernel: cg > 1 per-CTA partials of the L2 cluster reduction, or
                    // the balanced mode's published partials (or null)
    size_t scratch_bytes;
    unsigned* sk_flags;   // balanced mode: one "partial published" flag per CTA (zeroed after use)
    unsigned long long* status;   // the encoding's overflow word (lengths[3]): nonzero -> y = 0;
                                  // a balanced-mode wait timeout sets bit 2
    unsigned sa_types;            // stride-aware layout: mask of the coverage types present (0 = canonical)
    int cscc;                     // CSCC encoding (SI Alg. 5 layout): ptr = [0, c_0 .. c_{O_w-1}] per channel
    unsigned long long* omask;    // NEXT-1 fused encode: per output column (n, k, x) a bit per output
                                  // row holding an NZE of y (null = off); zeroed by its consumer
    int sk_ctas;          // balanced mode: persistent CTAs (0 = one CTA per unit x cluster rank)
    int sk_strips;        // balanced mode: column strips per image (unit = (k-block, image, strip))
    long long sk_units;   // balanced mode: strips x images x k-blocks
    // CPS decoded inside the warp-specialised conv (Alg. 4): cps_in = the CPS
    // IN stream, cin_off = its per-channel offsets; `in` is then the workspace buffer a chunk too
    // large for the producers' shared-memory stage is decoded into (null: CPO-form `in`)
    const int32_t* __restrict__ cps_in;
    const int64_t* __restrict__ cin_off;
};

// Strip-kernel configuration: a CTA owns a column strip of TX output columns and
// all output rows (rt row tiles of TY rows, one per warp), KPL output channels
// per lane (lane owns kbase + lane*KPL + [0, KPL), adjacent pairs as float2 for
// FFMA2 when KPL is even, so its taps load as one 64/128-bit word), CH input
// channels staged per chunk.
template <int R_, int S_, int SH_, int SW_, int TY_, int TX_, int KPL_, int MINB_ = 2, int MAXW_ = 8, int CH_ = 16,
          bool FLAT_ = false>
struct StripCfg {
    // P1 flattened over the chunk's NZEs across channels (one L2 round trip per chunk) instead
    // of warp per channel: measured faster only where a chunk holds many short channels per
    // warp AND the walk's code generation is unaffected (set per configuration)
    static constexpr bool FLAT = FLAT_;
    static constexpr int MINB = MINB_;   // CTAs per SM targeted by the register budget
    static constexpr int R = R_, S = S_, SH = SH_, SW = SW_, TY = TY_, TX = TX_, KPL = KPL_;
    static constexpr int MAXW = MAXW_, THREADS = 32 * MAXW;
    static constexpr int CH = CH_;        // input channels staged per chunk (fewer chunk barriers when larger)
    static constexpr int CW = 16 * CH;    // channels whose side-table entries are staged at once
    static constexpr int KB = 32 * KPL;               // output channels per CTA
    static constexpr int RS = R * S;
    static constexpr int NACC = KPL * TY * TX;        // accumulators per lane
    static constexpr int WH = (TY - 1) * SH + R;      // input window rows of a row tile
    static constexpr int WW = (TX - 1) * SW + S;      // input window cols of the strip
    static constexpr int NCASE = WH * WW;             // window positions
    static constexpr int MW = (NCASE + 31) / 32;      // 32-bit occupancy words per window
    static constexpr int NCP = 32 * MW;               // dense window slots (floats)
    static constexpr int RSTEP = TY * SH;             // input rows between row tiles
    static constexpr bool PACKED = (KPL % 2) == 0;
    static constexpr int GBH = 4, GBW = 2;            // skip-branch block of window positions
    static constexpr int NP = PACKED ? KPL / 2 : KPL; // accumulator words per position
    static_assert(WW <= 32, "window columns are mapped to lanes");
    static_assert(MW <= 4, "window too large");
};

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ float4 lds128(const float4* p) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}
// NEXT-1 (fused encode): mark the non-zero outputs of a 4-column output row chunk in the
// per-column row masks of y (consumed by encode_from_masks, which re-zeroes them)
__device__ __forceinline__ void emit_omask(unsigned long long* omask, const Geom& g, int n, int k, int oy, int ox0,
                                           const float4& v) {
    if (!omask) return;
    const float sv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; q++)
        if (ox0 + q < g.Ow && sv[q] != 0.0f)
            atomicOr(omask + ((long long)n * g.K + k) * g.Ow + ox0 + q, 1ull << oy);
}

// Balanced mode: wait for CTA b's "partial published" flag, bounded (a co-scheduled grid never
// reaches the bound).  Returns false on a timeout; the kernel reports it (bit 2 of the encoding's
// status word) once, after its segments -- the walk of the balanced strip kernel sits at its
// register cap, and the 64-bit atomic inside the segment loop measurably spilled it.
__device__ __forceinline__ bool sk_wait_flag(const unsigned* flag) {
    unsigned spin = 0;
    while (ld_acquire32(flag) == 0u && ++spin < (1u << 24)) __nanosleep(64);
    return spin < (1u << 24);
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

// One window position P of the replay: the NZE value v (already known to be
// non-zero) times each tap (l, m) whose output (y, x) lies in the row tile and
// on the stride grid; all indices are compile-time constants after unrolling.
template <class T>
__device__ __forceinline__ void tap_fma(int P, float v, float2 (&acc)[T::NP][T::TY][T::TX],
                                        const float2 (&w)[T::NP][T::R][T::S]) {
    const int hr = P / T::WW, wr = P % T::WW;
    const float2 vv = make_float2(v, v);
#pragma unroll
    for (int l = 0; l < T::R; ++l)
#pragma unroll
        for (int m = 0; m < T::S; ++m) {
            const int y1 = hr - l, x1 = wr - m;
            if (y1 >= 0 && x1 >= 0 && (y1 % T::SH) == 0 && (x1 % T::SW) == 0 && y1 / T::SH < T::TY &&
                x1 / T::SW < T::TX) {
#pragma unroll
                for (int p = 0; p < T::NP; ++p)
                    acc[p][y1 / T::SH][x1 / T::SW] = __ffma2_rn(vv, w[p][l][m], acc[p][y1 / T::SH][x1 / T::SW]);
            }
        }
}

template <class T>
__device__ __forceinline__ void tap_fma1(int P, float v, float (&acc)[T::NP][T::TY][T::TX],
                                         const float (&w)[T::NP][T::R][T::S]) {
    const int hr = P / T::WW, wr = P % T::WW;
#pragma unroll
    for (int l = 0; l < T::R; ++l)
#pragma unroll
        for (int m = 0; m < T::S; ++m) {
            const int y1 = hr - l, x1 = wr - m;
            if (y1 >= 0 && x1 >= 0 && (y1 % T::SH) == 0 && (x1 % T::SW) == 0 && y1 / T::SH < T::TY &&
                x1 / T::SW < T::TX) {
#pragma unroll
                for (int p = 0; p < T::NP; ++p)
                    acc[p][y1 / T::SH][x1 / T::SW] = fmaf(v, w[p][l][m], acc[p][y1 / T::SH][x1 / T::SW]);
            }
        }
}

// Balanced mode: work of one input channel of a unit in column strip sx, in column
// equivalents: a fixed part (tap staging, directory) plus the input columns of the
// strip's window that lie inside the map (the NZEs it scatters and walks).
constexpr int kSkBaseWork = 15;   // fitted: a chunk of the 3-column edge strip costs 0.86x (cfg5-L8)
template <class T>
__device__ __forceinline__ int sk_strip_work(const Geom& g, int sx) {
    const int w0 = sx * T::TX * T::SW;
    const int lo = max(w0, g.pl), hi = min(w0 + T::WW, g.pl + g.W);
    return kSkBaseWork + max(0, hi - lo);
}

// First work index (unit * C + channel, units ordered k-block, image, strip) of
// balanced-mode CTA b: where the cumulative work reaches b / sk_ctas of the total.
template <class T>
__device__ int sk_start(const ConvArgs& a, int b) {
    const Geom& g = a.g;
    const long long groups = a.sk_units / a.sk_strips;      // (k-block, image) pairs
    if (b >= a.sk_ctas) return (int)(a.sk_units * g.C);
    long long wsum = 0;
    for (int sx = 0; sx < a.sk_strips; sx++) wsum += sk_strip_work<T>(g, sx);
    const long long per_group = wsum * g.C;
    const long long X = (long long)b * (groups * per_group) / a.sk_ctas;
    const long long grp = X / per_group;
    long long rem = X - grp * per_group;
    int sx = 0;
    for (; sx < a.sk_strips - 1; sx++) {
        const long long ws = (long long)sk_strip_work<T>(g, sx) * g.C;
        if (rem < ws) break;
        rem -= ws;
    }
    const int c = (int)min((long long)g.C - 1, rem / sk_strip_work<T>(g, sx));
    return (int)((grp * a.sk_strips + sx) * g.C + c);
}

// Strip kernel.  CTA = (image n, column strip of TX outputs, KB output
// channels, input-channel range of its cluster rank); warp (r, cs) owns row
// tile r of the strip for the channels cs, cs+csplit, ...  Per chunk of CH
// input channels:
//  P0  stage the chunk's ptr segments (contiguous in the stream), DA offsets and
//      taps W[c][l][m][kbase..+KB) in shared memory (cp.async);
//  P1  one warp per channel: block directory from the staged ptr (NPC / NPF skip),
//      DA ranges of the strip's window columns, then every NZE of those columns
//      (many loads in flight) is scattered into the dense window array of each
//      row tile whose window holds it (1 or 2 tiles);
//  P2  warp (r, cs), per channel: occupancy mask of its window (2 ballots), then
//      a fully unrolled walk over the window positions: a warp-uniform skip
//      branch for empty positions, static FFMA2 taps for the NZEs.  Only NZEs
//      cost multiply-adds (Alg. 2 convSpMv), with no indirect branches.
// Epilogue: reduce the csplit warps of a row tile through smem, then the cg
// CTAs of the cluster through distributed shared memory; ReLU; NKHW store.
template <class T, bool BAL, bool SL = false, bool OM = false>   // SL: stride-aware / CSCC slot parse (P1);
// OM: NEXT-1 output row masks (only the fused conv + encode path carries their atomics)
__global__ void __launch_bounds__(T::THREADS, T::MINB) strip_conv_kernel(ConvArgs a) {
    namespace cgrp = cooperative_groups;
    const Geom& g = a.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nthreads = blockDim.x, nwarps = nthreads >> 5;
    const int RT = a.rt, CS = a.csplit;
    const int rtile = warp % RT, cs = warp / RT;
    const int rank = (a.cg > 1) ? (int)cgrp::this_cluster().block_rank() : 0;
    // current segment: image n, column strip at ox0, k-block at kbase, channels [c_begin, c_end)
    int n = 0, kbase = 0, ox0 = 0, wx0 = 0, c_begin = 0, c_end = 0;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* s_w = reinterpret_cast<float*>(smem_raw);                                  // [CH][RS][KB]
    float* s_val = s_w + T::CH * T::RS * T::KB;                                       // [CH][RT][NCP]
    int* s_ptr = reinterpret_cast<int*>(s_val + T::CH * RT * T::NCP);                 // [2][CH * pmax]
    int* s_coff = s_ptr + 2 * T::CH * a.pmax;       // [CW + 1] window's ptr offsets - cbase
    int* s_cz = s_coff + T::CW + 1;                 // [CW + 1] window's DA offsets - zbase
    int* s_scr = s_cz + T::CW + 1;                  // P1 column tables: [CH][65] (FLAT) or [MAXW][96]

    using AccT = typename std::conditional<T::PACKED, float2, float>::type;
    AccT acc[T::NP][T::TY][T::TX];
    const bool w16 = (g.K % 4) == 0;

    // channels per chunk (P1: warps stride the channels); a chunk slightly larger than the
    // warp count would leave one warp doing two channels' scatter, so trim it then
    const int CHS = (T::CH % nwarps == 0 || T::CH >= 2 * nwarps) ? T::CH : min(T::CH, nwarps);
    // Work.  Default grid: one segment per CTA (blockIdx = strip, k-block, image x cluster
    // rank).  Balanced mode (BAL, a.sk_ctas CTAs, one per resident slot): the units (strip,
    // k-block, image) x Q chunks of CHS channels are cut into equal contiguous ranges, one
    // per CTA; a unit split between CTAs is summed by the CTA holding its first chunk
    // (its last segment) from the partials the others published (their first segment).
    // balanced mode: this CTA's remaining work range [s_seg[0], s_seg[1]) in units of
    // (unit * C + channel); kept in shared memory (read at segment starts only, so it
    // does not hold registers through the walk).  s_seg[0] advances after the first
    // barrier of each segment.
    __shared__ int s_seg[2];
    __shared__ int s_flag;   // the encoding's status word != 0 (read by thread 0, published by a barrier)
    int t_next = 0;
    bool bad = false;
    if constexpr (BAL) {
        if (threadIdx.x == 0) {
            s_seg[0] = sk_start<T>(a, blockIdx.x);
            s_seg[1] = sk_start<T>(a, blockIdx.x + 1);
        }
        __syncthreads();
    }
    auto next_segment = [&](bool first) -> bool {
        if constexpr (BAL) {
            const int t = *reinterpret_cast<volatile int*>(&s_seg[0]);
            const int t1 = *reinterpret_cast<volatile int*>(&s_seg[1]);
            if (t >= t1) return false;
            const int u = t / g.C;
            c_begin = t - u * g.C;
            c_end = min(g.C, c_begin + (t1 - t));
            t_next = t + c_end - c_begin;
            const int sx = u % a.sk_strips, r2 = u / a.sk_strips;
            n = r2 % g.N;
            kbase = (r2 / g.N) * T::KB;
            ox0 = sx * T::TX;
        } else {
            if (!first) return false;
            n = blockIdx.z / a.cg;
            kbase = blockIdx.y * T::KB;
            ox0 = blockIdx.x * T::TX;
            const int cper = (g.C + a.cg - 1) / a.cg;
            c_begin = rank * cper;
            c_end = min(g.C, c_begin + cper);
        }
        wx0 = ox0 * T::SW;
        return true;
    };
    // taps W[c][l][m][kbase..+KB) of a chunk -> s_w (cp.async); independent of the encoding
    auto stage_w = [&](int c0, int chn) {
        const float* wsrc = a.wp + (long long)c0 * T::RS * g.K + kbase;   // row (j*RS+rs) at stride K
        const int rows = chn * T::RS;
        if (w16) {
            constexpr int VPR = T::KB / 4;                 // 16-byte vectors per row
            const int vq = threadIdx.x % VPR, kq = 4 * vq;
            const int nb = max(0, min(16, 4 * (g.K - (kbase + kq))));
            for (int r = threadIdx.x / VPR; r < rows; r += nthreads / VPR)
                cp_async16(s_w + r * T::KB + kq, wsrc + (long long)r * g.K + (nb ? kq : 0), nb);
        } else {
            for (int i = threadIdx.x; i < rows * T::KB; i += nthreads) {
                const int kk = i % T::KB, r = i / T::KB;
                const bool ok = kbase + kk < g.K;
                cp_async4(s_w + i, wsrc + (long long)r * g.K + (ok ? kk : 0), ok ? 4 : 0);
            }
        }
    };
    // Side tables of a window of CW channels (one L2 round trip per window instead of one
    // per chunk) and the ptr segments of the next chunk, prefetched during the walk.
    int cw0 = 0, cw1 = 0;
    long long cbase = 0, zbase = 0;
    // (pub: thread 0 also publishes the encoding's flag word, loaded before the side tables, through
    // the same barrier)
    auto stage_window = [&](int c, bool pub = false, unsigned long long st = 0ull) {
        const long long nc = (long long)n * g.C + c;
        cw0 = c;
        cw1 = min(c_end, c + T::CW);
        cbase = __ldg(a.cpo_off + nc);
        zbase = __ldg(a.cnz_off + nc);
        for (int i = threadIdx.x; i <= cw1 - cw0; i += nthreads) {
            s_coff[i] = (int)(__ldg(a.cpo_off + nc + i) - cbase);
            s_cz[i] = (int)(__ldg(a.cnz_off + nc + i) - zbase);
        }
        if (pub) s_flag = st != 0ull;
        __syncthreads();
    };
    auto stage_ptr = [&](int c0, int chn, int buf) {
        const int r0 = s_coff[c0 - cw0], plen = s_coff[c0 - cw0 + chn] - r0;
        const int32_t* src = a.ptr + cbase + r0;
        int* dst = s_ptr + buf * T::CH * a.pmax;
        for (int i = threadIdx.x; i < plen; i += nthreads) cp_async4(dst + i, src + i, 4);
    };
    // per segment
    for (bool first = true; next_segment(first); first = false) {
#pragma unroll
        for (int p = 0; p < T::NP; p++)
#pragma unroll
            for (int yy = 0; yy < T::TY; yy++)
#pragma unroll
                for (int xx = 0; xx < T::TX; xx++) {
                    if constexpr (T::PACKED) acc[p][yy][xx] = make_float2(0.f, 0.f);
                    else acc[p][yy][xx] = 0.f;
                }
        if (first) {
            // PDL prologue: the first chunk's taps load while the encoder finishes
            probe(0);
            if (c_begin < c_end) stage_w(c_begin, min(CHS, c_end - c_begin));
            probe(1);
            pdl_wait();
            probe(2);
        }
        // An encoding the encoder flagged (capacity overflow / wait timeout) is not read.  Its word is
        // loaded alongside the side tables (in bounds whatever the flag), not ahead of them.
        //  * balanced mode: every CTA sees the same word, writes zeros over each unit it touches and
        //    leaves -- no flag of the balanced mode is waited on, overlapping zero writes are
        //    harmless (a flag carried through the walk spilled the balanced kernel: measured);
        //  * default grid: the chunk loop is skipped and the epilogue writes the zero accumulators
        //    (the early-exit form cost the default kernel ~2 us on cfg3-s2 / cfg4a: measured).
        int buf = 0;
        if constexpr (BAL) {
            unsigned long long st0 = 0ull;
            if (first && threadIdx.x == 0) st0 = *reinterpret_cast<volatile unsigned long long*>(a.status);
            if (c_begin < c_end) {
                stage_window(c_begin, first && threadIdx.x == 0, st0);   // (its barrier orders every thread's read of s_seg before the update)
            } else if (first) {
                if (threadIdx.x == 0) s_flag = st0 != 0ull;
                __syncthreads();
            }
            if (first && (s_flag & 1)) {
                cp_async_wait_all();   // the prologue's tap copies land before the CTA leaves
                for (;;) {
                    const int rows = min(T::KB, g.K - kbase);
                    float* yb0 = a.y + (long long)n * g.K * g.Oh * g.Ow;
                    for (int i = threadIdx.x; i < rows * g.Oh * T::TX; i += nthreads) {
                        const int xx = i % T::TX, r = i / T::TX, oy = r % g.Oh, kk = r / g.Oh;
                        if (ox0 + xx < g.Ow) yb0[((long long)(kbase + kk) * g.Oh + oy) * g.Ow + ox0 + xx] = 0.f;
                    }
                    __syncthreads();
                    if (threadIdx.x == 0) s_seg[0] = t_next;
                    __syncthreads();
                    if (!next_segment(false)) break;
                }
                return;
            }
            if (c_begin < c_end) {
                if (threadIdx.x == 0) s_seg[0] = t_next;
                stage_ptr(c_begin, min(CHS, c_end - c_begin), 0);
            }
        } else {
            unsigned long long st0 = 0ull;
            if (first) st0 = *reinterpret_cast<volatile unsigned long long*>(a.status);
            if (c_begin < c_end) stage_window(c_begin);
            if (st0 != 0ull && !bad) {
                bad = true;
                cp_async_wait_all();   // the prologue's tap copies land before smem is reused
            }
            if (c_begin < c_end && !bad) stage_ptr(c_begin, min(CHS, c_end - c_begin), 0);
        }
        const int c_stop = bad ? c_begin : c_end;
        for (int c0 = c_begin; c0 < c_stop; c0 += CHS, buf ^= 1) {
            const int chn = min(CHS, c_end - c0);
            const bool stage = !(dev_phase_mode() == 1 && !(first && c0 == c_begin));
            // ---- P0: taps (cp.async, with this chunk's prefetched ptr segments in flight); zero the windows
            if (stage) {
                if ((!first || c0 != c_begin) && dev_phase_mode() != 3) stage_w(c0, chn);
                float4* v4 = reinterpret_cast<float4*>(s_val);
                for (int i = threadIdx.x; i < chn * RT * T::NCP / 4; i += nthreads) v4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
                cp_async_wait_all();
            }
            if (stage) __syncthreads();
            if (c0 == c_begin) probe(3);
            // P1 in two instantiations: window columns (canonical CPO) or window SLOTS -- (partition,
            // type) pairs of the stride-aware layout, submatrices of CSCC -- whose NZE column is the
            // slot's base + IN % K_w (so the canonical path keeps its compile-time column bounds)
            auto run_p1 = [&](auto slots_c) {
            if constexpr (T::FLAT) {
                // ---- P1: scatter every NZE of the strip's window columns into its row tiles' windows.
                //      (a) warp per channel: block directory (NPC / NPF skip) and the DA range of each
                //      window column -> per-channel column prefix table; (b) all threads over the
                //      chunk's NZEs flattened across channels, so one L2 round trip covers the chunk.
                const bool scatter = stage && !(dev_phase_mode() == 4 && !(first && c0 == c_begin));
                int* fpre = s_scr;                      // [CH][32] column (slot) prefix within the channel
                int* flo = fpre + T::CH * 32;           // [CH][32] DA offset of the column (slot)
                int* fcb = flo + T::CH * 32;            // [CH][32] slot column base (stride-aware / CSCC; SL only)
                int* ftot = SL ? fcb + T::CH * 32 : fcb; // [CH] NZEs of the channel in the window
                // slots: window columns, or (partition, type) pairs (stride-aware), or submatrices (CSCC)
                const int nsl = !SL ? T::WW
                              : a.cscc ? max(0, min(g.Ow - 1, (wx0 + T::WW - 1) / g.sw) - sa_slot_s_lo(g, wx0) + 1)
                              : sa_nslots(g, wx0, T::WW);
                for (int j = warp; scatter && j < chn; j += nwarps) {
                    const int* seg = s_ptr + buf * T::CH * a.pmax + (s_coff[c0 - cw0 + j] - s_coff[c0 - cw0]);
                    DirS<T::S> d;
                    int lo = 0, hi = 0, cb = 0;
                    if (SL && a.cscc) {
                        if (lane < nsl) {
                            const int s2 = sa_slot_s_lo(g, wx0) + lane;
                            lo = seg[s2];
                            hi = seg[s2 + 1];
                            cb = s2 * g.sw - wx0;
                        }
                    } else if (SL) {
                        parse_dir_sa<T::S>(g, seg, d, a.sa_types);
                        if (!d.npc && lane < nsl) sa_slot_range<T::S>(g, seg, d, wx0, T::WW, lane, lo, hi, cb);
                    } else {
                        parse_dir<T::S>(g, seg, d);
                        if (!d.npc && lane < T::WW) column_range_s<T::S>(g, seg, d, wx0 + lane, lo, hi);   // NPC: skip
                    }
                    int tot;
                    const int pre = warp_exclusive_scan(hi - lo, &tot);
                    fpre[j * 32 + lane] = (lane < nsl) ? pre : (1 << 30);
                    flo[j * 32 + lane] = lo;
                    if constexpr (SL) fcb[j * 32 + lane] = cb;
                    if (lane == 0) ftot[j] = tot;
                }
                if (scatter) __syncthreads();
                if (scatter) {
                    int total;
                    const int cpre = warp_exclusive_scan(lane < chn ? ftot[lane] : 0, &total);
                    constexpr int U = 4;
                    for (int f0 = warp * 32 * U; f0 < total; f0 += nwarps * 32 * U) {
                        int e[U], pos[U];
                        float v[U];
    #pragma unroll
                        for (int u = 0; u < U; u++) {
                            const int f = f0 + 32 * u + lane;
                            // channel: last j with cpre[j] <= f (all lanes shuffle)
                            int j = 0;
    #pragma unroll
                            for (int step = 16; step > 0; step >>= 1) {
                                const int cand = j + step;
                                const int cv = __shfl_sync(0xffffffffu, cpre, cand & 31);
                                if (cand < chn && cv <= f) j = cand;
                            }
                            const int fj = f - __shfl_sync(0xffffffffu, cpre, j);
                            e[u] = -1;
                            v[u] = 0.f;
                            pos[u] = 0;
                            if (f < total) {
                                const int* jp = fpre + j * 32;
                                int jc = 0;
    #pragma unroll
                                for (int step = 16; step > 0; step >>= 1)
                                    if (jc + step < nsl && jp[jc + step] <= fj) jc += step;
                                const long long Z = zbase + s_cz[c0 - cw0 + j];
                                const int idx = flo[j * 32 + jc] + (fj - jp[jc]);
                                e[u] = __ldg(a.in + Z + idx);
                                v[u] = __ldg(a.da + Z + idx);
                                pos[u] = j * RT * T::NCP + jc;
                                if constexpr (SL) {            // window column = slot base + L
                                    const int cc = fcb[j * 32 + jc] + e[u] % T::S;
                                    pos[u] = j * RT * T::NCP + cc;
                                    if (cc < 0 || cc >= T::WW) e[u] = -1;
                                }
                            }
                        }
    #pragma unroll
                        for (int u = 0; u < U; u++) {
                            if (e[u] < 0) continue;
                            const int h = e[u] / T::S;                 // IN = L + h*S with L < S
                            // row tiles whose window [r*RSTEP, r*RSTEP + WH) holds row h (at most 2)
                            const int rhi = min(RT - 1, h / T::RSTEP);
                            const int rlo = (h >= T::WH - 1) ? (h - T::WH + 1 + T::RSTEP - 1) / T::RSTEP : 0;
                            for (int r = rlo; r <= rhi; r++) s_val[pos[u] + r * T::NCP + (h - r * T::RSTEP) * T::WW] = v[u];
                        }
                    }
                }
            } else {
                // ---- P1: scatter every NZE of the strip's window columns into its row tiles' windows
                for (int j = warp; stage && j < chn && !(dev_phase_mode() == 4 && !(first && c0 == c_begin)); j += nwarps) {
                    const int* seg = s_ptr + buf * T::CH * a.pmax + (s_coff[c0 - cw0 + j] - s_coff[c0 - cw0]);
                    DirS<T::S> d;
                    if (SL && a.cscc) d.npc = 0;                          // CSCC: no NPC flag, no blocks
                    else if (SL) parse_dir_sa<T::S>(g, seg, d, a.sa_types);
                    else parse_dir<T::S>(g, seg, d);
                    if (d.npc) continue;                                  // NPC: skip channel
                    int lo = 0, hi = 0, cb = 0;
                    // slots: window columns (canonical layout) or (partition, type) pairs (stride-aware,
                    // CSCC with one "type": submatrix s = partition s)
                    const int nsl = !SL ? T::WW
                                  : a.cscc ? max(0, min(g.Ow - 1, (wx0 + T::WW - 1) / g.sw) - sa_slot_s_lo(g, wx0) + 1)
                                  : sa_nslots(g, wx0, T::WW);
                    if (lane < nsl) {
                        if (SL && a.cscc) {
                            // submatrix s holds [ptr[s], ptr[s+1]) (ptr[0] = 0, channel-cumulative, SI Alg. 5);
                            // an NZE sits at padded column s*s_w + (IN % K_w)
                            const int s2 = sa_slot_s_lo(g, wx0) + lane;
                            lo = seg[s2];
                            hi = seg[s2 + 1];
                            cb = s2 * g.sw - wx0;
                        } else if (SL) {
                            sa_slot_range<T::S>(g, seg, d, wx0, T::WW, lane, lo, hi, cb);
                        } else {
                            column_range_s<T::S>(g, seg, d, wx0 + lane, lo, hi);
                        }
                    }
                    int tot;
                    const int pre = warp_exclusive_scan(hi - lo, &tot);
                    int* spre = s_scr + warp * (SL ? 96 : 64);
                    int* slo = spre + 32;
                    int* scb = spre + 64;
                    spre[lane] = (lane < nsl) ? pre : (1 << 30);
                    slo[lane] = lo;
                    if constexpr (SL) scb[lane] = cb;
                    const int lo0 = __shfl_sync(0xffffffffu, lo, 0);
                    const bool contig = __all_sync(0xffffffffu, lane >= nsl || hi == lo || lo == lo0 + pre);
                    __syncwarp();
                    const long long Z = zbase + s_cz[c0 - cw0 + j];
                    float* win = s_val + j * RT * T::NCP;
                    constexpr int U = 4;
                    for (int f0 = 0; f0 < tot; f0 += 32 * U) {
                        int e[U], col[U];
                        float v[U];
    #pragma unroll
                        for (int u = 0; u < U; u++) {
                            const int f = f0 + 32 * u + lane;
                            e[u] = -1;
                            v[u] = 0.f;
                            col[u] = 0;
                            if (f < tot) {
                                int jc = 0;
    #pragma unroll
                                for (int step = 16; step > 0; step >>= 1)
                                    if (jc + step < nsl && spre[jc + step] <= f) jc += step;
                                col[u] = jc;
                                const int idx = contig ? lo0 + f : slo[jc] + (f - spre[jc]);
                                e[u] = __ldg(a.in + Z + idx);
                                v[u] = __ldg(a.da + Z + idx);
                                if constexpr (SL) {            // window column = partition base + L
                                    col[u] = scb[jc] + e[u] % T::S;
                                    if (col[u] < 0 || col[u] >= T::WW) e[u] = -1;
                                }
                            }
                        }
    #pragma unroll
                        for (int u = 0; u < U; u++) {
                            if (e[u] < 0) continue;
                            const int h = e[u] / T::S;                 // IN = L + h*S with L < S
                            // row tiles whose window [r*RSTEP, r*RSTEP + WH) holds row h (at most 2)
                            const int rhi = min(RT - 1, h / T::RSTEP);
                            const int rlo = (h >= T::WH - 1) ? (h - T::WH + 1 + T::RSTEP - 1) / T::RSTEP : 0;
                            for (int r = rlo; r <= rhi; r++) win[r * T::NCP + (h - r * T::RSTEP) * T::WW + col[u]] = v[u];
                        }
                    }
                }
            }
            };
            // (a compile-time choice: the canonical kernel does not carry the slot parse's registers)
            run_p1(std::integral_constant<bool, SL>{});
            if (stage) __syncthreads();
            if (c0 == c_begin) probe(4);
            // prefetch the next chunk's ptr segments (its buffer was last read before the barrier)
            if (c0 + CHS < c_end && stage) {
                const int cn = c0 + CHS, chnn = min(CHS, c_end - cn);
                if (cn + chnn > cw1) stage_window(cn);
                stage_ptr(cn, chnn, buf ^ 1);
                asm volatile("cp.async.commit_group;\n" ::: "memory");
            }
            // ---- P2: unrolled walk over the window positions of this warp's row tile
            for (int j = cs; j < chn && dev_phase_mode() != 2; j += CS) {
                const float* win = s_val + (j * RT + rtile) * T::NCP;
                unsigned mw[T::MW];
                bool any = false;
#pragma unroll
                for (int q = 0; q < T::MW; q++) {
                    mw[q] = __ballot_sync(0xffffffffu, win[32 * q + lane] != 0.0f);
                    any |= mw[q] != 0;
                }
                if (!any) continue;
                using WT = typename std::conditional<T::PACKED, float2, float>::type;
                // lane owns output channels kbase + lane*KPL + [0, KPL): its taps are contiguous
                // in s_w (one 64/128-bit load per tap)
                WT w[T::NP][T::R][T::S];
#pragma unroll
                for (int l = 0; l < T::R; l++)
#pragma unroll
                    for (int m = 0; m < T::S; m++) {
                        const float* ws = s_w + (j * T::RS + l * T::S + m) * T::KB + lane * T::KPL;
                        if constexpr (T::PACKED && T::KPL % 4 == 0) {
#pragma unroll
                            for (int p = 0; p < T::NP; p += 2) {
                                const float4 q4 = *reinterpret_cast<const float4*>(ws + 2 * p);
                                w[p][l][m] = make_float2(q4.x, q4.y);
                                w[p + 1][l][m] = make_float2(q4.z, q4.w);
                            }
                        } else if constexpr (T::PACKED) {
#pragma unroll
                            for (int p = 0; p < T::NP; p++) w[p][l][m] = *reinterpret_cast<const float2*>(ws + 2 * p);
                        } else {
#pragma unroll
                            for (int p = 0; p < T::NP; p++) w[p][l][m] = ws[p];
                        }
                    }
                // hierarchical walk: a warp-uniform branch skips each empty group of 4
                // consecutive window positions, then one per set position
                const float4* w4 = reinterpret_cast<const float4*>(win);
                constexpr int NQ = (T::NCASE + 3) / 4;
                float4 vn = lds128(w4);                      // prefetch: issued ahead of each skip branch
#pragma unroll
                for (int q = 0; q < NQ; q++) {
                    const unsigned nib = (mw[q >> 3] >> ((q & 7) * 4)) & 0xFu;
                    const float4 v4 = vn;
                    if (q + 1 < NQ) vn = lds128(w4 + q + 1);
                    if (nib) {
                        const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const int P = 4 * q + u;
                            if (P < T::NCASE && ((nib >> u) & 1u)) {
                                if constexpr (T::PACKED) tap_fma<T>(P, vv[u], acc, w);
                                else tap_fma1<T>(P, vv[u], acc, w);
                            }
                        }
                    }
                }
            }
            __syncthreads();
        }

        probe(5);
        // default grid: the next kernel may launch now (it waits for this grid's completion before
        // reading anything written here; its CTAs start on SMs this grid leaves idle)
        if constexpr (!BAL) pdl_trigger();
        // ---- epilogue: reduce the csplit warps of each row tile; partial -> part
        //      part = [RT*KB rows][TT positions], 16-byte chunks swizzled by (row & (NCH-1))
        //      so the lane-per-row float4 stores and the chunk-per-thread reads are conflict-free
        constexpr int TT = T::TY * T::TX, NCH = TT / 4;
        static_assert(T::TX == 4 && (TT & (TT - 1)) == 0 && (T::KB & (T::KB - 1)) == 0, "tile layout");
        float accf[T::NACC];   // index kk*TT + t
#pragma unroll
        for (int p = 0; p < T::NP; p++)
#pragma unroll
            for (int t = 0; t < TT; t++) {
                if constexpr (T::PACKED) {
                    accf[(2 * p) * TT + t] = acc[p][t / T::TX][t % T::TX].x;
                    accf[(2 * p + 1) * TT + t] = acc[p][t / T::TX][t % T::TX].y;
                } else {
                    accf[p * TT + t] = acc[p][t / T::TX][t % T::TX];
                }
            }
        float4* part4 = reinterpret_cast<float4*>(s_w);   // [RT*KB][NCH]
        float* yb = a.y + (long long)n * g.K * g.Oh * g.Ow;
        const bool vec_ok = (g.Ow % 4) == 0;
        if (CS > 1) {
            float4* red4 = part4 + RT * T::KB * NCH;       // [CS-1][RT][NACC/4][32]
            if (cs > 0) {
#pragma unroll
                for (int i = 0; i < T::NACC / 4; i++)
                    red4[(((cs - 1) * RT + rtile) * (T::NACC / 4) + i) * 32 + lane] =
                        make_float4(accf[4 * i], accf[4 * i + 1], accf[4 * i + 2], accf[4 * i + 3]);
            }
            __syncthreads();
            if (cs == 0) {
                for (int q = 1; q < CS; q++) {
#pragma unroll
                    for (int i = 0; i < T::NACC / 4; i++) {
                        const float4 v = red4[(((q - 1) * RT + rtile) * (T::NACC / 4) + i) * 32 + lane];
                        accf[4 * i] += v.x; accf[4 * i + 1] += v.y; accf[4 * i + 2] += v.z; accf[4 * i + 3] += v.w;
                    }
                }
            }
        }
        if (a.cg == 1) {
            // no cluster split: store straight from registers (a lane owns output channel
            // kk*32+lane and a 4-wide output row per accumulator chunk).  With a cluster split
            // the L2 (or, without scratch, DSMEM) reduction below wins: measured,
            // red.global.add.v4 of every rank's partial costs 8x the transactions and is
            // slower at cfg2/cfg3.
            auto emit = [&](bool add) {
#pragma unroll
                for (int i = 0; i < T::NACC / 4; i++) {
                    const int k = kbase + lane * T::KPL + (i / NCH), oy = rtile * T::TY + (i % NCH);
                    if (k >= g.K || oy >= g.Oh) continue;
                    float4 v = make_float4(accf[4 * i], accf[4 * i + 1], accf[4 * i + 2], accf[4 * i + 3]);
                    if (a.relu) { v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f); }
                    if constexpr (OM) emit_omask(a.omask, g, n, k, oy, ox0, v);
                    float* dst = yb + ((long long)k * g.Oh + oy) * g.Ow + ox0;
                    if (vec_ok && ox0 + 3 < g.Ow) {
                        if (add)
                            asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
                                         ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
                        else
                            *reinterpret_cast<float4*>(dst) = v;
                    } else {
                        const float sv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int q = 0; q < 4; q++)
                            if (ox0 + q < g.Ow) {
                                if (add) atomicAdd(dst + q, sv[q]);
                                else dst[q] = sv[q];
                            }
                    }
                }
            };
            if (!BAL || (c_begin == 0 && c_end == g.C)) {   // whole unit
            if (cs == 0) emit(false);
        } else if constexpr (BAL) {
            const int rows = RT * T::KB;
            float4* part = reinterpret_cast<float4*>(a.scratch);     // [sk_ctas][NCH][rows]
            if (c_begin > 0) {
                // not the unit's first channel: this is the CTA's first segment; publish it
                float4* mine = part + (long long)blockIdx.x * rows * NCH;
                if (cs == 0) {
#pragma unroll
                    for (int i = 0; i < T::NACC / 4; i++)
                        __stcg(mine + (i % NCH) * rows + rtile * T::KB + (i / NCH) * 32 + lane,
                               make_float4(accf[4 * i], accf[4 * i + 1], accf[4 * i + 2], accf[4 * i + 3]));
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    __threadfence();
                    st_release32(a.sk_flags + blockIdx.x, 1u);
                }
            } else {
                // the unit's first channel: the CTA's last segment.  The rest of the unit is the
                // first segment of the next non-empty CTA(s) whose ranges start before its end.
                const int uend = s_seg[0] - c_end + g.C;   // s_seg[0] = this segment's end
                if (threadIdx.x == 0) {
                    int sb = sk_start<T>(a, blockIdx.x + 1);
                    for (int b = blockIdx.x + 1; b < a.sk_ctas && sb < uend; b++) {
                        const int sn = sk_start<T>(a, b + 1);
                        if (sn > sb && !sk_wait_flag(a.sk_flags + b)) s_flag |= 2;   // bounded; reported below
                        sb = sn;
                    }
                }
                __syncthreads();
                if (cs == 0) {
                    int sb = sk_start<T>(a, blockIdx.x + 1);
                    for (int b = blockIdx.x + 1; b < a.sk_ctas && sb < uend; b++) {
                        const int sn = sk_start<T>(a, b + 1);
                        if (sn > sb) {
                            const float4* src = part + (long long)b * rows * NCH;
#pragma unroll
                            for (int i = 0; i < T::NACC / 4; i++) {
                                const float4 v = __ldcg(src + (i % NCH) * rows + rtile * T::KB + (i / NCH) * 32 + lane);
                                accf[4 * i] += v.x; accf[4 * i + 1] += v.y; accf[4 * i + 2] += v.z; accf[4 * i + 3] += v.w;
                            }
                        }
                        sb = sn;
                    }
                    emit(false);
                }
                if (threadIdx.x == 0) {   // consumed: leave the flags zeroed for the next launch
                    int sb = sk_start<T>(a, blockIdx.x + 1);
                    for (int b = blockIdx.x + 1; b < a.sk_ctas && sb < uend; b++) {
                        a.sk_flags[b] = 0u;
                        sb = sk_start<T>(a, b + 1);
                    }
                }
            }
        }
        __syncthreads();   // the epilogue's smem (aliasing the taps) is reused by the next segment
            continue;
        }
        if (a.scratch) {
            // cluster split, reduced through L2: each CTA stores its partial ([NCH][RT*KB] float4,
            // coalesced along rows), one cluster barrier (release / acquire) publishes them, then
            // each rank sums its share of the chunks over the cg partials (L2 reads, all peers'
            // loads in flight).  Measured: DSMEM moves this traffic ~10x slower on this part
            // (tools/microbench/dsmem.cu).
            const int rows = RT * T::KB;
            const long long slot0 = ((long long)(blockIdx.z - rank) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
            const long long sstride = (long long)gridDim.y * gridDim.x;       // next cluster rank
            float4* mine = reinterpret_cast<float4*>(a.scratch) + (slot0 + rank * sstride) * (long long)rows * NCH;
            if (cs == 0) {
#pragma unroll
                for (int i = 0; i < T::NACC / 4; i++) {
                    const int row = rtile * T::KB + (i / NCH) * 32 + lane, c = i % NCH;
                    mine[(long long)c * rows + row] = make_float4(accf[4 * i], accf[4 * i + 1], accf[4 * i + 2], accf[4 * i + 3]);
                }
            }
            probe(6);
            cgrp::this_cluster().sync();
            probe(7);
            const int total = rows * NCH;
            const int per = (total + a.cg - 1) / a.cg;
            const float4* base = reinterpret_cast<const float4*>(a.scratch) + slot0 * (long long)rows * NCH;
            const long long pstride = sstride * (long long)rows * NCH;
            for (int ci = rank * per + threadIdx.x; ci < min(total, (rank + 1) * per); ci += nthreads) {
                float4 v[8];
#pragma unroll
                for (int r = 0; r < 8; r++) v[r] = (r < a.cg) ? __ldcg(base + r * pstride + ci) : make_float4(0.f, 0.f, 0.f, 0.f);
                float4 sum = v[0];
#pragma unroll
                for (int r = 1; r < 8; r++) { sum.x += v[r].x; sum.y += v[r].y; sum.z += v[r].z; sum.w += v[r].w; }
                if (a.relu) { sum.x = fmaxf(sum.x, 0.f); sum.y = fmaxf(sum.y, 0.f); sum.z = fmaxf(sum.z, 0.f); sum.w = fmaxf(sum.w, 0.f); }
                const int c = ci / rows, row = ci % rows, kl = row & (T::KB - 1);   // kl = j*32 + lane
                const int k = kbase + (kl & 31) * T::KPL + (kl >> 5), oy = (row / T::KB) * T::TY + c;
                if (k >= g.K || oy >= g.Oh) continue;
                if constexpr (OM) emit_omask(a.omask, g, n, k, oy, ox0, sum);
                float* dst = yb + ((long long)k * g.Oh + oy) * g.Ow + ox0;
                if (vec_ok && ox0 + 3 < g.Ow) {
                    *reinterpret_cast<float4*>(dst) = sum;
                } else {
                    const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if (ox0 + q < g.Ow) dst[q] = sv[q];
                }
            }
            probe(9);
            probe(8);
            return;
        }
        if (cs == 0) {
#pragma unroll
            for (int i = 0; i < T::NACC / 4; i++) {
                const int row = rtile * T::KB + (i / NCH) * 32 + lane, c = i % NCH;
                part4[row * NCH + (c ^ (row & (NCH - 1)))] =
                    make_float4(accf[4 * i], accf[4 * i + 1], accf[4 * i + 2], accf[4 * i + 3]);
            }
        }
        probe(6);
        if (a.cg > 1) cgrp::this_cluster().sync(); else __syncthreads();
        probe(7);
        // ---- sum the cluster's partials (DSMEM, all peers' float4 loads in flight), ReLU,
        //      NKHW store (a chunk = 4 consecutive output columns of one row)
        const int total = RT * T::KB * NCH;
        const int per = (total + a.cg - 1) / a.cg;
        const int i0 = rank * per, i1 = min(total, i0 + per);
        auto cl = cgrp::this_cluster();
        const float4* peer[8];
#pragma unroll
        for (int r = 0; r < 8; r++) peer[r] = (a.cg > 1 && r < a.cg) ? cl.map_shared_rank(part4, r) : part4;
        for (int ci = i0 + threadIdx.x; ci < i1; ci += nthreads) {
            const int row = ci / NCH, c = ci % NCH;
            const int sidx = row * NCH + (c ^ (row & (NCH - 1)));
            float4 v[8];
#pragma unroll
            for (int r = 0; r < 8; r++) v[r] = (r < a.cg) ? peer[r][sidx] : make_float4(0.f, 0.f, 0.f, 0.f);
            float4 sum = v[0];
#pragma unroll
            for (int r = 1; r < 8; r++) { sum.x += v[r].x; sum.y += v[r].y; sum.z += v[r].z; sum.w += v[r].w; }
            if (a.relu) { sum.x = fmaxf(sum.x, 0.f); sum.y = fmaxf(sum.y, 0.f); sum.z = fmaxf(sum.z, 0.f); sum.w = fmaxf(sum.w, 0.f); }
            const int kl = row & (T::KB - 1), rr = row / T::KB;   // kl = j*32 + lane
            const int k = kbase + (kl & 31) * T::KPL + (kl >> 5), oy = rr * T::TY + c;   // chunk c = output row c
            if (k >= g.K || oy >= g.Oh) continue;
            if constexpr (OM) emit_omask(a.omask, g, n, k, oy, ox0, sum);
            float* dst = yb + ((long long)k * g.Oh + oy) * g.Ow + ox0;
            if (vec_ok && ox0 + 3 < g.Ow) {
                *reinterpret_cast<float4*>(dst) = sum;
            } else {
                const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
                for (int q = 0; q < 4; q++)
                    if (ox0 + q < g.Ow) dst[q] = sv[q];
            }
        }
        probe(9);
        if (a.cg > 1) cl.sync();
        probe(8);
    }
    if constexpr (BAL) {   // a balanced-mode wait that timed out (thread 0 set bit 1 of s_flag)
        if (threadIdx.x == 0 && (s_flag & 2)) atomicOr(a.status, 4ull);
    }
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
    pdl_wait();
    const bool bad = *reinterpret_cast<volatile unsigned long long*>(a.status) != 0ull;   // flagged: y = 0
    for (int c = warp; c < g.C && !bad; c += kGenWarps) {
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
        if (a.omask && s != 0.0f) atomicOr(a.omask + ((long long)n * g.K + kk) * g.Ow + ox, 1ull << oy);
        a.y[(((long long)n * g.K + kk) * g.Oh + oy) * g.Ow + ox] = s;
    }
}

template <class T>
static size_t strip_smem(const ConvArgs& a) {
    const int RT = a.rt, CS = a.csplit;
    const bool slots = a.sa_types || a.cscc;   // the slot layouts' P1 keeps a column-base table too
    const size_t scr = T::FLAT ? (size_t)T::CH * (slots ? 97 : 65) : (size_t)T::MAXW * (slots ? 96 : 64);
    const size_t main = (size_t)T::CH * T::RS * T::KB * 4 + (size_t)T::CH * RT * T::NCP * 4 +
                        (size_t)2 * T::CH * a.pmax * 4 + (size_t)2 * (T::CW + 1) * 4 + scr * 4;
    const size_t epi = (size_t)RT * T::KB * (T::TY * T::TX) * 4 +
                       (CS > 1 ? (size_t)(CS - 1) * RT * T::NACC * 32 * 4 : 0);
    return std::max(main, epi);
}

// Channel split across a cluster: the largest cg in {1,2,4,8} that keeps the
// grid within ~one wave of resident CTAs and at least 8 channels per CTA.
// Cluster split of the input channels: the largest cg in {2, 4, 8} whose grid still fits
// one wave, with >= 2 channels per CTA (cfg1, C = 16: cg 8 steps in 18.6 us vs 20.5 at cg 2;
// a floor of 8 channels per CTA used to hold it at 2).
static int pick_cg(long long ctas, int C, int per_sm) {
    int best = 1;
    for (int cg = 2; cg <= 8; cg *= 2)
        if (ctas * cg <= 148LL * per_sm && C >= 2 * cg) best = cg;
    return best;
}

// Development override: SPC_TUNE="<cg>" forces the cluster split.
static int tune_cg() {
    static const char* env = getenv("SPC_TUNE");
    return env ? atoi(env) : 0;
}

// The launch geometry of a strip config: strips, k-blocks, row tiles, cluster split.
template <class T>
struct StripPlan {
    int strips, kblocks, rt, csplit, cg;
    long long ctas;
    size_t scratch_bytes;   // L2 partials: cluster split (cg > 1) or balanced mode, whichever is larger
    size_t sk_slot_bytes;   // balanced mode: one CTA's published partial
};

// Balanced mode: at most kSkMaxCtas persistent CTAs (resident slots), one flag each at
// the head of the conv scratch region.
constexpr int kSkMaxCtas = 320;
constexpr size_t kSkFlagBytes = ((kSkMaxCtas * sizeof(unsigned)) + 255) / 256 * 256;

// Development override: SPC_BALANCE=0 disables the balanced mode.
static bool balance_enabled() {
    static const char* env = getenv("SPC_BALANCE");
    return !env || atoi(env) != 0;
}

static int sm_count() { return device_sm_count(); }
template <class T>
static StripPlan<T> plan_strip(const Geom& g) {
    StripPlan<T> p;
    p.strips = (g.Ow + T::TX - 1) / T::TX;
    p.rt = (g.Oh + T::TY - 1) / T::TY;
    p.csplit = std::max(1, T::MAXW / std::max(1, p.rt));
    p.kblocks = (g.K + T::KB - 1) / T::KB;
    p.ctas = (long long)p.strips * p.kblocks * g.N;
    int cg = tune_cg();
    if (cg <= 0) cg = pick_cg(p.ctas, g.C, T::MINB);
    p.cg = cg;
    p.sk_slot_bytes = (size_t)p.rt * T::KB * (T::TY * T::TX) * sizeof(float);
    p.scratch_bytes = std::max((cg > 1) ? (size_t)p.ctas * cg * p.sk_slot_bytes : 0,
                               (cg == 1) ? (size_t)kSkMaxCtas * p.sk_slot_bytes : 0);
    return p;
}

template <class T, bool BAL, bool SL, bool OM = false>
static cudaError_t launch_strip(const ConvArgs& a, dim3 grid, int cg, size_t smem, cudaStream_t st) {
    static std::atomic<size_t> attr_bytes[kMaxDevices];     // per instantiation and device
    {
        cudaError_t err = ensure_smem_attr((const void*)strip_conv_kernel<T, BAL, SL, OM>, smem, attr_bytes);
        if (err != cudaSuccess) return err;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(32 * a.rt * a.csplit);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[3];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = cg;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    // PDL (the prologue overlaps the encoder's tail) gains 1-3 us on most layers, but two
    // kinds of grid placed early next to a full encoder grid lose: an 8-CTA-cluster grid
    // larger than the SM count (cfg3 s2: 50.3 vs 36.9 us per step, measured with and
    // without) and the balanced mode at one persistent CTA per SM (its equal-work ranges
    // assume equal start times; cfg5-L0 216 vs 213 us, L1 248 vs 246).  Those launch after
    // the encoder instead.
    const long long ctas = (long long)grid.x * grid.y * grid.z;
    const bool pdl = !(cg >= 8 && ctas > sm_count()) && !(BAL && ctas <= sm_count());
    cfg.numAttrs = pdl ? 2 : 1;
    if (BAL && cooperative_launches()) {
        // the balanced mode's CTAs wait on one another: co-scheduled grid (cluster size 1 here)
        attr[cfg.numAttrs].id = cudaLaunchAttributeCooperative;
        attr[cfg.numAttrs].val.cooperative = 1;
        cfg.numAttrs++;
    }
    return cudaLaunchKernelEx(&cfg, strip_conv_kernel<T, BAL, SL, OM>, a);
}

template <class T>
static cudaError_t run_strip(ConvArgs& a, cudaStream_t st) {
    const Geom& g = a.g;
    const StripPlan<T> pl = plan_strip<T>(g);
    const int strips = pl.strips, kblocks = pl.kblocks, cg = pl.cg;
    a.rt = pl.rt;
    if (a.rt > T::MAXW) return cudaErrorNotSupported;          // the generic kernel runs instead
    a.csplit = pl.csplit;
    a.cg = cg;
    const size_t smem = strip_smem<T>(a);
    if (smem > 227 * 1024) return cudaErrorNotSupported;      // (very wide maps: long ptr segments)
    // Balanced mode when the units outnumber the SMs and the busiest SM would get >= 20%
    // more units than the average (a CTA's time changes little with a second co-resident
    // CTA, so the SM holding the most units sets the kernel time): one CTA per resident
    // slot, equal-work channel ranges.  Measured at batch 32 (cfg5): -10..-13% at skew 1.32
    // (L0, L3), -5% (L4); at skew 1.16 between -5% (L7) and +4% (L12), hence the threshold.
    // Re-measured on the round-2 kernel at skew 1.32 (conv us, balanced vs default grid, each
    // layer's own density): L0 196.6 vs 204.8, L1 231.6 vs 249.9, L6 184.3 vs 196.6, L2 137.3 vs
    // 133.1, L5 131.1 vs 129.0 (at rho 0.05 / 0.1 L0 and L4 lose ~5 %): the threshold stays.
    a.sk_ctas = 0;
    a.sk_strips = strips;
    a.sk_units = pl.ctas;
    const int nsm = sm_count();
    const double skew = (double)((pl.ctas + nsm - 1) / nsm) * nsm / (double)pl.ctas;
    const bool slots = a.sa_types || a.cscc;   // slot layouts: no balanced mode (one fewer instantiation)
    const bool om = a.omask != nullptr;          // fused encode: no balanced mode either
    if (!slots && !om && cg == 1 && a.scratch && a.sk_flags && balance_enabled() && pl.ctas > nsm && skew >= 1.2) {
        int occ = 0;
        if (cudaFuncSetAttribute(strip_conv_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, strip_conv_kernel<T, true>, 32 * a.rt * a.csplit, smem) != cudaSuccess) {
            (void)cudaGetLastError();   // not sticky: fall back to the default grid
            occ = 0;
        }
        const long long P = (long long)occ * nsm;
        if (P > 0 && P <= kSkMaxCtas && pl.ctas * g.C < (1LL << 31) && a.scratch_bytes >= (size_t)P * pl.sk_slot_bytes)
            a.sk_ctas = (int)P;
    }
    if (!a.sk_ctas && (cg <= 1 || a.scratch_bytes < pl.scratch_bytes)) a.scratch = nullptr;
    if (getenv("SPC_PLAN_DEBUG"))
        fprintf(stderr, "strip plan: units %lld strips %d kblocks %d rt %d csplit %d cg %d sk_ctas %d smem %zu\n",
                pl.ctas, strips, kblocks, a.rt, a.csplit, cg, a.sk_ctas, smem);
    if (a.sk_ctas) return launch_strip<T, true, false>(a, dim3(a.sk_ctas, 1, 1), 1, smem, st);
    if (slots) return launch_strip<T, false, true>(a, dim3(strips, kblocks, g.N * cg), cg, smem, st);
    if (om) return launch_strip<T, false, false, true>(a, dim3(strips, kblocks, g.N * cg), cg, smem, st);
    return launch_strip<T, false, false>(a, dim3(strips, kblocks, g.N * cg), cg, smem, st);
}

// Calls f(StripCfg<...>{}) for the strip configuration of this geometry; returns
// cudaErrorNotSupported when none applies (the generic kernel runs instead).
template <class F>
static cudaError_t visit_strip_cfg(const Geom& g, F&& f) {
    if (g.R == 3 && g.S == 3 && g.sh == 1 && g.sw == 1) {
        if (g.K <= 32 && g.Oh <= 64) return f(StripCfg<3, 3, 1, 1, 8, 4, 1, 1, 16, 32>{});
        if (g.K <= 64 && g.Oh <= 64) return f(StripCfg<3, 3, 1, 1, 8, 4, 2, 1, 16, 32, true>{});
        if (g.Oh <= 32) return f(StripCfg<3, 3, 1, 1, 4, 4, 4, 2, 8, 8>{});   // CH 8: CH 16 spills at 128 registers (L4 139 vs 147 us)
        if (g.Oh <= 64) return f(StripCfg<3, 3, 1, 1, 8, 4, 4, 1>{});
        if (g.Oh <= 128) return f(StripCfg<3, 3, 1, 1, 8, 4, 2, 1, 16, 16, true>{});   // up to 16 row tiles
    } else if (g.R == 5 && g.S == 5 && g.sh == 1 && g.sw == 1 && g.Oh <= 64) {
        return f(StripCfg<5, 5, 1, 1, 4, 4, 2, 1, 16, 16>{});
    } else if (g.R == 1 && g.S == 3 && g.sh == 1 && g.sw == 1 && g.Oh <= 32) {
        return f(StripCfg<1, 3, 1, 1, 4, 4, 4>{});
    } else if (g.R == 3 && g.S == 1 && g.sh == 1 && g.sw == 1 && g.Oh <= 32) {
        return f(StripCfg<3, 1, 1, 1, 4, 4, 4>{});
    } else if (g.R == 3 && g.S == 3 && g.sh == 2 && g.sw == 2) {
        if (g.K <= 64 && g.Oh <= 32) return f(StripCfg<3, 3, 2, 2, 4, 4, 2>{});
        if (g.Oh <= 16) return f(StripCfg<3, 3, 2, 2, 4, 4, 4, 2, 8, 16>{});
        if (g.Oh <= 32) return f(StripCfg<3, 3, 2, 2, 4, 4, 4, 2, 8, 8>{});   // 8: keeps 2 CTAs/SM
        if (g.Oh <= 64) return f(StripCfg<3, 3, 2, 2, 4, 4, 2, 1, 16, 16>{});  // up to 16 row tiles
    } else if (g.R == 1 && g.S == 7 && g.sh == 1 && g.sw == 1 && g.Oh <= 64) {
        return f(StripCfg<1, 7, 1, 1, 8, 4, 2, 2, 8, 16, true>{});
    } else if (g.R == 7 && g.S == 1 && g.sh == 1 && g.sw == 1 && g.Oh <= 64) {
        return f(StripCfg<7, 1, 1, 1, 8, 4, 2, 2, 8, 16, true>{});
    }
    return cudaErrorNotSupported;
}

#include "ws_conv.cuh"
#include "tile_conv.cuh"

static bool conv_v1_forced() {   // development A/B: SPC_CONV_V1=1 runs the round-1 strip kernel
    static const char* env = getenv("SPC_CONV_V1");
    return env && atoi(env) != 0;
}

size_t conv_scratch_bytes(const Geom& g) {
    size_t bytes = 0;
    visit_strip_cfg(g, [&](auto cfg) {
        bytes = plan_strip<decltype(cfg)>(g).scratch_bytes;
        return cudaSuccess;
    });
    const int pmax = (g.S == 1) ? (1 + g.Ow1) : (3 + (g.S - 1) * (1 + g.Ow1));
    visit_ws_cfg(g, [&](auto cfg) {
        WsPlan<decltype(cfg)> p;
        if (plan_ws<decltype(cfg)>(g, pmax, p)) bytes = std::max(bytes, p.scratch_bytes);
        return cudaSuccess;
    });
    return bytes ? kSkFlagBytes + bytes : 0;
}

// which kernel the calling thread's last sparse-conv launch ran (3 register-tiled, 2 warp-specialised, 1 strip,
// 0 generic, -1 none yet): reported by spc_last_conv_kernel() for benchmarks and tests
static thread_local int t_last_conv_kernel = -1;
int last_conv_kernel() { return t_last_conv_kernel; }

cudaError_t launch_sparse_conv(const Geom& g, const spc_encoding* e, const int32_t* in_override,
                               const float* w_packed, float* y, int relu, float* scratch, size_t scratch_bytes,
                               cudaStream_t st, unsigned long long* omask, unsigned sa_types, int cscc,
                               bool cps_inline) {
    ConvArgs a;
    a.cps_in = cps_inline ? e->in : nullptr;
    a.cin_off = cps_inline ? e->chan_in_off : nullptr;
    a.g = g;
    a.ptr = e->ptr;
    a.da = e->da;
    a.in = in_override ? in_override : e->in;
    a.cpo_off = e->chan_ptr_off;
    a.cnz_off = e->chan_nz_off;
    a.wp = w_packed;
    a.y = y;
    a.relu = relu;
    a.status = reinterpret_cast<unsigned long long*>(e->lengths + 3);
    a.omask = omask;
    a.sa_types = sa_types;
    a.cscc = cscc;
    a.tiles_x = 1;
    a.cg = 1;
    a.rt = 1;
    a.csplit = 1;
    // scratch = [balanced-mode flags][partials]
    a.sk_flags = nullptr;
    a.scratch = nullptr;
    a.scratch_bytes = 0;
    a.sk_ctas = 0;
    a.sk_strips = 1;
    a.sk_units = 0;
    if (scratch && scratch_bytes > kSkFlagBytes) {
        a.sk_flags = reinterpret_cast<unsigned*>(scratch);
        a.scratch = scratch + kSkFlagBytes / sizeof(float);
        a.scratch_bytes = scratch_bytes - kSkFlagBytes;
    }
    a.pmax = (g.S == 1) ? (1 + g.Ow1) : (3 + (g.S - 1) * (1 + g.Ow1));
    if (sa_types || cscc) a.pmax = std::max(a.pmax, g.S * (1 + g.Ow));
    cudaError_t err = cudaErrorNotSupported;
    if (!conv_v1_forced() && !cps_inline) err = visit_tc_cfg(g, [&](auto cfg) { return run_tc<decltype(cfg)>(a, st); });
    if (err != cudaErrorNotSupported) {
        t_last_conv_kernel = 3;
        return err;
    }
    if (!conv_v1_forced()) err = visit_ws_cfg(g, [&](auto cfg) { return run_ws<decltype(cfg)>(a, st); });
    if (err != cudaErrorNotSupported) {
        t_last_conv_kernel = 2;
        return err;
    }
    if (cps_inline) return cudaErrorNotSupported;   // only the ws kernel decodes CPS inline
    err = visit_strip_cfg(g, [&](auto cfg) { return run_strip<decltype(cfg)>(a, st); });
    if (err != cudaErrorNotSupported) {
        t_last_conv_kernel = 1;
        return err;
    }
    if (sa_types || cscc) return cudaErrorNotSupported;   // the layout's own kernel runs instead
    // generic
    const int WH = (kGenTY - 1) * g.sh + g.R, WW = (kGenTX - 1) * g.sw + g.S;
    if (WW > 32) return cudaErrorInvalidValue;
    a.tiles_x = (g.Ow + kGenTX - 1) / kGenTX;
    const int ty = (g.Oh + kGenTY - 1) / kGenTY;
    size_t smem = (size_t)kGenWarps * kGenTY * kGenTX * 32 * sizeof(float) + (size_t)kGenWarps * WH * WW * sizeof(float2);
    err = cudaFuncSetAttribute(sparse_conv_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    dim3 grid(a.tiles_x * ty, (g.K + 31) / 32, g.N);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kGenWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    t_last_conv_kernel = 0;
    return cudaLaunchKernelEx(&cfg, sparse_conv_generic_kernel, a, WH, WW);
}

}  // namespace spc

#ifdef SPC_PROBES
SPC_PROBE_ACCESSOR(spc_debug_probes_conv)
extern "C" int spc_debug_set_phase_mode(int m) {
    return (int)cudaMemcpyToSymbol(spc::g_dev_phase_mode, &m, sizeof m);
}
#endif
