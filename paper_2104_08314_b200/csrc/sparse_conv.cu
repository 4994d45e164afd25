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

// Block directory of one channel, from its ptr segment (Alg. 2 lines 9-20).
// pos[t]: index in ptr of the first count of block t (NOP: a, a+b), -1 when the
// block is absent or NPF; da[t]: DA offset of the block inside the channel.
struct ChanDir {
    int npc;
    int pos[kMaxS];
    int da[kMaxS];
};

__device__ __forceinline__ void parse_channel(const Geom& g, const int32_t* __restrict__ ptr, long long P,
                                              ChanDir& d) {
    for (int t = 0; t < kMaxS; t++) { d.pos[t] = -1; d.da[t] = 0; }
    const int32_t first = __ldg(ptr + P);
    d.npc = (first == SPC_NPC);
    if (d.npc) return;
    if (g.S == 1) {
        d.pos[0] = (int)(P + 1);
        return;
    }
    long long p = P;
    int dacur = 0;
    if (g.pl == 0) {                       // NOP [0, a, a+b]
        d.pos[0] = (int)(p + 1);
        dacur = __ldg(ptr + p + 2);
        p += 3;
    }
    for (int t = max(1, g.pl); t <= g.S - 1; t++) {
        const int32_t f = __ldg(ptr + p + 1);
        if (f == SPC_NPF) {                // skip pointer
            p += 2;
            continue;
        }
        d.pos[t] = (int)(p + 1);
        d.da[t] = dacur;
        const int last = (t < g.S - 1) ? (g.Ow1 - 1 - t) : (g.Ow1 - g.S);
        dacur += __ldg(ptr + p + 1 + last);
        p += 1 + g.Ow1;
    }
}

// DA range [lo, hi) (channel-relative) and local column of padded column w.
__device__ __forceinline__ void column_range(const Geom& g, const int32_t* __restrict__ ptr, const ChanDir& d,
                                             int w, int& lo, int& hi) {
    lo = hi = 0;
    if (w < 0 || w >= g.Wp) return;
    if (g.S == 1) {                                           // SI Alg. 5: channel-cumulative
        lo = (w == 0) ? 0 : __ldg(ptr + d.pos[0] + w - 1);
        hi = __ldg(ptr + d.pos[0] + w);
        return;
    }
    if (w >= g.S - 1 && w <= g.Wp - g.S) {                    // overlapK_w column of partition s
        const int t = g.S - 1, s = w - g.S + 1;
        if (d.pos[t] < 0) return;
        lo = d.da[t] + ((s == 0) ? 0 : __ldg(ptr + d.pos[t] + s - 1));
        hi = d.da[t] + __ldg(ptr + d.pos[t] + s);
        return;
    }
    const bool left = w < g.S - 1;
    const int t = left ? w : (g.Wp - 1 - w);
    if (t < g.pl || d.pos[t] < 0) return;                    // pad column or NPF block
    if (t == 0) {                                             // NOP: col 0 then col Wp-1
        const int a = __ldg(ptr + d.pos[0]);
        if (left) { lo = 0; hi = a; }
        else { lo = a; hi = __ldg(ptr + d.pos[0] + 1); }
        return;
    }
    const int c0 = __ldg(ptr + d.pos[t]);                     // left column owned by partition 0
    if (left) { lo = d.da[t]; hi = d.da[t] + c0; }
    else { lo = d.da[t] + c0; hi = d.da[t] + __ldg(ptr + d.pos[t] + g.Ow1 - 1 - t); }
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
};

template <int R_, int S_, int SH_, int SW_, int TY_, int TX_, int KPL_, int WARPS_>
struct TileCfg {
    static constexpr int R = R_, S = S_, SH = SH_, SW = SW_, TY = TY_, TX = TX_, KPL = KPL_, WARPS = WARPS_;
    static constexpr int WH = (TY - 1) * SH + R;   // input window rows
    static constexpr int WW = (TX - 1) * SW + S;   // input window cols
    static constexpr int NCASE = WH * WW;
    static_assert(WW <= 32, "window columns are mapped to lanes");
    static_assert(NCASE <= 256, "jump table size");
};

// One NZE at window position CASE = hr*WW + wr: static FFMAs into acc.
template <class T, int CASE>
__device__ __forceinline__ void apply_case(float v, float (&acc)[T::KPL][T::TY][T::TX],
                                           const float (&w)[T::KPL][T::R][T::S]) {
    constexpr int hr = CASE / T::WW, wr = CASE % T::WW;
#pragma unroll
    for (int l = 0; l < T::R; ++l) {
#pragma unroll
        for (int m = 0; m < T::S; ++m) {
            const int y1 = hr - l, x1 = wr - m;
            if (y1 >= 0 && x1 >= 0 && (y1 % T::SH) == 0 && (x1 % T::SW) == 0 && y1 / T::SH < T::TY &&
                x1 / T::SW < T::TX) {
#pragma unroll
                for (int kk = 0; kk < T::KPL; ++kk)
                    acc[kk][y1 / T::SH][x1 / T::SW] = fmaf(v, w[kk][l][m], acc[kk][y1 / T::SH][x1 / T::SW]);
            }
        }
    }
}

#define SPC_C1(i) \
    case (i):     \
        if constexpr ((i) < T::NCASE) apply_case<T, (i)>(v, acc, w); \
        break;
#define SPC_C4(i) SPC_C1(i) SPC_C1(i + 1) SPC_C1(i + 2) SPC_C1(i + 3)
#define SPC_C16(i) SPC_C4(i) SPC_C4(i + 4) SPC_C4(i + 8) SPC_C4(i + 12)
#define SPC_C64(i) SPC_C16(i) SPC_C16(i + 16) SPC_C16(i + 32) SPC_C16(i + 48)
#define SPC_C256(i) SPC_C64(i) SPC_C64(i + 64) SPC_C64(i + 128) SPC_C64(i + 192)

template <class T>
__device__ __forceinline__ void dispatch(int cs, float v, float (&acc)[T::KPL][T::TY][T::TX],
                                         const float (&w)[T::KPL][T::R][T::S]) {
    switch (cs) {
        SPC_C256(0)
        default:
            break;
    }
}

// Builds the list of NZEs of one channel that fall in the window
// [hy0, hy0+WH) x [wx0, wx0+WW) (padded coordinates); returns its length.
// lanes j < WW own window column wx0 + j.
__device__ __forceinline__ int build_list(const ConvArgs& a, const ChanDir& d, long long Z, int hy0, int wx0,
                                          int WH, int WW, float2* list) {
    const Geom& g = a.g;
    const int lane = threadIdx.x & 31;
    int lo = 0, hi = 0;
    if (lane < WW) column_range(g, a.ptr, d, wx0 + lane, lo, hi);
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
            // rows ascend within a column: stop once the chunk passed the window
            if (__shfl_sync(0xffffffffu, h, 31) >= hy0 + WH && b + 32 < chi) break;
        }
    }
    __syncwarp();
    return n;
}

template <class T>
__global__ void __launch_bounds__(T::WARPS * 32) sparse_conv_kernel(ConvArgs a) {
    const Geom& g = a.g;
    constexpr int KB = 32 * T::KPL;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = blockIdx.z;
    const int kbase = blockIdx.y * KB;
    const int tyi = blockIdx.x / a.tiles_x, txi = blockIdx.x % a.tiles_x;
    const int oy0 = tyi * T::TY, ox0 = txi * T::TX;
    const int hy0 = oy0 * T::SH, wx0 = ox0 * T::SW;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* list = reinterpret_cast<float2*>(smem_raw) + warp * T::NCASE;

    float acc[T::KPL][T::TY][T::TX];
#pragma unroll
    for (int kk = 0; kk < T::KPL; kk++)
#pragma unroll
        for (int yy = 0; yy < T::TY; yy++)
#pragma unroll
            for (int xx = 0; xx < T::TX; xx++) acc[kk][yy][xx] = 0.f;

    for (int c = warp; c < g.C; c += T::WARPS) {
        const long long nc = (long long)n * g.C + c;
        ChanDir d;
        parse_channel(g, a.ptr, a.cpo_off[nc], d);   // NPC -> skip channel
        if (d.npc) continue;
        const long long Z = a.cnz_off[nc];
        const int cnt = build_list(a, d, Z, hy0, wx0, T::WH, T::WW, list);
        if (cnt == 0) continue;
        float w[T::KPL][T::R][T::S];
#pragma unroll
        for (int kk = 0; kk < T::KPL; kk++) {
            const int k = kbase + kk * 32 + lane;
#pragma unroll
            for (int l = 0; l < T::R; l++)
#pragma unroll
                for (int m = 0; m < T::S; m++)
                    w[kk][l][m] = (k < g.K) ? __ldg(a.wp + (((long long)c * T::R + l) * T::S + m) * g.K + k) : 0.f;
        }
#pragma unroll 2
        for (int e = 0; e < cnt; e++) {
            const float2 it = list[e];
            dispatch<T>(__float_as_int(it.y), it.x, acc, w);
        }
        __syncwarp();
    }

    // ---- reduce the WARPS channel splits through smem, store NKHW coalesced over x
    __syncthreads();
    float* red = reinterpret_cast<float*>(smem_raw);   // [WARPS][KPL*TY*TX][32]
    constexpr int NACC = T::KPL * T::TY * T::TX;
#pragma unroll
    for (int kk = 0; kk < T::KPL; kk++)
#pragma unroll
        for (int yy = 0; yy < T::TY; yy++)
#pragma unroll
            for (int xx = 0; xx < T::TX; xx++)
                red[((size_t)warp * NACC + (kk * T::TY + yy) * T::TX + xx) * 32 + lane] = acc[kk][yy][xx];
    __syncthreads();
    for (int idx = threadIdx.x; idx < KB * T::TY * T::TX; idx += T::WARPS * 32) {
        const int xx = idx % T::TX;
        const int yy = (idx / T::TX) % T::TY;
        const int kl = idx / (T::TX * T::TY);        // 0..KB-1
        const int kk = kl / 32, ln = kl % 32;
        const int k = kbase + kl, oy = oy0 + yy, ox = ox0 + xx;
        if (k >= g.K || oy >= g.Oh || ox >= g.Ow) continue;
        float s = 0.f;
#pragma unroll
        for (int wv = 0; wv < T::WARPS; wv++) s += red[((size_t)wv * NACC + (kk * T::TY + yy) * T::TX + xx) * 32 + ln];
        if (a.relu) s = fmaxf(s, 0.f);
        a.y[(((long long)n * g.K + k) * g.Oh + oy) * g.Ow + ox] = s;
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
    for (int c = warp; c < g.C; c += kGenWarps) {
        const long long nc = (long long)n * g.C + c;
        ChanDir d;
        parse_channel(g, a.ptr, a.cpo_off[nc], d);
        if (d.npc) continue;
        const long long Z = a.cnz_off[nc];
        const int cnt = build_list(a, d, Z, hy0, wx0, WH, WW, list);
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
static cudaError_t run_tiled(ConvArgs& a, cudaStream_t st) {
    const Geom& g = a.g;
    const int tx = (g.Ow + T::TX - 1) / T::TX, ty = (g.Oh + T::TY - 1) / T::TY;
    a.tiles_x = tx;
    const int kgroups = (g.K + 32 * T::KPL - 1) / (32 * T::KPL);
    size_t list_bytes = (size_t)T::WARPS * T::NCASE * sizeof(float2);
    size_t red_bytes = (size_t)T::WARPS * T::KPL * T::TY * T::TX * 32 * sizeof(float);
    size_t smem = list_bytes > red_bytes ? list_bytes : red_bytes;
    cudaError_t err = cudaFuncSetAttribute(sparse_conv_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    dim3 grid(tx * ty, kgroups, g.N);
    sparse_conv_kernel<T><<<grid, T::WARPS * 32, smem, st>>>(a);
    return cudaGetLastError();
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
    const bool k_big = g.K > 32;
    if (g.R == 3 && g.S == 3 && g.sh == 1 && g.sw == 1) {
        if (k_big) return run_tiled<TileCfg<3, 3, 1, 1, 8, 8, 2, 4>>(a, st);
        return run_tiled<TileCfg<3, 3, 1, 1, 8, 8, 1, 4>>(a, st);
    }
    if (g.R == 3 && g.S == 3 && g.sh == 2 && g.sw == 2) {
        if (k_big) return run_tiled<TileCfg<3, 3, 2, 2, 4, 8, 2, 4>>(a, st);
        return run_tiled<TileCfg<3, 3, 2, 2, 4, 8, 1, 4>>(a, st);
    }
    if (g.R == 1 && g.S == 7 && g.sh == 1 && g.sw == 1) return run_tiled<TileCfg<1, 7, 1, 1, 8, 8, 2, 4>>(a, st);
    if (g.R == 7 && g.S == 1 && g.sh == 1 && g.sw == 1) return run_tiled<TileCfg<7, 1, 1, 1, 8, 8, 2, 4>>(a, st);
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
