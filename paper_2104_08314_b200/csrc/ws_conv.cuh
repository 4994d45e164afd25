// ws_conv.cuh -- warp-specialised strip convolution over the CPO encoding (sm_100a), v2.
// Included by sparse_conv.cu inside namespace spc (it reuses DirS / parse_dir /
// column_range_s / tap_fma / ConvArgs from there).
//
// What it computes: exactly what strip_conv_kernel computes (Alg. 2 convSpMv, PAPER.md:236-309;
// reading A15 for strides): every NZE v at padded (h, w) of channel c adds v * W[k,c,l,m] to the
// output that sees it through tap (l, m); NPC channels and NPF blocks are skipped.
//
// Why a second kernel: round 1's strip kernel runs each chunk of input channels as three
// phases behind CTA barriers -- P0 stage the taps, P1 parse the ptr directory and scatter the
// NZEs of the strip's window columns into dense windows, P2 walk the windows -- so on the
// 14x14 / 7x7 layers the two staging phases (L2 round trips) were 40-60 % of the time and the
// walk itself ran at ~4 warps per scheduler between barriers.  Here the phases run on
// DIFFERENT warps of one CTA per SM (warp specialisation, the Blackwell producer / consumer
// pattern):
//  * 4 producer warps: thread 0 issues TMA bulk copies (cp.async.bulk, mbarrier-counted) of the
//    chunk's filter taps [CH][R][S][KBC] (one contiguous block when the CTA covers all K) and of
//    its ptr segments; all producer threads parse the block directories, scatter the NZEs into
//    the window buffers of the stage and build each window's occupancy mask;
//  * consumer warps = (row tile, k-group): every k-group warp walks the SAME scattered window with
//    its own 32*KPL output channels (the scatter is shared by KG k-groups: K = 256 layers scatter
//    once per strip instead of once per 128 channels);
//  * NST-stage ring (full / empty mbarriers): the producers fill stage s+1 while the consumers
//    walk stage s, so staging and scatter hide behind the walk.
// Epilogue: direct float4 stores from the consumers' registers (ReLU optional), or -- when the
// input channels are split over a cluster of cg CTAs -- partials through L2 and one cluster
// barrier, as in the round-1 kernel.

template <int R_, int S_, int SH_, int SW_, int TY_, int KPL_, int KG_, int CH_, int NST_ = 4, int DCAP_ = 384>
struct WsCfg {
    static constexpr int DCAP = DCAP_;                    // DA / IN entries a producer stages per chunk
    static constexpr int R = R_, S = S_, SH = SH_, SW = SW_, TY = TY_, TX = 4, KPL = KPL_;
    static constexpr int KG = KG_;                        // k-groups per CTA (consumers share windows)
    static constexpr int CH = CH_, NST = NST_;
    static constexpr int KB = 32 * KPL;                   // output channels per consumer warp
    static constexpr int KBC = KB * KG;                   // output channels per CTA
    static constexpr int RS = R * S;
    static constexpr int WH = (TY - 1) * SH + R;
    static constexpr int WW = (TX - 1) * SW + S;
    static constexpr int NCASE = WH * WW;
    static constexpr int MW = (NCASE + 31) / 32;
    static constexpr int NCP = 32 * MW;
    static constexpr int RSTEP = TY * SH;
    static constexpr bool PACKED = (KPL % 2) == 0;
    static constexpr int NP = PACKED ? KPL / 2 : KPL;
    static constexpr int NACC = KPL * TY * TX;
    static constexpr int NPROD = 4;                       // producer warps
    // consumer warps at most.  The register file is split over the 4 schedulers (16 K registers
    // each), so a CTA of W warps needs ceil(W / 4) * 32 * regs <= 16384: 16 warps at 128 registers
    // (4 x 4 tiles x 4 channels per lane), 20 warps at 96 (smaller tiles)
    static constexpr int MAXCONS = (TY * KPL >= 16) ? 12 : 16;
    static constexpr int MAXREG = (MAXCONS == 12) ? 128 : 96;
    static_assert(WW <= 32, "window columns are mapped to lanes");
    static_assert(MW <= 4, "window too large");
    static_assert(PACKED, "v2 walks packed FFMA2 taps");
};

// shared-memory carve-up (host and device agree through this)
struct WsSmem {
    size_t w, val, msk, pbuf, pre, lo, tot, cb, coff, cz, cq, dec, bars, total;
    int pstride;   // ints of the ptr part of one producer buffer
    int bstride;   // bytes of one producer buffer: ptr | DA | IN
};
template <class T>
__host__ __device__ inline WsSmem ws_smem_layout(int RT, int pmax, int crange, bool cps = false) {
    WsSmem L;
    L.pstride = (int)align_up((size_t)T::CH * pmax + 8, 4);
    L.bstride = (int)((size_t)L.pstride * 4 + (size_t)2 * (T::DCAP + 8) * 4);
    L.w = 0;                                                                     // [NST][CH][RS][KBC]
    L.val = L.w + (size_t)T::NST * T::CH * T::RS * T::KBC * 4;                    // [NST][CH][RT][NCP]
    L.msk = L.val + (size_t)T::NST * T::CH * RT * T::NCP * 4;                     // [NST][CH][RT][MW]
    L.pbuf = align_up(L.msk + (size_t)T::NST * T::CH * RT * T::MW * 4, 16);      // [NPROD][2] ptr | DA | IN
    L.pre = align_up(L.pbuf + (size_t)T::NPROD * 2 * L.bstride, 16);             // [NPROD][CH][32] column prefix
    L.lo = L.pre + (size_t)T::NPROD * T::CH * 32 * 4;                             // [NPROD][CH][32] column DA start
    L.tot = L.lo + (size_t)T::NPROD * T::CH * 32 * 4;                             // [NPROD][CH]
    L.cb = L.tot + (size_t)T::NPROD * T::CH * 4;                                  // [NPROD][CH][32] slot column base
    L.coff = L.cb + (size_t)T::NPROD * T::CH * 32 * 4;                            // [crange+1] ptr offsets (rel)
    L.cz = L.coff + (size_t)(crange + 1) * 4;                                     // [crange+1] DA offsets (rel)
    L.cq = L.cz + (size_t)(crange + 1) * 4;                                       // [crange+1] CPS IN offsets (rel)
    L.dec = align_up(L.cq + (cps ? (size_t)(crange + 1) * 4 : 0), 16);            // [NPROD][DCAP+8] decoded CPS IN
    L.bars = align_up(L.dec + (cps ? (size_t)T::NPROD * (T::DCAP + 8) * 4 : 0) + 16, 16);   // full, empty [NST], pbar [NPROD][2]
    L.total = L.bars + (size_t)(2 * T::NST + 2 * T::NPROD) * 8 + 64;
    return L;
}

__device__ __forceinline__ void ws_mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void producer_sync() {   // named barrier 1 over the 4 producer warps
    asm volatile("bar.sync 1, 128;" ::: "memory");
}

struct WsArgs {
    ConvArgs a;
    int RT;          // row tiles (ceil(Oh / TY))
    int ncons;       // consumer warps = RT * KG
    int nkb;         // CTAs along K (gridDim.y): K > KBC
};

template <class T>
__global__ void __maxnreg__(T::MAXREG) ws_conv_kernel(WsArgs wa) {
    namespace cgrp = cooperative_groups;
    const ConvArgs& a = wa.a;
    const Geom& g = a.g;
    const int RT = wa.RT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool producer = warp < T::NPROD;
    const int rank = (a.cg > 1) ? (int)cgrp::this_cluster().block_rank() : 0;
    const int n = blockIdx.z / a.cg;
    const int kbase = blockIdx.y * T::KBC;
    const int ox0 = blockIdx.x * T::TX, wx0 = ox0 * T::SW;
    const int cper = (g.C + a.cg - 1) / a.cg;
    const int c_begin = min(g.C, rank * cper), c_end = min(g.C, c_begin + cper);
    const int nchunks = (c_end - c_begin + T::CH - 1) / T::CH;
    const int kvalid = min(T::KBC, g.K - kbase);      // output channels of this CTA that exist

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const bool cps = a.cps_in != nullptr;   // CPS stream decoded by the producers (Alg. 4)
    const WsSmem L = ws_smem_layout<T>(RT, a.pmax, cper, cps);
    float* s_w = reinterpret_cast<float*>(smem_raw + L.w);
    float* s_val = reinterpret_cast<float*>(smem_raw + L.val);
    unsigned* s_msk = reinterpret_cast<unsigned*>(smem_raw + L.msk);
    unsigned char* s_pbuf = smem_raw + L.pbuf;
    int* fpre = reinterpret_cast<int*>(smem_raw + L.pre);
    int* flo = reinterpret_cast<int*>(smem_raw + L.lo);
    int* ftot = reinterpret_cast<int*>(smem_raw + L.tot);
    int* fcb = reinterpret_cast<int*>(smem_raw + L.cb);
    int* s_coff = reinterpret_cast<int*>(smem_raw + L.coff);
    int* s_cz = reinterpret_cast<int*>(smem_raw + L.cz);
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem_raw + L.bars);
    unsigned long long* empty = full + T::NST;
    unsigned long long* pbar = empty + T::NST;              // [NPROD][2] producer-private copies

    const size_t tap_stage = (size_t)T::CH * T::RS * T::KBC;
    const size_t val_stage = (size_t)T::CH * RT * T::NCP;
    const size_t msk_stage = (size_t)T::CH * RT * T::MW;

    if (threadIdx.x == 0) {
        for (int s = 0; s < T::NST; s++) {
            mbar_init(&full[s], 2);              // the taps' expect_tx arrival + producer thread 0's arrival
            mbar_init(&empty[s], wa.ncons);      // one arrival per consumer warp
        }
        for (int q = 0; q < 2 * T::NPROD; q++) mbar_init(&pbar[q], 1);   // expect_tx of a chunk's copies
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // taps of chunk i -> stage s (TMA bulk; independent of the encoder, so the first NST chunks
    // are issued before griddepcontrol.wait: they overlap the encoder's tail)
    auto issue_taps = [&](int i) {
        const int s = i % T::NST;
        const int c0 = c_begin + i * T::CH, chn = min(T::CH, c_end - c0);
        float* dst = s_w + s * tap_stage;
        if (T::KBC == g.K) {
            const unsigned bytes = (unsigned)((size_t)chn * T::RS * g.K * 4);
            mbar_expect_tx(&full[s], bytes);
            const char* src = reinterpret_cast<const char*>(a.wp + (size_t)c0 * T::RS * g.K);
            for (unsigned off = 0; off < bytes; off += 32768u)
                bulk_g2s(reinterpret_cast<char*>(dst) + off, src + off, min(32768u, bytes - off), &full[s]);
        } else {
            const unsigned row = (unsigned)kvalid * 4;
            mbar_expect_tx(&full[s], row * (unsigned)(chn * T::RS));
            for (int r = 0; r < chn * T::RS; r++)
                bulk_g2s(dst + (size_t)r * T::KBC, a.wp + ((size_t)c0 * T::RS + r) * g.K + kbase, row, &full[s]);
        }
    };

    using AccT = float2;
    AccT acc[T::NP][T::TY][T::TX];
#pragma unroll
    for (int p = 0; p < T::NP; p++)
#pragma unroll
        for (int yy = 0; yy < T::TY; yy++)
#pragma unroll
            for (int xx = 0; xx < T::TX; xx++) acc[p][yy][xx] = make_float2(0.f, 0.f);

    if (producer) {
        // Producer warp p owns the chunks i == p (mod NPROD) and their stage s = i % NST (NST ==
        // NPROD): each warp runs its own chain (side tables from smem -> ptr bulk copy -> parse
        // -> IN / DA loads -> scatter -> masks), so NPROD chunks' L2 round trips are in flight at
        // once instead of one chunk's after another's.
        static_assert(T::NST == T::NPROD, "one stage per producer warp");
        const int p = warp;
        if (lane == 0 && p == 0) probe_any(0);
        if (lane == 0)
            for (int i = p; i < min(T::NST, nchunks); i += T::NPROD) issue_taps(i);
        pdl_wait();
        if (lane == 0 && p == 0) probe_any(1);
        // the encoding's flag word is loaded together with the side tables (in bounds whatever
        // the flag), not ahead of them; a flagged encoding's streams are never read
        const unsigned long long st0 = *reinterpret_cast<volatile unsigned long long*>(a.status);
        const long long ncb = (long long)n * g.C;
        // side tables of the CTA's channel range, once: ptr / DA offsets relative to the range start
        const long long pbase = __ldg(a.cpo_off + ncb + c_begin);
        const long long zbase = __ldg(a.cnz_off + ncb + c_begin);
        int* s_pof = s_coff;                       // [C range + 1]
        int* s_zof = s_cz;                         // [C range + 1]
        const bool bad = st0 != 0ull;
        const long long qbase = cps ? __ldg(a.cin_off + ncb + c_begin) : 0;
        int* s_qof = reinterpret_cast<int*>(smem_raw + L.cq);   // [C range + 1] (CPS only)
        for (int q = threadIdx.x; q <= c_end - c_begin; q += 32 * T::NPROD) {
            s_pof[q] = (int)(__ldg(a.cpo_off + ncb + c_begin + q) - pbase);
            s_zof[q] = (int)(__ldg(a.cnz_off + ncb + c_begin + q) - zbase);
            if (cps) s_qof[q] = (int)(__ldg(a.cin_off + ncb + c_begin + q) - qbase);
        }
        producer_sync();
        int* wpre = fpre + p * T::CH * 32;         // this warp's column tables
        int* wlo = flo + p * T::CH * 32;
        int* wcb = fcb + p * T::CH * 32;           // stride-aware slots: window column of the partition
        // Producer-private double buffer: the ptr segments and the DA / IN segments of the warp's
        // NEXT chunk are copied (TMA bulk, 16-byte aligned part; the < 16-byte tails with plain
        // loads) while it scatters the current one, so a chunk's chain no longer waits on L2
        // round trips.  A chunk with more than DCAP NZEs reads DA / IN from global memory instead.
        auto pb_ptr = [&](int b) { return reinterpret_cast<int*>(s_pbuf + (size_t)(2 * p + b) * L.bstride); };
        auto pb_da = [&](int b) { return reinterpret_cast<float*>(pb_ptr(b) + L.pstride); };
        auto pb_in = [&](int b) { return reinterpret_cast<int*>(pb_da(b) + T::DCAP + 8); };
        auto prefetch = [&](int i, int b) {
            const int c0 = c_begin + i * T::CH, chn = min(T::CH, c_end - c0), r0 = c0 - c_begin;
            const long long P0 = pbase + s_pof[r0], P1 = pbase + s_pof[r0 + chn];
            const long long Z0 = zbase + s_zof[r0], Z1 = zbase + s_zof[r0 + chn];
            const long long pa = P0 & ~3ll, za = Z0 & ~3ll;
            const long long pn = ((P1 - pa) >> 2) << 2, zn = ((Z1 - za) >> 2) << 2;
            const bool fits = (Z1 - za) <= T::DCAP + 4;
            // IN: the CPO-form stream at the DA positions, or the CPS stream (never longer than DA)
            const long long Q0 = cps ? qbase + s_qof[r0] : za, Q1 = cps ? qbase + s_qof[r0 + chn] : Z1;
            const long long qa = Q0 & ~3ll, qn = ((Q1 - qa) >> 2) << 2;
            const int32_t* isrc = cps ? a.cps_in : a.in;
            int* dp = pb_ptr(b);
            if (lane == 0) {
                fence_proxy_async();   // generic reads of this buffer (two chunks ago) before the copies
                mbar_expect_tx(&pbar[2 * p + b], (unsigned)(4 * (pn + (fits ? zn + qn : 0))));
                if (pn > 0) bulk_g2s(dp, a.ptr + pa, (unsigned)(pn * 4), &pbar[2 * p + b]);
                if (fits && zn > 0) bulk_g2s(pb_da(b), a.da + za, (unsigned)(zn * 4), &pbar[2 * p + b]);
                if (fits && qn > 0) bulk_g2s(pb_in(b), isrc + qa, (unsigned)(qn * 4), &pbar[2 * p + b]);
            }
            if (pa + pn + lane < P1) dp[pn + lane] = __ldg(a.ptr + pa + pn + lane);
            if (fits && za + zn + lane < Z1) pb_da(b)[zn + lane] = __ldg(a.da + za + zn + lane);
            if (fits && qa + qn + lane < Q1) pb_in(b)[qn + lane] = __ldg(isrc + qa + qn + lane);
        };
        if (!bad && p < nchunks) prefetch(p, 0);
        int k = 0;   // this warp's chunk counter (buffer k & 1)
        for (int i = p; i < nchunks; i += T::NPROD, k++) {
            const int s = i % T::NST;
            const unsigned ph = (unsigned)(i / T::NST) & 1u;
            const int c0 = c_begin + i * T::CH, chn = min(T::CH, c_end - c0);
            const int r0 = c0 - c_begin;
            const int b = k & 1;
            if (bad) {
                if (i >= T::NST) mbar_wait(&empty[s], ph ^ 1u);
                // flagged encoding: publish empty windows (y = 0); the taps still land
                unsigned* mk = s_msk + s * msk_stage;
                for (int q = lane; q < chn * RT * T::MW; q += 32) mk[q] = 0u;
                if (lane == 0 && i >= T::NST) issue_taps(i);
                __syncwarp();
                if (lane == 0) ws_mbar_arrive(&full[s]);
                continue;
            }
            __syncwarp();
            if (i + T::NPROD < nchunks) prefetch(i + T::NPROD, b ^ 1);
            if (i >= T::NST) mbar_wait(&empty[s], ph ^ 1u);   // the consumers released stage s
            if (lane == 0 && i >= T::NST) issue_taps(i);
            const long long P0 = pbase + s_pof[r0];
            const int shift = (int)(P0 - (P0 & ~3ll));
            const long long Z0 = zbase + s_zof[r0], Z1 = zbase + s_zof[r0 + chn];
            const long long za = Z0 & ~3ll;
            const bool fits = (Z1 - za) <= T::DCAP + 4;
            const int* sp = pb_ptr(b);
            const float* sda = pb_da(b) + (Z0 - za);   // DA / IN of the chunk's first channel
            int* const sdec = reinterpret_cast<int*>(smem_raw + L.dec) + p * (T::DCAP + 8);
            const int* sin = cps ? sdec : pb_in(b) + (Z0 - za);
            // masks of this stage start empty; the window VALUES are never zeroed -- a consumer only
            // reads a window slot whose mask bit the scatter below set
            unsigned* mk = s_msk + s * msk_stage;
            for (int q = lane; q < chn * RT * T::MW; q += 32) mk[q] = 0u;
            mbar_wait(&pbar[2 * p + b], (unsigned)(k >> 1) & 1u);
            // (a) LPC lanes per channel, one window column per lane: every lane parses its channel's
            //     block directory (the chunk's channels in parallel), takes its column's DA range,
            //     and a segmented scan gives the column prefix inside the channel
            const int nsl = a.sa_types ? sa_nslots(g, wx0, T::WW) : T::WW;   // slots per channel
            {
                constexpr int LPC = (T::WW <= 8) ? 8 : 16;          // (stride-aware slots: <= 16, host-checked)
                constexpr int CPP = 32 / LPC;                       // channels per pass
                const int jl = lane / LPC, col = lane % LPC;
                for (int j0 = 0; j0 < chn; j0 += CPP) {
                    const int j = j0 + jl;
                    int lo = 0, hi = 0, cb = 0;
                    if (j < chn) {
                        const int* seg = sp + shift + (s_pof[r0 + j] - s_pof[r0]);   // (chunk-relative)
                        DirS<T::S> d;
                        if (a.sa_types) {
                            parse_dir_sa<T::S>(g, seg, d, a.sa_types);
                            if (!d.npc && col < nsl) sa_slot_range<T::S>(g, seg, d, wx0, T::WW, col, lo, hi, cb);
                        } else {
                            parse_dir<T::S>(g, seg, d);
                            if (!d.npc && col < T::WW) column_range_s<T::S>(g, seg, d, wx0 + col, lo, hi);
                            // CPS: DA start of the overlapK_w block (the entries before it are 1:1)
                            if (cps && col == 0)
                                wcb[j * 32 + 31] = (d.npc || d.pos[T::S - 1] < 0) ? (1 << 30) : d.da[T::S - 1];
                        }
                    }
                    int inc = hi - lo;
#pragma unroll
                    for (int o = 1; o < LPC; o <<= 1) {
                        const int t = __shfl_up_sync(0xffffffffu, inc, o);
                        if (col >= o) inc += t;
                    }
                    if (j < chn) {
                        wpre[j * 32 + col] = (col < nsl) ? inc - (hi - lo) : (1 << 30);
                        wlo[j * 32 + col] = lo;
                        wcb[j * 32 + col] = cb;
                        if (col == LPC - 1) ftot[p * T::CH + j] = inc;
                    }
                }
            }
            __syncwarp();
            if (cps) {
                // (a') Alg. 4 over the chunk's CPS IN entries flattened across its
                //      channels (their segments are contiguous): entries below a channel's overlapK_w
                //      block are 1:1 with DA; inside it a negative entry is a singleton at -e, a
                //      non-negative one an index followed by its pattern P (rows e + S*(bit - lowest
                //      bit)).  Indices and patterns alternate after the last 1:1 / negative entry (the
                //      role is the parity of the distance to it, carried across 32-entry slices); NZE
                //      counts scanned give the DA positions.  Output: CPO-form indices at the chunk's
                //      DA positions, in shared memory when the chunk was staged, else in the
                //      workspace buffer `a.in`.
                const long long Q0 = qbase + s_qof[r0];
                const int* qsrc = fits ? pb_in(b) + (int)(Q0 & 3ll) : a.cps_in + Q0;
                int* zdst = fits ? sdec : const_cast<int*>(a.in) + Z0;
                const int nq = s_qof[r0 + chn] - s_qof[r0];
                const int qj = (lane < chn) ? s_qof[r0 + lane] - s_qof[r0] : (1 << 30);
                const int dmj = (lane < chn) ? wcb[lane * 32 + 31] : 0;
                int dpos = 0;
                bool carry = false;
                for (int q = 0; q < nq; q += 32) {
                    const int i = q + lane;
                    const bool valid = i < nq;
                    const int e = valid ? qsrc[i] : -1;
                    int j = 0;
#pragma unroll
                    for (int step = T::CH / 2; step > 0; step >>= 1) {
                        const int cand = j + step;
                        const int cv = __shfl_sync(0xffffffffu, qj, cand & 31);
                        if (cand < chn && cv <= i) j = cand;
                    }
                    const int rel = i - __shfl_sync(0xffffffffu, qj, j);
                    const int dm = __shfl_sync(0xffffffffu, dmj, j);
                    const bool one = valid && rel < dm;
                    const bool brk = valid && (one || e < 0);
                    const unsigned before = __ballot_sync(0xffffffffu, brk) & lanemask_lt();
                    const int r = before ? (32 - __clz(before)) : 0;
                    const bool base_pat = (r == 0) ? carry : false;
                    const bool nonneg = valid && !brk;
                    const bool is_pat = nonneg && (base_pat ^ (((lane - r) & 1) != 0));
                    const bool is_idx = nonneg && !is_pat;
                    int nxt = __shfl_down_sync(0xffffffffu, e, 1);
                    if (lane == 31) nxt = (i + 1 < nq) ? qsrc[i + 1] : -1;
                    const int cnt = brk ? 1 : (is_idx ? __popc(nxt & 0xF) : 0);
                    int tot;
                    const int o = dpos + warp_exclusive_scan(cnt, &tot);
                    if (brk) {
                        zdst[o] = one ? e : -e;
                    } else if (is_idx) {
                        const unsigned pm = (unsigned)nxt & 0xFu;
                        const int b0 = __ffs(pm) - 1;
                        int u = 0;
#pragma unroll
                        for (int bb = 0; bb < 4; bb++)
                            if ((pm >> bb) & 1u) zdst[o + u++] = e + T::S * (bb - b0);
                    }
                    carry = __shfl_sync(0xffffffffu, is_idx, 31);
                    dpos += tot;
                }
                if (!fits) __threadfence_block();
                __syncwarp();
            }
            // (b) the chunk's NZEs flattened across its channels (staged DA / IN, or global memory
            //     for a chunk beyond DCAP): value into every row tile window holding the row, and the
            //     window's occupancy bit (shared-memory atomic OR)
            {
                int total;
                const int cpre = warp_exclusive_scan(lane < chn ? ftot[p * T::CH + lane] : 0, &total);
                float* win0 = s_val + s * val_stage;
                constexpr int U = 4;
                for (int f0 = 0; f0 < total; f0 += 32 * U) {
                    int e[U], pos[U];
                    float v[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int f = f0 + 32 * u + lane;
                        int j = 0;
#pragma unroll
                        for (int step = T::CH / 2; step > 0; step >>= 1) {
                            const int cand = j + step;
                            const int cv = __shfl_sync(0xffffffffu, cpre, cand & 31);
                            if (cand < chn && cv <= f) j = cand;
                        }
                        const int fj = f - __shfl_sync(0xffffffffu, cpre, j);
                        e[u] = -1;
                        v[u] = 0.f;
                        pos[u] = 0;
                        if (f < total) {
                            const int* jp = wpre + j * 32;
                            int jc = 0;
#pragma unroll
                            for (int step = 16; step > 0; step >>= 1)
                                if (jc + step < nsl && jp[jc + step] <= fj) jc += step;
                            const int zr = s_zof[r0 + j] - s_zof[r0];    // channel's DA offset in the chunk
                            const int idx = wlo[j * 32 + jc] + (fj - jp[jc]);
                            if (fits) {
                                e[u] = sin[zr + idx];
                                v[u] = sda[zr + idx];
                            } else {
                                // (decoded by this warp just above when CPS: L2 loads, not the nc path)
                                e[u] = cps ? __ldcg(a.in + Z0 + zr + idx) : __ldg(a.in + Z0 + zr + idx);
                                v[u] = __ldg(a.da + Z0 + zr + idx);
                            }
                            pos[u] = j * RT + jc * 65536;          // window (j, 0) and column jc
                            if (a.sa_types) {                      // window column = partition base + L
                                const int cc = wcb[j * 32 + jc] + e[u] % T::S;
                                pos[u] = j * RT + cc * 65536;
                                if (cc < 0 || cc >= T::WW) e[u] = -1;
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        if (e[u] < 0) continue;
                        const int h = e[u] / T::S;                 // IN = L + h*S with L < S
                        const int rhi = min(RT - 1, h / T::RSTEP);
                        const int rlo = (h >= T::WH - 1) ? (h - T::WH + 1 + T::RSTEP - 1) / T::RSTEP : 0;
                        const int wj = pos[u] & 0xFFFF, jc = pos[u] >> 16;
                        for (int r = rlo; r <= rhi; r++) {
                            const int slot = (h - r * T::RSTEP) * T::WW + jc;
                            win0[(wj + r) * T::NCP + slot] = v[u];
                            atomicOr(mk + (wj + r) * T::MW + (slot >> 5), 1u << (slot & 31));
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0 && i < 6) probe_any(2 + i);
            if (lane == 0) ws_mbar_arrive(&full[s]);   // release: windows + masks visible to the consumers
        }
    } else {
        pdl_wait();
        const int cw = warp - T::NPROD;
        const int rtile = cw % RT, kg = cw / RT;
        for (int i = 0; i < nchunks; i++) {
            const int s = i % T::NST;
            const unsigned ph = (unsigned)(i / T::NST) & 1u;
            const int c0 = c_begin + i * T::CH, chn = min(T::CH, c_end - c0);
            mbar_wait(&full[s], ph);
            const float* wst = s_w + s * tap_stage + kg * T::KB + lane * T::KPL;
            const float* vst = s_val + s * val_stage;
            const unsigned* mst = s_msk + s * msk_stage;
            for (int j = 0; j < chn; j++) {
                unsigned mw[T::MW];
                bool any = false;
#pragma unroll
                for (int q = 0; q < T::MW; q++) {
                    mw[q] = mst[(j * RT + rtile) * T::MW + q];
                    any |= mw[q] != 0;
                }
                if (!any) continue;
                float2 w[T::NP][T::R][T::S];
#pragma unroll
                for (int l = 0; l < T::R; l++)
#pragma unroll
                    for (int m = 0; m < T::S; m++) {
                        const float* ws = wst + (j * T::RS + l * T::S + m) * T::KBC;
                        if constexpr (T::KPL % 4 == 0) {
#pragma unroll
                            for (int p = 0; p < T::NP; p += 2) {
                                const float4 q4 = *reinterpret_cast<const float4*>(ws + 2 * p);
                                w[p][l][m] = make_float2(q4.x, q4.y);
                                w[p + 1][l][m] = make_float2(q4.z, q4.w);
                            }
                        } else {
#pragma unroll
                            for (int p = 0; p < T::NP; p++) w[p][l][m] = *reinterpret_cast<const float2*>(ws + 2 * p);
                        }
                    }
                const float4* w4 = reinterpret_cast<const float4*>(vst + (j * RT + rtile) * T::NCP);
                constexpr int NQ = (T::NCASE + 3) / 4;
                float4 vn = lds128(w4);
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
                            if (P < T::NCASE && ((nib >> u) & 1u)) tap_fma<T>(P, vv[u], acc, w);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0 && cw == 0 && i < 6) probe_any(8 + i);
            if (lane == 0 && cw == 0 && i == nchunks - 1) probe_any(14);
            if (lane == 0) ws_mbar_arrive(&empty[s]);
        }
    }

    // ---- epilogue
    // The next kernel (the next layer's or step's encoder) may launch now: it waits
    // (griddepcontrol.wait) for this grid's completion before it reads anything we write, and its
    // CTAs start on the SMs this grid leaves idle.
    pdl_trigger();
    constexpr int TT = T::TY * T::TX, NCH = TT / 4;
    float* yb = a.y + (long long)n * g.K * g.Oh * g.Ow;
    const bool vec_ok = (g.Ow % 4) == 0;
    const int cw = warp - T::NPROD;
    const int rtile = producer ? 0 : cw % RT, kg = producer ? 0 : cw / RT;
    auto store4 = [&](float* dst, float4 v, int k, int oy) {
        if (a.relu) { v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f); }
        emit_omask(a.omask, g, n, k, oy, ox0, v);
        if (vec_ok && ox0 + 3 < g.Ow) {
            *reinterpret_cast<float4*>(dst) = v;
        } else {
            const float sv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (ox0 + q < g.Ow) dst[q] = sv[q];
        }
    };
    // accumulator chunk i = (kk, output row): lane owns k = kbase + kg*KB + lane*KPL + kk
    auto accv = [&](int i) -> float4 {
        const int kk = i / NCH, yy = i % NCH, p = kk >> 1;
        const bool hi = kk & 1;
        float4 v;
        v.x = hi ? acc[p][yy][0].y : acc[p][yy][0].x;
        v.y = hi ? acc[p][yy][1].y : acc[p][yy][1].x;
        v.z = hi ? acc[p][yy][2].y : acc[p][yy][2].x;
        v.w = hi ? acc[p][yy][3].y : acc[p][yy][3].x;
        return v;
    };
    if (a.cg == 1) {
        if (threadIdx.x == 32 * T::NPROD) probe_any(15);
        if (!producer) {
#pragma unroll
            for (int i = 0; i < T::NACC / 4; i++) {
                const int k = kbase + kg * T::KB + lane * T::KPL + (i / NCH), oy = rtile * T::TY + (i % NCH);
                if (k >= g.K || oy >= g.Oh) continue;
                store4(yb + ((long long)k * g.Oh + oy) * g.Ow + ox0, accv(i), k, oy);
            }
        }
        return;
    }
    // cluster split: partials [NCH][rows] float4 in L2 (rows = RT*KBC), one cluster barrier,
    // then each rank sums its share over the cg partials
    const int rows = RT * T::KBC;
    const long long slot0 = ((long long)(blockIdx.z - rank) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    const long long sstride = (long long)gridDim.y * gridDim.x;
    if (!producer) {
        float4* mine = reinterpret_cast<float4*>(a.scratch) + (slot0 + rank * sstride) * (long long)rows * NCH;
#pragma unroll
        for (int i = 0; i < T::NACC / 4; i++) {
            const int row = rtile * T::KBC + kg * T::KB + (i / NCH) * 32 + lane, c = i % NCH;
            mine[(long long)c * rows + row] = accv(i);
        }
    }
    cgrp::this_cluster().sync();
    if (threadIdx.x == 32 * T::NPROD) probe_any(15);
    const int total = rows * NCH;
    const int per = (total + a.cg - 1) / a.cg;
    const float4* base = reinterpret_cast<const float4*>(a.scratch) + slot0 * (long long)rows * NCH;
    const long long pstride = sstride * (long long)rows * NCH;
    for (int ci = rank * per + threadIdx.x; ci < min(total, (rank + 1) * per); ci += blockDim.x) {
        float4 v[8];
#pragma unroll
        for (int r = 0; r < 8; r++) v[r] = (r < a.cg) ? __ldcg(base + r * pstride + ci) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 sum = v[0];
#pragma unroll
        for (int r = 1; r < 8; r++) { sum.x += v[r].x; sum.y += v[r].y; sum.z += v[r].z; sum.w += v[r].w; }
        const int c = ci / rows, row = ci % rows;
        const int rt = row / T::KBC, kl = row % T::KBC;            // kl = kg*KB + kk*32 + lane
        const int kgi = kl / T::KB, kin = kl % T::KB;
        const int k = kbase + kgi * T::KB + (kin & 31) * T::KPL + (kin >> 5), oy = rt * T::TY + c;
        if (k >= g.K || oy >= g.Oh) continue;
        store4(yb + ((long long)k * g.Oh + oy) * g.Ow + ox0, sum, k, oy);
    }
}

// Launch geometry of a v2 configuration; returns false when it does not apply.
template <class T>
struct WsPlan {
    int strips, RT, ncons, nkb, cg;
    long long units;
    size_t smem, scratch_bytes;
};

template <class T>
static bool plan_ws(const Geom& g, int pmax, WsPlan<T>& p, bool cps = false) {
    p.strips = (g.Ow + T::TX - 1) / T::TX;
    p.RT = (g.Oh + T::TY - 1) / T::TY;
    p.ncons = p.RT * T::KG;
    if (p.ncons > T::MAXCONS) return false;
    if (g.K % 4 != 0) return false;                           // 16-byte tap rows for the bulk copies
    p.nkb = (g.K + T::KBC - 1) / T::KBC;
    if (p.nkb > 1 && g.K % T::KBC != 0) return false;
    p.units = (long long)p.strips * p.nkb * g.N;
    // cluster split of the input channels while the grid stays within one wave (1 CTA/SM),
    // >= 2 chunks per CTA
    const int sms = device_sm_count();
    p.cg = 1;
    for (int cg = 2; cg <= 8; cg *= 2)
        if (p.units * cg <= sms && g.C >= 2 * cg * T::CH) p.cg = cg;
    p.smem = ws_smem_layout<T>(p.RT, pmax, (g.C + p.cg - 1) / p.cg, cps).total;
    if (p.smem > 227 * 1024) return false;
    p.scratch_bytes = (p.cg > 1) ? (size_t)p.units * p.cg * p.RT * T::KBC * T::TY * T::TX * 4 : 0;
    return true;
}

template <class T>
static cudaError_t run_ws(ConvArgs& a, cudaStream_t st) {
    const Geom& g = a.g;
    // CSCC encodings run on the strip kernel (its P1 reads CSCC's per-submatrix rows); the
    // stride-aware layout's (partition, type) slots are parsed by the producers here as well
    // (SPC_WS_SLOTS=0: strip kernel, development A/B)
    static const int ws_slots = [] { const char* v = getenv("SPC_WS_SLOTS"); return v ? atoi(v) : 1; }();
    if (a.cscc || (a.sa_types && !ws_slots)) return cudaErrorNotSupported;
    WsPlan<T> p;
    if (!plan_ws<T>(g, a.pmax, p, a.cps_in != nullptr)) return cudaErrorNotSupported;
    if (p.cg > 1 && (!a.scratch || a.scratch_bytes < p.scratch_bytes)) {          // no scratch: no split
        p.cg = 1;
        p.smem = ws_smem_layout<T>(p.RT, a.pmax, g.C, a.cps_in != nullptr).total;   // one CTA's side tables cover every channel
        if (p.smem > 227 * 1024) return cudaErrorNotSupported;
    }
    WsArgs wa;
    wa.a = a;
    wa.a.cg = p.cg;
    wa.RT = p.RT;
    wa.ncons = p.ncons;
    wa.nkb = p.nkb;
    static std::atomic<size_t> attr_bytes[kMaxDevices];
    cudaError_t err = ensure_smem_attr((const void*)ws_conv_kernel<T>, p.smem, attr_bytes);
    if (err != cudaSuccess) return err;
    {
        static std::atomic<int> max_threads[kMaxDevices];
        std::atomic<int>& mt = max_threads[current_device()];
        if (mt.load() == 0) {
            cudaFuncAttributes fa;
            if (cudaFuncGetAttributes(&fa, (const void*)ws_conv_kernel<T>) != cudaSuccess) return cudaErrorNotSupported;
            mt.store(fa.maxThreadsPerBlock);
            if (getenv("SPC_PLAN_DEBUG"))
                fprintf(stderr, "ws kernel: regs %d maxThreadsPerBlock %d\n", fa.numRegs, fa.maxThreadsPerBlock);
        }
        if (32 * (T::NPROD + p.ncons) > mt.load()) return cudaErrorNotSupported;   // registers: round-1 kernel
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.strips, p.nkb, g.N * p.cg);
    cfg.blockDim = dim3(32 * (T::NPROD + p.ncons));
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = p.cg;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (getenv("SPC_PLAN_DEBUG"))
        fprintf(stderr, "ws plan: units %lld strips %d RT %d cons %d nkb %d cg %d smem %zu\n", p.units, p.strips, p.RT,
                p.ncons, p.nkb, p.cg, p.smem);
    return cudaLaunchKernelEx(&cfg, ws_conv_kernel<T>, wa);
}

// v2 configuration of a geometry (cudaErrorNotSupported: use the round-1 strip kernel).
template <class F>
static cudaError_t visit_ws_cfg(const Geom& g, F&& f) {
    // Per-shape choices, measured against each other and against the round-1 strip kernel
    // (tools/ab_conv.py, back to back over L2-cold buffer sets): 2x4 output tiles
    // x 4 channels per lane (14 consumer warps) on the 14x14 @ 256 layers, 4x4 tiles x 2
    // channels per lane (16 consumer warps, 16 outputs per tap load) on the K = 512 layers; the
    // 56x56 / 28x28 / cfg3-s2 shapes stay on the strip kernel (faster there).
    static const char* env = getenv("SPC_WS_CFG");   // development A/B: 1 = 2x4 x 4, 2 = 4x4 x 2 everywhere
    const int alt = env ? atoi(env) : 0;
    if (g.R == 3 && g.S == 3 && g.sh == 1 && g.sw == 1) {
        if (alt == 1) {
            if (g.K % 256 == 0 && g.Oh <= 14) return f(WsCfg<3, 3, 1, 1, 2, 4, 2, 4>{});
            if (g.K % 128 == 0 && g.Oh <= 28) return f(WsCfg<3, 3, 1, 1, 2, 4, 1, 4>{});
            if (g.K % 64 == 0 && g.Oh <= 56) return f(WsCfg<3, 3, 1, 1, 4, 2, 1, 4>{});
        } else if (alt == 2) {
            if (g.K % 256 == 0 && g.Oh <= 16) return f(WsCfg<3, 3, 1, 1, 4, 2, 4, 4>{});
            if (g.K % 128 == 0 && g.Oh <= 28) return f(WsCfg<3, 3, 1, 1, 4, 2, 2, 4>{});
            if (g.K % 64 == 0 && g.Oh <= 56) return f(WsCfg<3, 3, 1, 1, 4, 2, 1, 4>{});
        }
        if (g.K % 512 == 0 && g.Oh <= 8) return f(WsCfg<3, 3, 1, 1, 4, 2, 8, 2>{});                // 7x7 @ 512
        if (g.K % 256 == 0 && g.Oh <= 14) return f(WsCfg<3, 3, 1, 1, 2, 4, 2, 4>{});               // 14x14 @ 256
    } else if (g.R == 3 && g.S == 3 && g.sh == 2 && g.sw == 2) {
        if (g.K % 512 == 0 && g.Oh <= 8) return f(WsCfg<3, 3, 2, 2, 4, 2, 8, 2>{});                // 14 -> 7 @ 512
        if (g.K % 256 == 0 && g.Oh > 8 && g.Oh <= 14) return f(WsCfg<3, 3, 2, 2, 2, 4, 2, 4>{});   // 28 -> 14 @ 256
    }
    return cudaErrorNotSupported;
}
