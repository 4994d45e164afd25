// tile_conv.cuh -- register-tiled convSpMv over the CPO encoding (sm_100a).
// Included by sparse_conv.cu inside namespace spc (reuses DirS / parse_dir / column_range_s /
// ConvArgs / the mbarrier + bulk-copy helpers).
//
// What it computes: Alg. 2 convSpMv -- every NZE v at padded (h, w) of input
// channel c adds v * W[k, c, l, m] to output (h - l, w - m) for every output channel k; NPC
// channels and NPF blocks contribute nothing (they are never listed) -- exactly what
// strip_conv_kernel / ws_conv_kernel compute, stride 1 only.
//
// Why a third kernel.  At rho = 0.1 the other two kernels are bound by shared-memory tap loads:
// a lane reloads its taps W[k, c, :, :] for every input channel of every small output tile
// (2x4 or 4x4), and a loaded tap then serves TY*TX*rho < 2 multiply-adds, while the SM loads
// 32 floats per clock against 128 FMAs.  Here a lane owns a 7x7 output tile for two adjacent
// output channels (98 accumulators, FFMA2 on (k, k+1) pairs), so a tap serves ~49*rho ~ 5
// multiply-adds, and the walk is per NZE, not per window position: each NZE of the tile's
// 9x9 input window is one (case, value) entry, and `case` selects through a jump table the
// statically indexed FFMA2s of the outputs it reaches.
// (Measured: the per-NZE indirect branch -- a generated brx.idx jump table (git history) --
// is latency-bound at ~170 cycles per NZE per warp; the walk below is the dense-window nibble walk
// of ws_conv_kernel over the larger tile: forward uniform branches only.)
//  * consumer warp = (image, 7x7 tile) pair x 64 output channels; G <= 8 pairs per CTA share
//    the CTA's filter taps (one TMA bulk copy per chunk, not one load per tile);
//  * 4 producer warps: per chunk of CH input channels, TMA bulk copies of the taps and of the
//    chunk's ptr / DA / IN segments of every image the CTA's pairs touch, then lane (pair,
//    channel) parses the block directory and lists the NZEs of its window -- the CPO column
//    ranges and the row index h = IN / K_w (IN = Z + h*K_w, reading A8);
//  * NST-stage ring (full / empty mbarriers) between them;
//  * input channels split over a thread-block cluster of CS CTAs when the grid is below a wave;
//    the partial tiles are summed through distributed shared memory (no L2 round trip).

template <int R_, int S_, int TY_, int TX_>
struct TcCfg {
    static constexpr int R = R_, S = S_, TY = TY_, TX = TX_;
    static constexpr int RS = R * S;
    static constexpr int WH = TY + R - 1, WW = TX + S - 1;   // input window of a tile (stride 1)
    static constexpr int NCASE = WH * WW;
    static constexpr int NQ = (NCASE + 3) / 4;                // nibbles of the occupancy mask
    static constexpr int NCP = 4 * NQ;                        // window slots (floats, 16-byte rows)
    static constexpr int KW = 64;                             // output channels per consumer warp
    static constexpr int GMAX = 8;                            // consumer warps (pairs) per CTA
    static constexpr int CH = 4;                              // input channels per chunk (GMAX*CH = 32 lists)
    static constexpr int NPROD = 4, NST = 4;
    static constexpr int PCAP = 2048;                         // ptr ints a producer stages per chunk
    static constexpr int ECAP = 1536;                         // DA / IN entries a producer stages per chunk
    static constexpr int NIMG = 8;                            // images a CTA's pairs touch at most
    static constexpr int TT = TY * TX;
    static_assert(NCASE <= 128, "case switch covers 128 window positions");
    static_assert(GMAX * CH == 32, "one producer lane per list");
};

struct TcSmem {
    size_t wst, lst, cnt, pbuf, soff, sbase, stab, spair, bars, part, total;
    size_t stage_w, stage_l;   // bytes per stage
    size_t pb;                 // bytes per producer buffer
};
template <class T>
__host__ __device__ inline TcSmem tc_smem_layout(int G, int cslice, int nimg) {
    TcSmem L;
    L.stage_w = (size_t)T::CH * T::RS * T::KW * 4;
    L.stage_l = (size_t)32 * T::NCP * 4;
    L.pb = (size_t)(T::PCAP + 2 * T::ECAP + 3 * 8) * 4;
    L.wst = 0;                                                           // [NST][CH][RS][KW] taps
    L.lst = L.wst + (size_t)T::NST * L.stage_w;                          // [NST][32][NCP] window values
    L.cnt = L.lst + (size_t)T::NST * L.stage_l;                          // [NST][32][4] occupancy masks
    L.pbuf = align_up(L.cnt + (size_t)T::NST * 32 * 16, 16);            // [2] ptr | DA | IN (double-buffered)
    L.soff = L.pbuf + (size_t)2 * L.pb;                                  // [nimg][2][cslice+1] rel. offsets
    L.sbase = align_up(L.soff + (size_t)nimg * 2 * (cslice + 1) * 4, 16);   // [NIMG][2] int64 bases
    L.stab = L.sbase + (size_t)T::NIMG * 2 * 8;                          // [2][2*NIMG+1] staging table
    L.spair = align_up(L.stab + (size_t)2 * (2 * T::NIMG + 1) * 4, 16);  // [GMAX] int64 y base, [GMAX] int limits
    L.bars = align_up(L.spair + (size_t)T::GMAX * 12, 16);
    L.total = L.bars + (size_t)(2 * T::NST + 2) * 8;
    L.part = 0;                                                          // epilogue: [G][KW][TT] (aliases)
    const size_t part = (size_t)G * T::KW * T::TT * 4;
    if (part > L.soff) L.total = part + L.total;                         // (never for 3x3 / 7x7)
    return L;
}

// The FFMA2s of window position P (a constant after unrolling): outputs (P/WW - l, P%WW - m).
template <class T>
__device__ __forceinline__ void tc_tap(int P, float v, float2 (&acc)[T::TY][T::TX], const float2 (&w)[T::R][T::S]) {
    const int hr = P / T::WW, wr = P % T::WW;
    const float2 vv = make_float2(v, v);
#pragma unroll
    for (int l = 0; l < T::R; ++l)
#pragma unroll
        for (int m = 0; m < T::S; ++m) {
            const int y1 = hr - l, x1 = wr - m;
            if (y1 >= 0 && x1 >= 0 && y1 < T::TY && x1 < T::TX) acc[y1][x1] = __ffma2_rn(vv, w[l][m], acc[y1][x1]);
        }
}

struct TcArgs {
    ConvArgs a;
    int G;          // consumer warps (pairs) per CTA
    int npairs;     // N * tiles
    int tiles_x, ntiles;
    int cs;         // cluster size (input-channel split)
    int cslice;     // input channels per cluster rank
    int nimg;       // images a CTA's pairs touch at most (side-table rows)
    int dbg;        // development phase switch (SPC_TC_DBG): 1 no walk, 2 no lists, 4 no reduction
};

template <class T>
__global__ void __launch_bounds__(32 * (T::NPROD + T::GMAX), 1) tile_conv_kernel(TcArgs ta) {
    namespace cgrp = cooperative_groups;
    const ConvArgs& a = ta.a;
    const Geom& g = a.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = ta.G, CS = ta.cs;
    const bool producer = warp >= G;   // producers = the highest warp ids (the scheduler prefers them)
    const int rank = (CS > 1) ? (int)cgrp::this_cluster().block_rank() : 0;
    const int gbase = blockIdx.x * G;
    const int kbase = blockIdx.y * T::KW;
    const int c_begin = min(g.C, rank * ta.cslice), c_end = min(g.C, c_begin + ta.cslice);
    const int crange = c_end - c_begin;
    const int nchunks = (crange + T::CH - 1) / T::CH;
    const int n_lo = gbase / ta.ntiles;
    const int n_hi = min(ta.npairs - 1, gbase + G - 1) / ta.ntiles;
    const int nimg = n_hi - n_lo + 1;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const TcSmem L = tc_smem_layout<T>(G, ta.cslice, ta.nimg);
    float* s_w = reinterpret_cast<float*>(smem_raw + L.wst);
    float* s_win = reinterpret_cast<float*>(smem_raw + L.lst);
    unsigned* s_msk = reinterpret_cast<unsigned*>(smem_raw + L.cnt);
    int* s_off = reinterpret_cast<int*>(smem_raw + L.soff);                   // [q][0: ptr, 1: DA][cslice+1]
    long long* s_base = reinterpret_cast<long long*>(smem_raw + L.sbase);    // [q][2]
    int* s_tab = reinterpret_cast<int*>(smem_raw + L.stab);                  // [b][2*NIMG+1]
    long long* s_pyb = reinterpret_cast<long long*>(smem_raw + L.spair);     // [g] y offset of (n, 0, oy0, ox0)
    int* s_plim = reinterpret_cast<int*>(s_pyb + T::GMAX);                   // [g] valid rows << 8 | cols (0: none)
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem_raw + L.bars);
    unsigned long long* empty = full + T::NST;
    unsigned long long* pbar = empty + T::NST;
    const int orow = ta.cslice + 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < T::NST; s++) {
            mbar_init(&full[s], 2);      // the taps' expect_tx arrival + the lists' arrival
            mbar_init(&empty[s], G);     // one arrival per consumer warp
        }
        for (int b = 0; b < 2; b++) mbar_init(&pbar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x == 0) probe_any(0);
    if ((int)threadIdx.x < T::GMAX) {   // output placement of the CTA's pairs (epilogue)
        const int pg = gbase + (int)threadIdx.x;
        long long yb = 0;
        int lim = 0;
        if ((int)threadIdx.x < G && pg < ta.npairs) {
            const int n = pg / ta.ntiles, t = pg - n * ta.ntiles;
            const int ty = t / ta.tiles_x, tx = t - ty * ta.tiles_x;
            const int oy0 = ty * T::TY, ox0 = tx * T::TX;
            yb = (long long)n * g.K * g.Oh * g.Ow + (long long)oy0 * g.Ow + ox0;
            lim = (min(T::TY, g.Oh - oy0) << 8) | min(T::TX, g.Ow - ox0);
        }
        s_pyb[threadIdx.x] = yb;
        s_plim[threadIdx.x] = lim;
    }
    __syncthreads();

    // taps of chunk i -> stage i % NST (TMA bulk): [CH][RS][KW], rows of KW floats
    auto issue_taps = [&](int i) {   // one thread
        const int s = i % T::NST;
        const int c0 = c_begin + i * T::CH, chn = min(T::CH, c_end - c0);
        float* dst = s_w + (size_t)s * T::CH * T::RS * T::KW;
        const int rows = chn * T::RS;
        mbar_expect_tx(&full[s], (unsigned)(rows * T::KW * 4));
        if (g.K == T::KW) {
            bulk_g2s(dst, a.wp + (size_t)c0 * T::RS * T::KW, (unsigned)(rows * T::KW * 4), &full[s]);
        } else {
            for (int r = 0; r < rows; r++)
                bulk_g2s(dst + (size_t)r * T::KW, a.wp + ((size_t)c0 * T::RS + r) * g.K + kbase, T::KW * 4, &full[s]);
        }
    };

    static_assert(T::NCASE <= 96, "occupancy mask: 3 words");
    float2 acc[T::TY][T::TX];   // (k, k+1) accumulator pairs of output (yy, xx)
#pragma unroll
    for (int yy = 0; yy < T::TY; yy++)
#pragma unroll
        for (int xx = 0; xx < T::TX; xx++) acc[yy][xx] = make_float2(0.f, 0.f);

    const int cw = warp;   // consumer index = pair slot
    if (producer) {
        // The 4 producer warps work on one chunk at a time: thread 0 stages (TMA bulk copies of
        // the taps and of the chunk's ptr / DA / IN segments, double-buffered two chunks ahead),
        // and every producer thread takes (list, window column) tasks of the chunk's decode.
        const int p = warp - G;
        const int ptid = (int)threadIdx.x - 32 * G;
        constexpr int NPT = 32 * T::NPROD;
        if (ptid == 0)
            for (int i = 0; i < min(T::NST, nchunks); i++) issue_taps(i);
        pdl_wait();
        if (ptid == 0) probe_any(1);
        const bool bad = *reinterpret_cast<volatile unsigned long long*>(a.status) != 0ull;
        // side tables of the CTA's images x channel range, once (relative to the range start)
        for (int q = 0; q < nimg && !bad; q++) {
            const long long ncb = (long long)(n_lo + q) * g.C + c_begin;
            const long long pb0 = __ldg(a.cpo_off + ncb), zb0 = __ldg(a.cnz_off + ncb);
            for (int r = ptid; r <= crange; r += NPT) {
                s_off[(q * 2 + 0) * orow + r] = (int)(__ldg(a.cpo_off + ncb + r) - pb0);
                s_off[(q * 2 + 1) * orow + r] = (int)(__ldg(a.cnz_off + ncb + r) - zb0);
            }
            if (ptid == 0) { s_base[2 * q] = pb0; s_base[2 * q + 1] = zb0; }
        }
        producer_sync();
        if (ptid == 0) probe_any(2);
        auto sb_ptr = [&](int b) { return reinterpret_cast<int*>(smem_raw + L.pbuf + (size_t)b * L.pb); };
        auto sb_da = [&](int b) { return reinterpret_cast<float*>(sb_ptr(b) + T::PCAP + 8); };
        auto sb_in = [&](int b) { return reinterpret_cast<int*>(sb_da(b) + T::ECAP + 8); };
        // chunk i -> buffer i & 1 (thread 0): per image q, the buffer index of the chunk's first
        // ptr / DA entry, and whether everything fit (else the decode reads global memory)
        auto stage = [&](int i) {
            const int b = i & 1;
            int* tb = s_tab + b * (2 * T::NIMG + 1);
            const int c0 = c_begin + i * T::CH, chn = min(T::CH, c_end - c0), r0 = c0 - c_begin;
            int ptot = 0, ztot = 0;
            unsigned bytes = 0;
            for (int q = 0; q < nimg && !bad; q++) {
                const long long P0 = s_base[2 * q] + s_off[(q * 2) * orow + r0];
                const long long P1 = s_base[2 * q] + s_off[(q * 2) * orow + r0 + chn];
                const long long Z0 = s_base[2 * q + 1] + s_off[(q * 2 + 1) * orow + r0];
                const long long Z1 = s_base[2 * q + 1] + s_off[(q * 2 + 1) * orow + r0 + chn];
                const int pn = (int)(P1 - (P0 & ~3ll)), zn = (int)(Z1 - (Z0 & ~3ll));
                tb[2 * q] = ptot + (int)(P0 & 3ll);
                tb[2 * q + 1] = ztot + (int)(Z0 & 3ll);
                ptot += (pn + 3) & ~3;
                ztot += (zn + 3) & ~3;
                bytes += 4u * (unsigned)((pn & ~3) + 2 * (zn & ~3));
            }
            const bool fits = !bad && ptot <= T::PCAP && ztot <= T::ECAP && !(ta.dbg & 8);
            tb[2 * T::NIMG] = fits;
            mbar_expect_tx(&pbar[b], fits ? bytes : 0u);
            if (!fits) return;
            int po = 0, zo = 0;
            for (int q = 0; q < nimg; q++) {
                const long long P0 = (s_base[2 * q] + s_off[(q * 2) * orow + r0]) & ~3ll;
                const long long P1 = s_base[2 * q] + s_off[(q * 2) * orow + r0 + chn];
                const long long Z0 = (s_base[2 * q + 1] + s_off[(q * 2 + 1) * orow + r0]) & ~3ll;
                const long long Z1 = s_base[2 * q + 1] + s_off[(q * 2 + 1) * orow + r0 + chn];
                const int pn = (int)(P1 - P0), zn = (int)(Z1 - Z0);
                const int pbk = pn & ~3, zbk = zn & ~3;
                if (pbk) bulk_g2s(sb_ptr(b) + po, a.ptr + P0, 4u * pbk, &pbar[b]);
                if (zbk) {
                    bulk_g2s(sb_da(b) + zo, a.da + Z0, 4u * zbk, &pbar[b]);
                    bulk_g2s(sb_in(b) + zo, a.in + Z0, 4u * zbk, &pbar[b]);
                }
                for (int t = pbk; t < pn; t++) sb_ptr(b)[po + t] = __ldg(a.ptr + P0 + t);
                for (int t = zbk; t < zn; t++) {
                    sb_da(b)[zo + t] = __ldg(a.da + Z0 + t);
                    sb_in(b)[zo + t] = __ldg(a.in + Z0 + t);
                }
                po += (pn + 3) & ~3;
                zo += (zn + 3) & ~3;
            }
        };
        if (ptid == 0) {
            stage(0);
            if (nchunks > 1) stage(1);
        }
        for (int i = 0; i < nchunks; i++) {
            const int s = i % T::NST, b = i & 1;
            const unsigned ph = (unsigned)(i / T::NST) & 1u;
            const int c0 = c_begin + i * T::CH, chn = min(T::CH, c_end - c0), r0 = c0 - c_begin;
            if (i >= T::NST) mbar_wait(&empty[s], ph ^ 1u);   // the consumers released stage s
            if (ptid == 0 && i >= T::NST) issue_taps(i);
            if (ptid == 0 && i < 2) probe_any(3 + 3 * i);
            for (int l = ptid; l < 32 * 4; l += NPT) s_msk[(size_t)s * 128 + l] = 0u;
            mbar_wait(&pbar[b], (unsigned)(i >> 1) & 1u);
            producer_sync();   // masks cleared; the staged segments (and their tails) visible
            if (ptid == 0 && i < 2) probe_any(4 + 3 * i);
            const int* tb = s_tab + b * (2 * T::NIMG + 1);
            const bool fits = tb[2 * T::NIMG] != 0;
            // task = (list l = pair slot * CH + channel, window column): the NZEs of one column of
            // one window go to the dense window slots P = dy*WW + dx, bit P of the list's mask
            for (int t = ptid; t < 32 * T::WW; t += NPT) {
                const int l = t / T::WW, col = t - l * T::WW;
                const int gl = l / T::CH, j = l - gl * T::CH;
                const int pg = gbase + gl;
                if (bad || (ta.dbg & 2) || gl >= G || pg >= ta.npairs || j >= chn) continue;
                const int n = pg / ta.ntiles, tt = pg - n * ta.ntiles;
                const int q = n - n_lo;
                const int ty = tt / ta.tiles_x, tx = tt - ty * ta.tiles_x;
                const int hy0 = ty * T::TY, wx = tx * T::TX + col;   // padded window origin row, column
                const int pcur = s_off[(q * 2) * orow + r0 + j], zcur = s_off[(q * 2 + 1) * orow + r0 + j];
                const int32_t* seg;
                const float* da;
                const int32_t* in;
                if (fits) {
                    seg = sb_ptr(b) + tb[2 * q] + (pcur - s_off[(q * 2) * orow + r0]);
                    const int zr = tb[2 * q + 1] + (zcur - s_off[(q * 2 + 1) * orow + r0]);
                    da = sb_da(b) + zr;
                    in = sb_in(b) + zr;
                } else {
                    seg = a.ptr + s_base[2 * q] + pcur;
                    da = a.da + s_base[2 * q + 1] + zcur;
                    in = a.in + s_base[2 * q + 1] + zcur;
                }
                DirS<T::S> d;
                parse_dir<T::S>(g, seg, d);
                if (d.npc) continue;
                int lo, hi;
                column_range_s<T::S>(g, seg, d, wx, lo, hi);
                float* win = s_win + ((size_t)s * 32 + l) * T::NCP;
                unsigned* mk = s_msk + ((size_t)s * 32 + l) * 4;
                for (int z0 = lo; z0 < hi; z0 += 4) {
                    int hh[4];
                    float vv[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const bool ok = z0 + u < hi;
                        hh[u] = ok ? in[z0 + u] / T::S - hy0 : -1;   // IN = Z + h*K_w, Z < K_w (A8)
                        vv[u] = ok ? da[z0 + u] : 0.f;
                    }
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        if (hh[u] >= 0 && hh[u] < T::WH) {
                            const int P = hh[u] * T::WW + col;
                            win[P] = vv[u];
                            atomicOr(mk + (P >> 5), 1u << (P & 31));
                        }
                }
            }
            producer_sync();   // the stage's windows and masks are complete
            if (ptid == 0) {
                if (i < 2) probe_any(5 + 3 * i);
                ws_mbar_arrive(&full[s]);   // release: windows visible to the consumers
                if (i + 2 < nchunks) {
                    fence_proxy_async();    // the decode's generic reads of buffer b before the copies
                    stage(i + 2);
                }
            }
        }
    } else {
        const int pg = gbase + cw;
        const bool active = cw < G && pg < ta.npairs;
        const float* wl = s_w + 2 * lane;
        for (int i = 0; i < nchunks; i++) {
            const int s = i % T::NST;
            const unsigned ph = (unsigned)(i / T::NST) & 1u;
            const int chn = min(T::CH, c_end - (c_begin + i * T::CH));
            mbar_wait(&full[s], ph);
            if (cw == 0 && lane == 0 && i == 0) probe_any(9);
            if (active && !(ta.dbg & 1)) {
                for (int j = 0; j < chn; j++) {
                    const int li = s * 32 + cw * T::CH + j;
                    const uint4 mk = *reinterpret_cast<const uint4*>(s_msk + (size_t)li * 4);
                    if ((mk.x | mk.y | mk.z) == 0u) continue;
                    float2 w[T::R][T::S];
                    const float* ws = wl + ((size_t)s * T::CH + j) * T::RS * T::KW;
#pragma unroll
                    for (int l = 0; l < T::R; l++)
#pragma unroll
                        for (int m = 0; m < T::S; m++) w[l][m] = *reinterpret_cast<const float2*>(ws + (l * T::S + m) * T::KW);
                    const float4* w4 = reinterpret_cast<const float4*>(s_win + (size_t)li * T::NCP);
                    constexpr int PD = 4;   // window loads in flight ahead of the walk (LDS latency)
                    float4 vb[PD];
#pragma unroll
                    for (int q = 0; q < PD; q++) vb[q] = lds128(w4 + q);
#pragma unroll
                    for (int q = 0; q < T::NQ; q++) {
                        const unsigned word = (q < 8) ? mk.x : (q < 16) ? mk.y : mk.z;
                        const unsigned nib = (word >> ((q & 7) * 4)) & 0xFu;
                        const float4 v4 = vb[q % PD];
                        if (q + PD < T::NQ) vb[q % PD] = lds128(w4 + q + PD);   // issued ahead of the skip branch
                        if (nib) {
                            const float vq[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                            for (int u = 0; u < 4; u++)
                                if (4 * q + u < T::NCASE && ((nib >> u) & 1u)) tc_tap<T>(4 * q + u, vq[u], acc, w);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) ws_mbar_arrive(&empty[s]);
        }
        if (cw == 0 && lane == 0) probe_any(10);
        pdl_wait();   // y may still be read by the previous grid
    }

    // ---- epilogue: partial tiles [G][KW][TT] in smem (aliasing the ring), summed over the
    // cluster's ranks through distributed shared memory, stored coalesced along output rows
    __syncthreads();
    float* part = reinterpret_cast<float*>(smem_raw + L.part);
    if (!producer && cw < G) {
#pragma unroll
        for (int yy = 0; yy < T::TY; yy++)
#pragma unroll
            for (int xx = 0; xx < T::TX; xx++) {
                part[((size_t)cw * T::KW + 2 * lane) * T::TT + yy * T::TX + xx] = acc[yy][xx].x;
                part[((size_t)cw * T::KW + 2 * lane + 1) * T::TT + yy * T::TX + xx] = acc[yy][xx].y;
            }
    }
    if (threadIdx.x == 0) probe_any(11);
    if (CS > 1) cgrp::this_cluster().sync();
    else __syncthreads();
    if (threadIdx.x == 0) probe_any(12);
    const int total4 = G * T::KW * T::TT / 4;   // float4 items (KW*TT is a multiple of 4)
    const int per = (total4 + CS - 1) / CS;
    const int e0 = rank * per, e1 = min(total4, e0 + per);
    const float4* part4 = reinterpret_cast<const float4*>(part);
    for (int e = e0 + (int)threadIdx.x; e < e1; e += (int)blockDim.x) {
        float4 v = part4[e];
        if (CS > 1 && !(ta.dbg & 4)) {
            float4 rv[7];
#pragma unroll
            for (int r = 1; r < 8; r++)
                if (r < CS) rv[r - 1] = cgrp::this_cluster().map_shared_rank(part4, (rank + r) % CS)[e];
#pragma unroll
            for (int r = 1; r < 8; r++)
                if (r < CS) { v.x += rv[r - 1].x; v.y += rv[r - 1].y; v.z += rv[r - 1].z; v.w += rv[r - 1].w; }
        }
        const float sv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int el = 4 * e + u;
            const int gl = el / (T::KW * T::TT), rem = el - gl * (T::KW * T::TT);   // compile-time divisors
            const int kl = rem / T::TT, pos = rem - kl * T::TT;
            const int yy = pos / T::TX, xx = pos - yy * T::TX;
            const int lim = s_plim[gl];
            const int k = kbase + kl;
            if (yy >= (lim >> 8) || xx >= (lim & 0xFF) || k >= g.K) continue;
            float o = sv[u];
            if (a.relu) o = fmaxf(o, 0.f);
            const long long yo = s_pyb[gl] + (long long)k * g.Oh * g.Ow + (long long)yy * g.Ow + xx;
            a.y[yo] = o;
            if (a.omask && o != 0.0f) {
                const long long img = s_pyb[gl] / ((long long)g.K * g.Oh * g.Ow);
                const int oy = (int)((s_pyb[gl] - img * g.K * g.Oh * g.Ow) / g.Ow) + yy;
                const int ox = (int)((s_pyb[gl] - img * g.K * g.Oh * g.Ow) % g.Ow) + xx;
                atomicOr(a.omask + (img * g.K + k) * g.Ow + ox, 1ull << oy);
            }
        }
    }
    if (threadIdx.x == 0) probe_any(13);
    if (CS > 1) cgrp::this_cluster().sync();   // remote partials stay alive until every rank has read them
}

template <class T>
struct TcPlan {
    int G, ngroups, nkb, cs, cslice, tiles_x, tiles_y, ntiles, npairs, nimg;
    size_t smem;
};

template <class T>
static bool plan_tc(const Geom& g, TcPlan<T>& p, int G) {
    if (g.sh != 1 || g.sw != 1 || g.R != T::R || g.S != T::S) return false;
    if (g.K % T::KW != 0) return false;
    p.tiles_x = (g.Ow + T::TX - 1) / T::TX;
    p.tiles_y = (g.Oh + T::TY - 1) / T::TY;
    p.ntiles = p.tiles_x * p.tiles_y;
    p.npairs = g.N * p.ntiles;
    p.nkb = g.K / T::KW;
    const int sms = device_sm_count();
    static const int env_cs = [] { const char* v = getenv("SPC_TC_CS"); return v ? atoi(v) : 0; }();
    p.G = G;
    p.ngroups = (p.npairs + p.G - 1) / p.G;
    const long long units = (long long)p.ngroups * p.nkb;
    p.cs = 1;
    for (int cs = 2; cs <= 8; cs *= 2)
        if (units * cs <= sms && g.C >= 2 * cs * T::CH) p.cs = cs;
    if (env_cs) p.cs = env_cs;
    p.cslice = (g.C + p.cs - 1) / p.cs;
    // images a group of G consecutive pairs touches
    p.nimg = (p.G + p.ntiles - 2) / p.ntiles + 1;
    if (p.nimg > T::NIMG) return false;
    p.smem = tc_smem_layout<T>(p.G, p.cslice, p.nimg).total;
    return p.smem <= 227 * 1024;
}

// Halve the cluster split until the grid's clusters are co-resident (B200: 15 clusters of 8 CTAs
// at this kernel's 1 CTA / SM, not 148 / 8).
template <class T>
static bool fit_clusters(const Geom& g, TcPlan<T>& p) {
    static std::atomic<int> max_clusters[kMaxDevices][T::GMAX + 1][4];   // [G][cs = 1, 2, 4, 8]
    while (p.cs > 1) {
        const int ci = p.cs == 2 ? 1 : p.cs == 4 ? 2 : 3;
        std::atomic<int>& mc = max_clusters[current_device()][p.G][ci];
        if (mc.load() == 0) {
            cudaLaunchConfig_t qc = {};
            qc.gridDim = dim3(p.ngroups, p.nkb, p.cs);
            qc.blockDim = dim3(32 * (T::NPROD + p.G));
            qc.dynamicSmemBytes = p.smem;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = 1;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = p.cs;
            qc.attrs = qa;
            qc.numAttrs = 1;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, (const void*)tile_conv_kernel<T>, &qc) != cudaSuccess || n <= 0) n = 1;
            mc.store(n);
        }
        if ((long long)p.ngroups * p.nkb <= mc.load()) break;
        p.cs /= 2;
        p.cslice = (g.C + p.cs - 1) / p.cs;
        p.smem = tc_smem_layout<T>(p.G, p.cslice, p.nimg).total;
        if (p.smem > 227 * 1024) return false;
    }
    return true;
}

template <class T>
static cudaError_t run_tc(ConvArgs& a, cudaStream_t st) {
    const Geom& g = a.g;
    if (a.cscc || a.sa_types) return cudaErrorNotSupported;
    static std::atomic<size_t> attr_bytes[kMaxDevices];
    cudaError_t err = ensure_smem_attr((const void*)tile_conv_kernel<T>, 227 * 1024, attr_bytes);
    if (err != cudaSuccess) return err;
    // pairs per CTA: 8 (more CTAs share a tap copy) unless 4 gives a fuller grid
    static const int env_g = [] { const char* v = getenv("SPC_TC_G"); return v ? atoi(v) : 0; }();
    TcPlan<T> p;
    bool ok = false;
    for (int G : {T::GMAX, T::GMAX / 2}) {
        if (env_g && G != env_g) continue;
        TcPlan<T> c;
        if (!plan_tc<T>(g, c, G) || !fit_clusters<T>(g, c)) continue;
        if (!ok || (long long)c.ngroups * c.nkb * c.cs > (long long)p.ngroups * p.nkb * p.cs) p = c;
        ok = true;
    }
    if (env_g && !ok) {
        TcPlan<T> c;
        if (plan_tc<T>(g, c, std::max(1, std::min(T::GMAX, env_g))) && fit_clusters<T>(g, c)) { p = c; ok = true; }
    }
    if (!ok) return cudaErrorNotSupported;
    TcArgs ta;
    ta.nimg = p.nimg;
    static const int env_dbg = [] { const char* v = getenv("SPC_TC_DBG"); return v ? atoi(v) : 0; }();
    ta.dbg = env_dbg;
    ta.a = a;
    ta.G = p.G;
    ta.npairs = p.npairs;
    ta.tiles_x = p.tiles_x;
    ta.ntiles = p.ntiles;
    ta.cs = p.cs;
    ta.cslice = p.cslice;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.ngroups, p.nkb, p.cs);
    cfg.blockDim = dim3(32 * (T::NPROD + p.G));
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = p.cs;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (getenv("SPC_PLAN_DEBUG")) {
        int nclu = -1;
        cudaOccupancyMaxActiveClusters(&nclu, (const void*)tile_conv_kernel<T>, &cfg);
        fprintf(stderr, "tc plan: pairs %d G %d groups %d nkb %d cs %d cslice %d smem %zu max_active_clusters %d\n",
                p.npairs, p.G, p.ngroups, p.nkb, p.cs, p.cslice, p.smem, nclu);
    }
    return cudaLaunchKernelEx(&cfg, tile_conv_kernel<T>, ta);
}

// register-tiled configuration of a geometry (cudaErrorNotSupported: the other kernels run)
template <class F>
static cudaError_t visit_tc_cfg(const Geom& g, F&& f) {
    // development switch: SPC_TC=1 runs this kernel (measured slower than ws_conv_kernel on every
    // layer, DESIGN.md §7 "register-tiled conv"); off by default
    static const char* env = getenv("SPC_TC");
    if (!env || atoi(env) == 0) return cudaErrorNotSupported;
    if (g.R == 3 && g.S == 3 && g.sh == 1 && g.sw == 1) return f(TcCfg<3, 3, 7, 7>{});
    return cudaErrorNotSupported;
}
