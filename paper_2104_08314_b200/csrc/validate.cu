// validate.cu -- debug stream validator (SPC_ECORRUPT, SPEC.md:295 / :713).
//
// Checks that an encoding is a well-formed canonical CPO / CPS encoding of SOME dense map
// with the descriptor's geometry (DESIGN.md Appendix A; Alg. 1, Alg. 3
// :316-372, SI Alg. 5 :1346-1392), so that a foreign or corrupted encoding is rejected
// before the convolution indexes with it.  One thread per (n, c) channel segment walks its
// ptr blocks, IN and DA sequentially (a debug path, not the hot path):
//   * side tables: non-decreasing, totals equal the device lengths;
//   * ptr: NPC segments are exactly [NPC] with no NZEs; otherwise the block sequence of the
//     geometry (NOP iff pad_left = 0, then tags t+1 for t = max(1, pad_left) .. S-1, each
//     [t+1, NPF] or [t+1, c_0 .. c_{Ow1-1}] with -1 exactly where partition s owns no
//     column of type t and non-decreasing block-relative counts elsewhere; SI Alg. 5's
//     [0, c_0 ..] for S = 1); block totals add up to the channel's NZE count;
//   * IN (CPO form): local column == the column's local index, padded row inside the real
//     rows, rows strictly ascending within a column; CPS overlapK_w: negated singles or
//     {first index, pattern} pairs with >= 3 pattern bits inside the set4 of the first
//     index, in column / group order, decoding to the block's NZE count;
//   * DA: every value non-zero and finite (reading A21).
// The first failing channel (lowest index) and a reason code land in a 16-byte device record.
#include <cstdio>

#include "common.cuh"

namespace spc {
namespace {

enum : int {
    V_OK = 0, V_SIDE = 1, V_NPC = 2, V_TAG = 3, V_COUNT = 4, V_NEG = 5, V_TOTAL = 6, V_LOCAL = 7, V_ROW = 8,
    V_ORDER = 9, V_DA = 10, V_CPS = 11, V_LEN = 12
};

struct VRec {
    unsigned long long first;   // (channel << 8) | code of the lowest failing channel, or ~0
};

__device__ __forceinline__ int owner_of(const Geom& g, int w) { return max(0, w - g.S + 1); }
__device__ __forceinline__ int local_col(const Geom& g, int w) { return w - owner_of(g, w); }

// NZEs of one padded column (in stream order) against its IN entries (CPO form); returns a
// reason code.  rows must be strictly ascending and inside the real (unpadded) rows.
__device__ int check_column_cpo(const Geom& g, const int32_t* in, const float* da, int lo, int hi, int w) {
    int prev = -1;
    const int L = local_col(g, w);
    for (int i = lo; i < hi; i++) {
        const int e = in[i];
        if (e < 0 || e >= g.S * g.Hp) return V_ROW;
        if (e % g.S != L) return V_LOCAL;
        const int h = e / g.S;
        if (h < g.pt || h >= g.pt + g.H) return V_ROW;
        if (h <= prev) return V_ORDER;
        prev = h;
        const float v = da[i];
        if (!(v != 0.0f) || isinf(v) || isnan(v)) return V_DA;
    }
    return V_OK;
}

__global__ void validate_kernel(Geom g, const int32_t* __restrict__ ptr, const float* __restrict__ da,
                                const int32_t* __restrict__ in, const int64_t* __restrict__ cpo,
                                const int64_t* __restrict__ cnz, const int64_t* __restrict__ cin,
                                const int64_t* __restrict__ lengths, int64_t ptr_cap, int64_t da_cap,
                                int64_t in_cap, int cps, VRec* rec) {
    const long long nc = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (nc >= g.NC) return;
    auto fail = [&](int code) {
        atomicMin(&rec->first, ((unsigned long long)nc << 8) | (unsigned)code);
    };
    const long long P = cpo[nc], P1 = cpo[nc + 1], Z = cnz[nc], Z1 = cnz[nc + 1], Q = cin[nc], Q1 = cin[nc + 1];
    if (P < 0 || Z < 0 || Q < 0 || P1 <= P || Z1 < Z || Q1 < Q || P1 > ptr_cap || Z1 > da_cap || Q1 > in_cap) return fail(V_SIDE);
    if (nc == g.NC - 1 && (P1 != lengths[0] || Z1 != lengths[1] || Q1 != lengths[2])) return fail(V_SIDE);
    if (nc == 0 && (P != 0 || Z != 0 || Q != 0)) return fail(V_SIDE);
    const int32_t* seg = ptr + P;
    const int plen = (int)(P1 - P), nnz = (int)(Z1 - Z), nin = (int)(Q1 - Q);
    const int32_t* ii = in + Q;
    const float* dd = da + Z;
    if (seg[0] == SPC_NPC) {
        if (plen != 1 || nnz != 0 || nin != 0) return fail(V_NPC);
        return;
    }
    if (nnz == 0) return fail(V_NPC);   // a non-NPC channel holds at least one NZE
    const int Ow1 = g.Ow1;
    if (g.S == 1) {                     // SI Alg. 5: [0, c_0 .. c_{Ow1-1}], channel-cumulative
        if (plen != 1 + Ow1 || seg[0] != 0) return fail(V_TAG);
        if (nin != nnz) return fail(V_LEN);
        int prev = 0;
        for (int s = 0; s < Ow1; s++) {
            const int c = seg[1 + s];
            if (c < prev) return fail(V_COUNT);
            const int r = check_column_cpo(g, ii, dd, prev, c, s);
            if (r) return fail(r);
            prev = c;
        }
        if (prev != nnz) return fail(V_TOTAL);
        return;
    }
    int q = 0, dbase = 0, ibase = 0;
    auto col_cpo = [&](int lo, int hi, int w) -> int {   // DA / IN offsets within the channel
        return check_column_cpo(g, ii + ibase - dbase, dd, lo, hi, w);
    };
    if (g.pl == 0) {                                     // NOP [0, a, a+b]: col 0 then col Wp-1
        if (plen < 3 || seg[0] != 0) return fail(V_TAG);
        const int a = seg[1], ab = seg[2];
        if (a < 0 || ab < a || ab > nnz) return fail(V_COUNT);
        int r = col_cpo(0, a, 0);
        if (!r) r = col_cpo(a, ab, g.Wp - 1);
        if (r) return fail(r);
        dbase = ab; ibase = ab; q = 3;
    }
    for (int t = max(1, g.pl); t <= g.S - 1; t++) {
        if (q + 2 > plen || seg[q] != t + 1) return fail(V_TAG);
        if (seg[q + 1] == SPC_NPF) { q += 2; continue; }
        if (q + 1 + Ow1 > plen) return fail(V_LEN);
        const int32_t* c = seg + q + 1;
        const bool mid = (t == g.S - 1);
        int prev = 0;
        int total = 0;
        for (int s = 0; s < Ow1; s++) {
            // does partition s own a column of type t?  mid: s <= Ow1 - S; else s == 0 (left
            // column t) or s == Ow1-1-t (right column Wp-1-t)
            const bool owns = mid ? (s <= Ow1 - g.S) : (s == 0 || s == Ow1 - 1 - t);
            if (!owns) {
                if (c[s] != -1) return fail(V_NEG);
                continue;
            }
            if (c[s] < prev) return fail(V_COUNT);
            prev = c[s];
            total = c[s];
        }
        if (total <= 0 || dbase + total > nnz) return fail(V_TOTAL);
        if (!mid || !cps) {
            // CPO-form IN for this block: column by column
            int lo = 0;
            for (int s = 0; s < Ow1; s++) {
                const bool owns = mid ? (s <= Ow1 - g.S) : (s == 0 || s == Ow1 - 1 - t);
                if (!owns) continue;
                const int w = mid ? (s + g.S - 1) : (s == 0 ? t : g.Wp - 1 - t);
                const int r = col_cpo(dbase + lo, dbase + c[s], w);
                if (r) return fail(r);
                lo = c[s];
            }
            ibase += total;
        } else {
            // CPS overlapK_w (Alg. 3): per column, set4 groups in row order; negated singles
            // (k = 1, 2) or {first index, pattern} (k >= 3); decoded count == block count
            int lo = 0, e = 0;
            for (int s = 0; s <= Ow1 - g.S; s++) {
                const int want = c[s] - lo;
                int got = 0, prev_row = -1;
                while (got < want) {
                    if (ibase + e >= nin) return fail(V_CPS);
                    const int v = ii[ibase + e];
                    if (v < 0) {
                        const int x = -v;
                        if (x % g.S != g.S - 1) return fail(V_LOCAL);
                        const int h = x / g.S;
                        if (h <= prev_row || h < g.pt || h >= g.pt + g.H) return fail(V_ROW);
                        prev_row = h; got++; e++;
                    } else {
                        if (ibase + e + 1 >= nin) return fail(V_CPS);
                        const int pat = ii[ibase + e + 1];
                        if (v % g.S != g.S - 1) return fail(V_LOCAL);
                        const int h0 = v / g.S;
                        if (pat < 0 || pat > 15 || __popc(pat) < 3) return fail(V_CPS);
                        const int b0 = __ffs(pat) - 1;
                        if ((h0 & 3) != b0 || h0 <= prev_row) return fail(V_CPS);
                        const int grp = h0 - b0;
                        for (int b = 0; b < 4; b++)
                            if ((pat >> b) & 1) {
                                const int h = grp + b;
                                if (h < g.pt || h >= g.pt + g.H) return fail(V_ROW);
                                prev_row = h; got++;
                            }
                        e += 2;
                    }
                }
                if (got != want) return fail(V_CPS);
                for (int i = dbase + lo; i < dbase + c[s]; i++) {
                    const float v = dd[i];
                    if (!(v != 0.0f) || isinf(v) || isnan(v)) return fail(V_DA);
                }
                lo = c[s];
            }
            ibase += e;
        }
        dbase += total;
        q += 1 + Ow1;
    }
    if (q != plen) return fail(V_LEN);
    if (dbase != nnz) return fail(V_TOTAL);
    if (ibase != nin) return fail(V_LEN);
}

}  // namespace

const char* validate_reason(int code) {
    switch (code) {
        case V_SIDE: return "side tables inconsistent with the lengths / capacities";
        case V_NPC: return "NPC segment malformed (or a non-NPC channel without NZEs)";
        case V_TAG: return "ptr block tag / block sequence does not match the geometry";
        case V_COUNT: return "ptr counts decrease or exceed the channel's NZEs";
        case V_NEG: return "-1 / count placement does not match column ownership";
        case V_TOTAL: return "block totals do not add up to the channel's NZE count";
        case V_LOCAL: return "IN local column does not match the column type";
        case V_ROW: return "IN row outside the real rows";
        case V_ORDER: return "IN rows not strictly ascending within a column";
        case V_DA: return "DA value zero or not finite";
        case V_CPS: return "CPS pattern set malformed";
        case V_LEN: return "segment length mismatch";
        default: return "unknown";
    }
}

cudaError_t launch_validate(const Geom& g, const spc_encoding* e, void* rec_dev, cudaStream_t st,
                            long long* bad_channel, int* code) {
    VRec* rec = static_cast<VRec*>(rec_dev);
    cudaError_t err = cudaMemsetAsync(rec, 0xFF, sizeof(VRec), st);
    if (err != cudaSuccess) return err;
    const int threads = 128;
    const long long blocks = (g.NC + threads - 1) / threads;
    validate_kernel<<<(unsigned)blocks, threads, 0, st>>>(g, e->ptr, e->da, e->in, e->chan_ptr_off, e->chan_nz_off,
                                                          e->chan_in_off, e->lengths, e->ptr_cap, e->da_cap,
                                                          e->in_cap, e->algo == SPC_ALGO_CPS ? 1 : 0, rec);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    VRec h;
    err = cudaMemcpyAsync(&h, rec, sizeof h, cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) return err;
    if (h.first == ~0ull) {
        *bad_channel = -1;
        *code = 0;
    } else {
        *bad_channel = (long long)(h.first >> 8);
        *code = (int)(h.first & 0xFF);
    }
    return cudaSuccess;
}

}  // namespace spc
