/*
 * oracle.c -- plain, slow, single-threaded CPU oracle for arXiv 2104.08314
 *             (CPO / CPS sparse-activation convolution).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2104_08314_b200/), and never includes anything from it.
 *
 * Every function follows the paper's definition or algorithm in the paper's
 * order and notation; "PAPER.md:<line>" cites the passage, "reading Ax" cites
 * the DESIGN.md / SURVEY.md §8(c) reading of an ambiguous passage.
 *
 * Floating point: convolution results accumulate in FP64 (products of two
 * fp32 values are exact in FP64); encodings copy fp32 bits verbatim.
 * An element is a non-zero element (NZE) iff I(h,w) != 0,
 * evaluated in IEEE fp32 (-0.0 is zero; denormals are NZEs; reading A21).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OC_NPC ((int32_t)INT32_MIN)       /* No Ptr Channel, reading A7 */
#define OC_NPF ((int32_t)(INT32_MIN + 1)) /* No Ptr Flag, reading A7 */

/* Problem statement (Table 1): I is I_n x I_c x I_h x I_w here
 * in NCHW order; W is K x I_c x K_h x K_w (KCRS); strides s_h, s_w; zero
 * padding (top, bottom, left, right). */
typedef struct {
    int32_t N, C, H, W, K, R, S;
    int32_t sh, sw, pt, pb, pl, pr;
} oc_desc;

/* ---------------------------------------------------------------- geometry */

/* Output size O = 1 + (I - K)/s; with padding and a stride
 * that does not divide, floor (reading A14). */
static int32_t out_dim(int32_t in, int32_t p0, int32_t p1, int32_t k, int32_t s)
{
    return (in + p0 + p1 - k) / s + 1;
}

int32_t oc_out_h(const oc_desc *d) { return out_dim(d->H, d->pt, d->pb, d->R, d->sh); }
int32_t oc_out_w(const oc_desc *d) { return out_dim(d->W, d->pl, d->pr, d->S, d->sw); }

/* I(h, w) of one channel plane in the zero-padded frame (reading A8). */
static float I_at(const float *plane, const oc_desc *d, int32_t h, int32_t w)
{
    int32_t hh = h - d->pt, ww = w - d->pl;
    if (hh < 0 || hh >= d->H || ww < 0 || ww >= d->W) return 0.0f;
    return plane[(size_t)hh * d->W + ww];
}

static const float *plane_of(const float *x, const oc_desc *d, int32_t n, int32_t c)
{
    return x + ((size_t)n * d->C + c) * (size_t)d->H * d->W;
}

/* ------------------------------------------------ Eq. 1: direct convolution */

/* O(n,y,x,k) = sum_c sum_h sum_w I(n,c,y*s_h+h, x*s_w+w) W(h,w,c,k)
 * (Eq. 1), accumulated in FP64.  y is NKHW (Oh x Ow). */
void oc_direct_conv(const oc_desc *d, const float *x, const float *w, double *y)
{
    int32_t Oh = oc_out_h(d), Ow = oc_out_w(d);
    for (int32_t n = 0; n < d->N; n++)
        for (int32_t k = 0; k < d->K; k++)
            for (int32_t oy = 0; oy < Oh; oy++)
                for (int32_t ox = 0; ox < Ow; ox++) {
                    double acc = 0.0;
                    for (int32_t c = 0; c < d->C; c++) {
                        const float *pl = plane_of(x, d, n, c);
                        for (int32_t h = 0; h < d->R; h++)
                            for (int32_t ww = 0; ww < d->S; ww++)
                                acc += (double)I_at(pl, d, oy * d->sh + h, ox * d->sw + ww) *
                                       (double)w[(((size_t)k * d->C + c) * d->R + h) * d->S + ww];
                    }
                    y[(((size_t)n * d->K + k) * Oh + oy) * Ow + ox] = acc;
                }
}

/* Eq. 1 at a list of output coordinates idx[i] = {n, k, y, x} (for parity at
 * full size, where the whole output would take the oracle too long). */
void oc_direct_conv_at(const oc_desc *d, const float *x, const float *w, const int32_t *idx, int64_t count,
                       double *out)
{
    for (int64_t i = 0; i < count; i++) {
        int32_t n = idx[4 * i], k = idx[4 * i + 1], oy = idx[4 * i + 2], ox = idx[4 * i + 3];
        double acc = 0.0;
        for (int32_t c = 0; c < d->C; c++) {
            const float *pl = plane_of(x, d, n, c);
            for (int32_t h = 0; h < d->R; h++)
                for (int32_t ww = 0; ww < d->S; ww++)
                    acc += (double)I_at(pl, d, oy * d->sh + h, ox * d->sw + ww) *
                           (double)w[(((size_t)k * d->C + c) * d->R + h) * d->S + ww];
        }
        out[i] = acc;
    }
}

/* ---------------------------------------------- im2col lowering */

/* im2col: each kernel-sized patch of every channel becomes one row of the
 * lowered matrix; per image the matrix is (Oh*Ow) x (C*R*S),
 * element count SI Eq. 6.  L is [N][Oh*Ow][C*R*S]. */
int64_t oc_im2col(const oc_desc *d, const float *x, float *L)
{
    int32_t Oh = oc_out_h(d), Ow = oc_out_w(d);
    int64_t cols = (int64_t)d->C * d->R * d->S, idx = 0;
    for (int32_t n = 0; n < d->N; n++)
        for (int32_t oy = 0; oy < Oh; oy++)
            for (int32_t ox = 0; ox < Ow; ox++)
                for (int32_t c = 0; c < d->C; c++) {
                    const float *pl = plane_of(x, d, n, c);
                    for (int32_t h = 0; h < d->R; h++)
                        for (int32_t ww = 0; ww < d->S; ww++)
                            L[idx++] = I_at(pl, d, oy * d->sh + h, ox * d->sw + ww);
                }
    (void)cols;
    return idx; /* number of elements materialised */
}

/* Naive GEMM on the lowered matrix: y[n,k,p] = sum_j L[n][p][j] * W[k][j]. */
void oc_gemm_lowered(const oc_desc *d, const float *L, const float *w, double *y)
{
    int32_t Oh = oc_out_h(d), Ow = oc_out_w(d);
    int64_t P = (int64_t)Oh * Ow, J = (int64_t)d->C * d->R * d->S;
    for (int32_t n = 0; n < d->N; n++)
        for (int32_t k = 0; k < d->K; k++)
            for (int64_t p = 0; p < P; p++) {
                double acc = 0.0;
                const float *row = L + ((size_t)n * P + p) * J;
                for (int64_t j = 0; j < J; j++) acc += (double)row[j] * (double)w[(size_t)k * J + j];
                y[((size_t)n * d->K + k) * P + p] = acc;
            }
}

/* MEC lowering: O_w horizontal partitions of I_h x K_w, each one
 * row; per channel O_w x (I_h*K_w) elements, SI Eq. 11.
 * The padded height is used (MEC lowers the padded map).  M is [N][C][Ow][Hp*S]. */
int64_t oc_mec_lower(const oc_desc *d, const float *x, float *M)
{
    int32_t Ow = oc_out_w(d), Hp = d->H + d->pt + d->pb;
    int64_t idx = 0;
    for (int32_t n = 0; n < d->N; n++)
        for (int32_t c = 0; c < d->C; c++) {
            const float *pl = plane_of(x, d, n, c);
            for (int32_t s = 0; s < Ow; s++)            /* partition s, separated by s_w */
                for (int32_t h = 0; h < Hp; h++)
                    for (int32_t ww = 0; ww < d->S; ww++)
                        M[idx++] = I_at(pl, d, h, s * d->sw + ww);
        }
    return idx;
}

/* --------------------------------------------------- CPO / CPS encoding */

typedef struct {
    int32_t *ptr; float *da; int32_t *in;
    int64_t cap_ptr, cap_da, cap_in;
    int64_t n_ptr, n_da, n_in;
    int overflow;
} oc_streams;

static void push_ptr(oc_streams *st, int32_t v)
{
    if (st->n_ptr < st->cap_ptr) st->ptr[st->n_ptr] = v; else st->overflow = 1;
    st->n_ptr++;
}
static void push_da(oc_streams *st, float v)
{
    if (st->n_da < st->cap_da) st->da[st->n_da] = v; else st->overflow = 1;
    st->n_da++;
}
static void push_in(oc_streams *st, int32_t v)
{
    if (st->n_in < st->cap_in) st->in[st->n_in] = v; else st->overflow = 1;
    st->n_in++;
}

/* Alg. 1, function G: scan column w of I top to bottom;
 * each NZE goes to DA, its index Z + h*K_w to IN, and nz_ptr counts it.
 * Z is the column's local index inside its owner partition. */
static void G(oc_streams *st, const float *plane, const oc_desc *d, int32_t w, int32_t Z, int32_t *nz_ptr)
{
    int32_t Hp = d->H + d->pt + d->pb;
    for (int32_t h = 0; h < Hp; h++) {
        float v = I_at(plane, d, h, w);
        if (v != 0.0f) {
            push_da(st, v);
            push_in(st, Z + h * d->S);
            (*nz_ptr)++;
        }
    }
}

/* Alg. 3 lines 6-20 with readings A9-A12: one overlapK_w
 * column in sets of 4 rows (set4) anchored at padded row 0; the trailing set
 * is completed with zeros.  A set4 with >= 3 NZEs becomes
 * {index of its first NZE, pattern}, pattern bit b <=> NZE at set row b
 * ("read from bottom to top", pattern += 2^(h%4)); a set4 with
 * 1 or 2 NZEs stores each index multiplied by -1.  DA is
 * filled exactly as CPO. */
static void G_cps(oc_streams *st, const float *plane, const oc_desc *d, int32_t w, int32_t Z, int32_t *nz_ptr)
{
    int32_t Hp = d->H + d->pt + d->pb;
    for (int32_t g = 0; 4 * g < Hp; g++) {
        int32_t rows[4], nz_col = 0, pattern = 0;
        for (int32_t b = 0; b < 4; b++) {
            int32_t h = 4 * g + b;
            if (h >= Hp) break;                     /* extra zeros complete the set4 */
            float v = I_at(plane, d, h, w);
            if (v != 0.0f) {
                push_da(st, v);
                pattern += 1 << b;                  /* 2^(h%4) */
                rows[nz_col++] = h;
                (*nz_ptr)++;
            }
        }
        if (nz_col > 2) {
            push_in(st, Z + rows[0] * d->S);        /* first NZE index (reading A9) */
            push_in(st, pattern);
        } else {
            for (int32_t i = 0; i < nz_col; i++) push_in(st, -(Z + rows[i] * d->S));
        }
    }
}

static int plane_is_zero(const float *plane, const oc_desc *d)
{
    for (int64_t i = 0; i < (int64_t)d->H * d->W; i++)
        if (plane[i] != 0.0f) return 0;
    return 1;
}

/* One channel of cpoEncode (Alg. 1) or cpsEncode (Alg. 3,
 * PAPER.md:335-370); K_w = 1 per SI Alg. 5.
 * Readings: tag = overlap count (A1); NOP block of 3 iff Pad_Left = 0 (A2);
 * NPF block = [tag, NPF] (A3); block-relative cumulative counts (A4); -1 iff
 * the partition owns no column of the type (A5); geometry of left/right
 * columns (A6); K_w = 1 is CPO for CPS too (A13). */
static void encode_channel(oc_streams *st, const float *plane, const oc_desc *d, int cps)
{
    int32_t Wp = d->W + d->pl + d->pr, S = d->S, Ow1 = Wp - S + 1;
    int32_t *c = (int32_t *)malloc(sizeof(int32_t) * (size_t)Ow1);

    if (plane_is_zero(plane, d)) {                 /* NPC: skip channel */
        push_ptr(st, OC_NPC);
        free(c);
        return;
    }
    if (S == 1) {                                  /* SI Alg. 5: ptr = [0, cumulative per column] */
        int32_t nz_ptr = 0;
        push_ptr(st, 0);
        for (int32_t w = 0; w < Wp; w++) {
            G(st, plane, d, w, 0, &nz_ptr);        /* IN = w + h*K_w - s = h */
            push_ptr(st, nz_ptr);
        }
        free(c);
        return;
    }
    int32_t pType = d->pl;                         /* pType = Pad_Left */
    if (pType == 0) {                              /* NOP, Alg. 1 lines 11-16 */
        int32_t nz_ptr = 0;
        push_ptr(st, 0);
        G(st, plane, d, 0, 0, &nz_ptr);            /* {w, w^} = {0, 0} */
        push_ptr(st, nz_ptr);
        G(st, plane, d, Wp - 1, S - 1, &nz_ptr);   /* {I_w - 1, K_w - 1} */
        push_ptr(st, nz_ptr);
        pType++;
    }
    for (; pType <= S - 2; pType++) {              /* overlap(pType+1), Alg. 1 lines 17-24 */
        int32_t nz_ptr = 0;
        for (int32_t s = 0; s < Ow1; s++) c[s] = -1;
        G(st, plane, d, pType, pType, &nz_ptr);            /* left column, partition 0 */
        c[0] = nz_ptr;
        G(st, plane, d, Wp - 1 - pType, S - 1, &nz_ptr);   /* right column, partition Ow-1-pType */
        c[Ow1 - 1 - pType] = nz_ptr;
        push_ptr(st, pType + 1);
        if (nz_ptr == 0) push_ptr(st, OC_NPF);             /* skip pointer */
        else for (int32_t s = 0; s < Ow1; s++) push_ptr(st, c[s]);
    }
    {                                              /* overlapK_w, Alg. 1 lines 25-29 / Alg. 3 */
        int32_t nz_ptr = 0;
        for (int32_t s = 0; s < Ow1; s++) c[s] = -1;
        for (int32_t w = S - 1; w <= Wp - S; w++) {
            if (cps) G_cps(st, plane, d, w, S - 1, &nz_ptr);
            else     G(st, plane, d, w, S - 1, &nz_ptr);   /* w^ = w - idx = K_w - 1 */
            c[w - S + 1] = nz_ptr;
        }
        push_ptr(st, S);
        if (nz_ptr == 0) push_ptr(st, OC_NPF);
        else for (int32_t s = 0; s < Ow1; s++) push_ptr(st, c[s]);
    }
    free(c);
}

/* Encode the whole tensor, channels concatenated n-major then c (reading A19).
 * chan_off (optional, [3][N*C+1]) receives the exclusive prefix offsets of
 * each channel segment in ptr / DA / IN (the GPU side tables).
 * lens = {ptr_len, da_len, in_len}.  Returns 0, or -1 if a capacity was too small
 * (lens then holds the required lengths). */
int oc_encode(const oc_desc *d, const float *x, int cps,
              int32_t *ptr, int64_t cap_ptr, float *da, int64_t cap_da, int32_t *in, int64_t cap_in,
              int64_t *chan_off, int64_t *lens)
{
    oc_streams st = {ptr, da, in, cap_ptr, cap_da, cap_in, 0, 0, 0, 0};
    int64_t NC = (int64_t)d->N * d->C;
    for (int32_t n = 0; n < d->N; n++)
        for (int32_t c = 0; c < d->C; c++) {
            int64_t j = (int64_t)n * d->C + c;
            if (chan_off) {
                chan_off[j] = st.n_ptr;
                chan_off[NC + 1 + j] = st.n_da;
                chan_off[2 * (NC + 1) + j] = st.n_in;
            }
            encode_channel(&st, plane_of(x, d, n, c), d, cps);
        }
    if (chan_off) {
        chan_off[NC] = st.n_ptr;
        chan_off[NC + 1 + NC] = st.n_da;
        chan_off[2 * (NC + 1) + NC] = st.n_in;
    }
    lens[0] = st.n_ptr; lens[1] = st.n_da; lens[2] = st.n_in;
    return st.overflow ? -1 : 0;
}

/* ------------------------------------------------- CPS index reconstruction */

/* getPatternSize (Alg. 4): NZEs of the set4 after its first one. */
static int32_t getPatternSize(int32_t pattern)
{
    int32_t n = 0;
    for (int32_t b = 0; b < 4; b++) n += (pattern >> b) & 1;
    return n - 1;
}

/* nextOffset (Alg. 4): row gap between the (g-1)-th and g-th set
 * bits of the pattern, scanning from bit 0 ("bottom to top", reading A12). */
static int32_t nextOffset(int32_t pattern, int32_t g)
{
    int32_t bits[4], nb = 0;
    for (int32_t b = 0; b < 4; b++) if ((pattern >> b) & 1) bits[nb++] = b;
    return bits[g] - bits[g - 1];
}

int32_t oc_pattern_size(int32_t pattern) { return getPatternSize(pattern); }
int32_t oc_next_offset(int32_t pattern, int32_t g) { return nextOffset(pattern, g); }

/* ------------------------------------------ decoder: streams -> dense map */

/* Independent inverse of the encoding: walk each channel's ptr blocks and
 * scatter DA back to (h, w) = (index / K_w, owner + index % K_w), where the
 * owner partition comes from the cumulative counts.
 * Returns 0, or -1 if the streams are inconsistent (corruption). */
int oc_decode(const oc_desc *d, int cps, const int32_t *ptr, int64_t n_ptr, const float *da,
              int64_t n_da, const int32_t *in, int64_t n_in, float *x)
{
    int32_t Hp = d->H + d->pt + d->pb, Wp = d->W + d->pl + d->pr, S = d->S, Ow1 = Wp - S + 1;
    int64_t p = 0, z = 0, q = 0;               /* cursors in ptr, DA, IN */
    memset(x, 0, sizeof(float) * (size_t)d->N * d->C * d->H * d->W);
#define PUT(n_, c_, h_, w_, v_) do {                                                    \
        int32_t hh_ = (h_) - d->pt, ww_ = (w_) - d->pl;                                 \
        if (hh_ < 0 || hh_ >= d->H || ww_ < 0 || ww_ >= d->W) return -1;               \
        x[(((size_t)(n_) * d->C + (c_)) * d->H + hh_) * d->W + ww_] = (v_);            \
    } while (0)
    for (int32_t n = 0; n < d->N; n++)
        for (int32_t c = 0; c < d->C; c++) {
            if (p >= n_ptr) return -1;
            if (ptr[p] == OC_NPC) { p++; continue; }
            /* list of blocks: (tag, first col type) */
            int32_t tags[64], nb = 0;
            if (S == 1) tags[nb++] = 0;
            else {
                if (d->pl == 0) tags[nb++] = 0;
                for (int32_t t = (d->pl > 1 ? d->pl : 1); t <= S - 1; t++) tags[nb++] = t + 1;
            }
            for (int32_t b = 0; b < nb; b++) {
                if (p >= n_ptr || ptr[p] != tags[b]) return -1;
                if (S > 1 && tags[b] == 0) {                          /* NOP [0, a, a+b] */
                    int32_t a = ptr[p + 1], ab = ptr[p + 2];
                    for (int32_t j = 0; j < ab; j++, z++, q++) {
                        if (z >= n_da || q >= n_in) return -1;
                        int32_t s = (j < a) ? 0 : Ow1 - 1;
                        PUT(n, c, in[q] / S, s + in[q] % S, da[z]);
                    }
                    p += 3;
                    continue;
                }
                if (ptr[p + 1] == OC_NPF) { p += 2; continue; }
                int32_t prev = 0, last_block = (S == 1) || (tags[b] == S);
                for (int32_t s = 0; s < Ow1; s++) {
                    int32_t cs = ptr[p + 1 + s];
                    if (cs < 0) continue;                                 /* no column in partition s */
                    if (cs < prev) return -1;
                    int32_t j = prev;
                    while (j < cs) {
                        if (z >= n_da || q >= n_in) return -1;
                        int32_t e = in[q];
                        if (cps && S > 1 && last_block) {
                            if (e < 0) {                                  /* singleton / pair */
                                PUT(n, c, (-e) / S, s + (-e) % S, da[z]);
                                z++; q++; j++;
                            } else {                                      /* {index, pattern} */
                                int32_t pat = in[q + 1], idx = e;
                                PUT(n, c, idx / S, s + idx % S, da[z]);
                                z++; j++;
                                for (int32_t g = 1; g <= getPatternSize(pat); g++) {
                                    idx += S * nextOffset(pat, g);
                                    if (z >= n_da) return -1;
                                    PUT(n, c, idx / S, s + idx % S, da[z]);
                                    z++; j++;
                                }
                                q += 2;
                            }
                        } else {
                            PUT(n, c, e / S, s + e % S, da[z]);
                            z++; q++; j++;
                        }
                    }
                    if (j != cs) return -1;
                    prev = cs;
                }
                p += 1 + Ow1;
            }
        }
#undef PUT
    (void)Hp;
    return (p == n_ptr && z == n_da && q == n_in) ? 0 : -1;
}

/* ----------------------------------------- CPO / CPS sparse convolution */

/* convSpMv (Alg. 2 lines 1-8): the NZE DA[x] with row-major
 * index `index` in partition s contributes, for every kernel row l, to output
 * row y = index/K_w - l at columns s..s+pType with kernel taps t, t-1, ...
 * (t = index%K_w + l*K_w).  Bounds: l in [0,K_h), i in [0,pType] (reading A28).
 * Stride extension (reading A15 / SURVEY.md A.7): the stride-1 output (y, s+i)
 * is kept iff it lies on the stride grid, and lands at (y/s_h, (s+i)/s_w).
 * `wkc` is the row-major kernel vector of (k, c). */
static void convSpMv(const oc_desc *d, int32_t Oh, int32_t Ow, int32_t Oh1, int32_t pType,
                     double v, int32_t s, int32_t index, const float *wkc, double *O)
{
    int32_t K_w = d->S;
    for (int32_t l = 0; l < d->R; l++) {
        int32_t y = index / K_w - l;
        int32_t t = index % K_w + l * K_w;
        if (y >= 0 && y < Oh1) {
            for (int32_t i = 0; i <= pType; i++) {
                int32_t x1 = s + i;
                if (y % d->sh || x1 % d->sw) continue;
                if (y / d->sh >= Oh || x1 / d->sw >= Ow) continue;
                O[(size_t)(y / d->sh) * Ow + x1 / d->sw] += v * (double)wkc[t - i];
            }
        }
    }
}

/* cpoAlg (Alg. 2) / cpsAlg (Alg. 4) /
 * SI Alg. 6 (K_w = 1), for every image and kernel k,
 * channel by channel; y is NKHW in FP64.  Stream cursors per channel come
 * from walking the streams in order (the per-channel indexing omitted in
 * PAPER.md:236).  Returns 0 or -1 on corrupt streams. */
int oc_sparse_conv(const oc_desc *d, int cps, const int32_t *ptr, int64_t n_ptr, const float *da,
                   const int32_t *in, const float *w, double *y)
{
    int32_t Hp = d->H + d->pt + d->pb, Wp = d->W + d->pl + d->pr, S = d->S, Ow1 = Wp - S + 1;
    int32_t Oh1 = Hp - d->R + 1, Oh = oc_out_h(d), Ow = oc_out_w(d);
    memset(y, 0, sizeof(double) * (size_t)d->N * d->K * Oh * Ow);
    for (int32_t k = 0; k < d->K; k++) {
        int64_t p = 0, zc = 0, qc = 0;          /* channel-start cursors in ptr, DA, IN */
        for (int32_t n = 0; n < d->N; n++) {
            double *O = y + ((size_t)n * d->K + k) * Oh * Ow;
            for (int32_t c = 0; c < d->C; c++) {
                const float *wkc = w + ((size_t)k * d->C + c) * d->R * d->S;
                if (p >= n_ptr) return -1;
                if (ptr[p] == OC_NPC) { p++; continue; }              /* skip channel */
                int64_t z = zc, q = qc;
                if (S == 1) {                                          /* SI Alg. 6 */
                    int32_t x = 0;
                    for (int32_t s = 0; s < Ow1; s++) {
                        for (int32_t tx = x; tx < ptr[p + 1 + s]; tx++) {
                            convSpMv(d, Oh, Ow, Oh1, 0, (double)da[z + tx], s, in[q + tx], wkc, O);
                        }
                        x = ptr[p + 1 + s];
                    }
                    zc += x; qc += x; p += 1 + Ow1;
                    continue;
                }
                if (d->pl == 0) {                                      /* NOP (Alg. 2 lines 11-18) */
                    if (ptr[p] != 0) return -1;
                    int32_t a = ptr[p + 1], ab = ptr[p + 2];
                    for (int32_t x = 0; x < a; x++)
                        convSpMv(d, Oh, Ow, Oh1, 0, (double)da[z + x], 0, in[q + x], wkc, O);
                    for (int32_t x = a; x < ab; x++)
                        convSpMv(d, Oh, Ow, Oh1, 0, (double)da[z + x], Ow1 - 1, in[q + x], wkc, O);
                    z += ab; q += ab; p += 3;
                }
                for (int32_t pType = (d->pl > 1 ? d->pl : 1); pType <= S - 1; pType++) {
                    if (ptr[p] != pType + 1) return -1;
                    if (ptr[p + 1] == OC_NPF) { p += 2; continue; }    /* skip ptr */
                    int32_t x = 0;
                    int decode_cps = cps && pType == S - 1;
                    int64_t qi = q;                                    /* IN cursor (CPS: != DA cursor) */
                    for (int32_t s = 0; s < Ow1; s++) {
                        int32_t end = ptr[p + 1 + s];
                        if (end < 0) end = x;                          /* ptr < 0: repeat previous */
                        int32_t tx = x;
                        while (tx < end) {
                            if (!decode_cps) {
                                convSpMv(d, Oh, Ow, Oh1, pType, (double)da[z + tx], s, in[q + tx], wkc, O);
                                tx++;
                                continue;
                            }
                            /* Alg. 4 lines 7-17: negative -> singleton; else {index, pattern} */
                            int32_t index = in[qi], pattern = -1;
                            if (index < 0) { index = -index; qi += 1; }
                            else { pattern = in[qi + 1]; qi += 2; }
                            convSpMv(d, Oh, Ow, Oh1, pType, (double)da[z + tx], s, index, wkc, O);
                            int32_t nnzSet4 = pattern < 0 ? 0 : getPatternSize(pattern);
                            for (int32_t g = 1; g <= nnzSet4; g++) {
                                index += S * nextOffset(pattern, g);
                                tx++;
                                convSpMv(d, Oh, Ow, Oh1, pType, (double)da[z + tx], s, index, wkc, O);
                            }
                            tx++;
                        }
                        x = end;
                    }
                    z += x;
                    q = decode_cps ? qi : q + x;
                    p += 1 + Ow1;
                }
                zc = z; qc = q;
            }
        }
    }
    return 0;
}

/* MAC count of the sparse convolution for a given map: for each NZE, the number
 * of (output, tap) pairs it meets, times K (reading A27; SPEC.md:195-203 idea).
 * Counted by brute-force enumeration of kernel windows covering each NZE. */
int64_t oc_mac_count(const oc_desc *d, const float *x)
{
    int32_t Oh = oc_out_h(d), Ow = oc_out_w(d);
    int64_t macs = 0;
    for (int32_t n = 0; n < d->N; n++)
        for (int32_t c = 0; c < d->C; c++) {
            const float *pl = plane_of(x, d, n, c);
            for (int32_t oy = 0; oy < Oh; oy++)
                for (int32_t ox = 0; ox < Ow; ox++)
                    for (int32_t h = 0; h < d->R; h++)
                        for (int32_t ww = 0; ww < d->S; ww++)
                            if (I_at(pl, d, oy * d->sh + h, ox * d->sw + ww) != 0.0f) macs++;
        }
    return macs * d->K;
}

/* ------------------------------------------------------- set4 census */

/* C'_k and C''_k of SI Eq. 5: number of set4 groups with k
 * NZEs outside (C') and inside (C'') the overlapK_w region, per channel,
 * summed over the tensor.  Groups of 4 padded rows anchored at row 0 in every
 * column (reading A10).  cen = {C'_1..C'_4, C''_1..C''_4}.  For K_w = 1 every
 * column is outside overlapK_w. */
void oc_set4_census(const oc_desc *d, const float *x, int64_t *cen)
{
    int32_t Hp = d->H + d->pt + d->pb, Wp = d->W + d->pl + d->pr, S = d->S;
    for (int i = 0; i < 8; i++) cen[i] = 0;
    for (int32_t n = 0; n < d->N; n++)
        for (int32_t c = 0; c < d->C; c++) {
            const float *pl = plane_of(x, d, n, c);
            for (int32_t w = 0; w < Wp; w++) {
                int inner = (S > 1) && (w >= S - 1) && (w <= Wp - S);
                for (int32_t g = 0; 4 * g < Hp; g++) {
                    int32_t k = 0;
                    for (int32_t b = 0; b < 4 && 4 * g + b < Hp; b++)
                        k += I_at(pl, d, 4 * g + b, w) != 0.0f;
                    if (k) cen[(inner ? 4 : 0) + k - 1]++;
                }
            }
        }
}

/* Count of NPF flags and NPC flags in a ptr stream (for SI Eq. 3). */
void oc_count_flags(const int32_t *ptr, int64_t n_ptr, int64_t *npf, int64_t *npc)
{
    *npf = 0; *npc = 0;
    for (int64_t i = 0; i < n_ptr; i++) {
        if (ptr[i] == OC_NPF) (*npf)++;
        if (ptr[i] == OC_NPC) (*npc)++;
    }
}

/* ------------------------------------------------- CSCC (the paper's comparison method) */

/* CSCC encoding (fan2019cscc, as simplified by SI Alg. 5, which the
 * paper says is "designed for any value of K_w and s_w"): every output
 * column s (stride s_w) owns the K_w-wide submatrix of padded columns
 * [s*s_w, s*s_w + K_w) -- the lowered matrix LM of SI Eq. 17 -- and
 * its NZEs are stored row-major inside the submatrix (Alg. 5 lines 10-27: w runs to
 * s + K_w - 1, then h++), IN = (w - s*s_w) + h*K_w, with ptr = [0, c_0 .. c_{O_w-1}]
 * channel-cumulative counts per submatrix (O_w + 1 entries per channel; CSCC has no
 * NPC flag: Eq. 17 charges every channel O_w + 1).  Padded frame (reading A30).
 * chan_off (optional, [3][N*C+1]) and lens as oc_encode.  Returns 0 or -1 (capacity). */
int oc_cscc_encode(const oc_desc *d, const float *x, int32_t *ptr, int64_t cap_ptr, float *da, int64_t cap_da,
                   int32_t *in, int64_t cap_in, int64_t *chan_off, int64_t *lens)
{
    int32_t Hp = d->H + d->pt + d->pb, Ow = oc_out_w(d), K_w = d->S;
    int64_t np = 0, nz = 0, NC = (int64_t)d->N * d->C;
    int overflow = 0;
    for (int32_t n = 0; n < d->N; n++)
        for (int32_t c = 0; c < d->C; c++) {
            int64_t j = (int64_t)n * d->C + c;
            if (chan_off) { chan_off[j] = np; chan_off[NC + 1 + j] = nz; chan_off[2 * (NC + 1) + j] = nz; }
            const float *pl = plane_of(x, d, n, c);
            int32_t nz_ptr = 0;
            if (np < cap_ptr) ptr[np] = 0; else overflow = 1;
            np++;
            for (int32_t s = 0; s < Ow; s++) {                 /* one submatrix per output column */
                for (int32_t h = 0; h < Hp; h++)
                    for (int32_t w = s * d->sw; w < s * d->sw + K_w; w++) {
                        float v = I_at(pl, d, h, w);
                        if (v != 0.0f) {
                            if (nz < cap_da && nz < cap_in) { da[nz] = v; in[nz] = (w - s * d->sw) + h * K_w; }
                            else overflow = 1;
                            nz++;
                            nz_ptr++;
                        }
                    }
                if (np < cap_ptr) ptr[np] = nz_ptr; else overflow = 1;
                np++;
            }
        }
    if (chan_off) { chan_off[NC] = np; chan_off[NC + 1 + NC] = nz; chan_off[2 * (NC + 1) + NC] = nz; }
    lens[0] = np; lens[1] = nz; lens[2] = nz;
    return overflow ? -1 : 0;
}

/* CSCC convolution (SI Alg. 6, with the stride of SI Eq. 17's
 * submatrices): the NZE DA[x] with index `index` of submatrix s contributes, for every
 * kernel row l, to output row y = index/K_w - l of output column s with tap
 * t = index%K_w + l*K_w (Alg. 6 lines 1-9); a vertical stride keeps y on the grid
 * (reading A15).  No NPC skip (CSCC).  y is NKHW in FP64.  Returns 0 or -1. */
int oc_cscc_conv(const oc_desc *d, const int32_t *ptr, int64_t n_ptr, const float *da, int64_t n_da,
                 const int32_t *in, const float *w, double *y)
{
    int32_t Hp = d->H + d->pt + d->pb, Oh1 = Hp - d->R + 1, Oh = oc_out_h(d), Ow = oc_out_w(d), K_w = d->S;
    memset(y, 0, sizeof(double) * (size_t)d->N * d->K * Oh * Ow);
    for (int32_t k = 0; k < d->K; k++) {
        int64_t p = 0, z = 0;
        for (int32_t n = 0; n < d->N; n++) {
            double *O = y + ((size_t)n * d->K + k) * Oh * Ow;
            for (int32_t c = 0; c < d->C; c++) {
                const float *wkc = w + ((size_t)k * d->C + c) * d->R * d->S;
                if (p + Ow >= n_ptr || ptr[p] != 0) return -1;
                int32_t x = 0;                                   /* x = ptr[ptr_sh] (Alg. 6 line 16) */
                for (int32_t s = 0; s < Ow; s++) {
                    int32_t end = ptr[p + 1 + s];
                    if (end < x || z + end > n_da) return -1;
                    for (int32_t tx = x; tx < end; tx++) {       /* convSpMv(K_h, K_w, O_h, tx, s, IN[tx]) */
                        int32_t index = in[z + tx];
                        for (int32_t l = 0; l < d->R; l++) {
                            int32_t yy = index / K_w - l;
                            int32_t t = index % K_w + l * K_w;
                            if (yy >= 0 && yy < Oh1 && yy % d->sh == 0 && yy / d->sh < Oh)
                                O[(size_t)(yy / d->sh) * Ow + s] += (double)da[z + tx] * (double)wkc[t];
                        }
                    }
                    x = end;
                }
                z += x;
                p += 1 + Ow;
            }
        }
        if (p != n_ptr || z != n_da) return -1;
    }
    return 0;
}

/* Independent inverse of the CSCC streams: every copy of an NZE (one per submatrix that
 * holds its column) is written back to (h, s*s_w + index%K_w); copies must agree.
 * Columns no submatrix covers stay 0.  Returns 0 or -1 on inconsistency. */
int oc_cscc_decode(const oc_desc *d, const int32_t *ptr, int64_t n_ptr, const float *da, int64_t n_da,
                   const int32_t *in, float *x)
{
    int32_t Ow = oc_out_w(d), K_w = d->S;
    int64_t p = 0, z = 0;
    memset(x, 0, sizeof(float) * (size_t)d->N * d->C * d->H * d->W);
    for (int32_t n = 0; n < d->N; n++)
        for (int32_t c = 0; c < d->C; c++) {
            if (p + Ow >= n_ptr + 1 || ptr[p] != 0) return -1;
            int32_t prev = 0;
            for (int32_t s = 0; s < Ow; s++) {
                int32_t end = ptr[p + 1 + s];
                if (end < prev || z + end > n_da) return -1;
                for (int32_t tx = prev; tx < end; tx++) {
                    int32_t e = in[z + tx], h = e / K_w - d->pt, ww = s * d->sw + e % K_w - d->pl;
                    if (e < 0 || h < 0 || h >= d->H || ww < 0 || ww >= d->W) return -1;
                    float *dst = &x[(((size_t)n * d->C + c) * d->H + h) * d->W + ww];
                    if (*dst != 0.0f && *dst != da[z + tx]) return -1;
                    *dst = da[z + tx];
                }
                prev = end;
            }
            z += prev;
            p += 1 + Ow;
        }
    return (p == n_ptr && z == n_da) ? 0 : -1;
}

/* ------------------------------------- stride-aware CPO layout (NEXT-4, reading A32) */

/* SI Eq. 2 sizes the overlap pointer with ceil(K_w/s_w) types, i.e. a
 * layout whose partitions are the O_w output columns at stride s_w -- which the paper never
 * spells out (it encodes at stride 1).  Reading A32 makes it concrete for
 * s_w >= 2: partition s (0 <= s < O_w) covers padded columns [s*s_w, s*s_w + K_w); column w
 * has coverage cov(w) = #partitions covering it (0 .. ceil(K_w/s_w)); its owner is the first
 * covering partition and its local column L = w - owner*s_w; its type is t = cov - 1.  Per
 * channel: [NPC] if no covered column holds an NZE, else for every type t present in the
 * geometry (ascending, as the paper orders NOP, overlap2, .. overlapK_w) the
 * block [t+1, c_0 .. c_{O_w-1}] with block-relative cumulative counts through partition s's
 * owned columns of type t (-1 if it owns none), or [t+1, NPF] if the block is empty.  DA / IN
 * take the block's columns ascending, rows ascending, IN = L + h*K_w.  Columns no partition
 * covers are never read by the convolution and are not stored. */
static int32_t sa_ow(const oc_desc *d) { return oc_out_w(d); }

static int32_t sa_cov(const oc_desc *d, int32_t w)
{
    int32_t n = 0;
    for (int32_t s = 0; s < sa_ow(d); s++)
        if (s * d->sw <= w && w < s * d->sw + d->S) n++;
    return n;
}

static int32_t sa_owner(const oc_desc *d, int32_t w)
{
    for (int32_t s = 0; s < sa_ow(d); s++)
        if (s * d->sw <= w && w < s * d->sw + d->S) return s;
    return -1;
}

/* types present in the geometry: type t has at least one covered column */
static int32_t sa_type_present(const oc_desc *d, int32_t t)
{
    int32_t Wp = d->W + d->pl + d->pr;
    for (int32_t w = 0; w < Wp; w++)
        if (sa_cov(d, w) == t + 1) return 1;
    return 0;
}

static int32_t sa_ntypes(const oc_desc *d) { return (d->S + d->sw - 1) / d->sw; }

int oc_encode_sa(const oc_desc *d, const float *x, int32_t *ptr, int64_t cap_ptr, float *da, int64_t cap_da,
                 int32_t *in, int64_t cap_in, int64_t *chan_off, int64_t *lens)
{
    int32_t Hp = d->H + d->pt + d->pb, Wp = d->W + d->pl + d->pr, Ow = sa_ow(d), S = d->S;
    int64_t np = 0, nz = 0, NC = (int64_t)d->N * d->C;
    int overflow = 0;
    int32_t *c = (int32_t *)malloc(sizeof(int32_t) * (size_t)Ow);
#define PUSHP(v_) do { if (np < cap_ptr) ptr[np] = (v_); else overflow = 1; np++; } while (0)
    for (int32_t n = 0; n < d->N; n++)
        for (int32_t ch = 0; ch < d->C; ch++) {
            int64_t j = (int64_t)n * d->C + ch;
            if (chan_off) { chan_off[j] = np; chan_off[NC + 1 + j] = nz; chan_off[2 * (NC + 1) + j] = nz; }
            const float *pl = plane_of(x, d, n, ch);
            int32_t any = 0;
            for (int32_t w = 0; w < Wp && !any; w++)
                if (sa_cov(d, w) > 0)
                    for (int32_t h = 0; h < Hp; h++) any |= I_at(pl, d, h, w) != 0.0f;
            if (!any) { PUSHP(OC_NPC); continue; }
            for (int32_t t = 0; t < sa_ntypes(d); t++) {
                if (!sa_type_present(d, t)) continue;
                int32_t nz_ptr = 0;
                for (int32_t s = 0; s < Ow; s++) c[s] = -1;
                for (int32_t w = 0; w < Wp; w++) {            /* the block's columns, ascending */
                    if (sa_cov(d, w) != t + 1) continue;
                    int32_t s = sa_owner(d, w), L = w - s * d->sw;
                    for (int32_t h = 0; h < Hp; h++) {
                        float v = I_at(pl, d, h, w);
                        if (v != 0.0f) {
                            if (nz < cap_da && nz < cap_in) { da[nz] = v; in[nz] = L + h * S; }
                            else overflow = 1;
                            nz++;
                            nz_ptr++;
                        }
                    }
                    c[s] = nz_ptr;                              /* cumulative through partition s */
                }
                PUSHP(t + 1);
                if (nz_ptr == 0) PUSHP(OC_NPF);
                else for (int32_t s = 0; s < Ow; s++) PUSHP(c[s]);
            }
        }
#undef PUSHP
    if (chan_off) { chan_off[NC] = np; chan_off[NC + 1 + NC] = nz; chan_off[2 * (NC + 1) + NC] = nz; }
    lens[0] = np; lens[1] = nz; lens[2] = nz;
    free(c);
    return overflow ? -1 : 0;
}

/* Walk the stride-aware streams of one tensor and call back per NZE (n, c, s, t, index, v);
 * mode 0 = decode into x, 1 = convolution into y.  Returns 0 or -1 (inconsistent). */
static int sa_walk(const oc_desc *d, const int32_t *ptr, int64_t n_ptr, const float *da, int64_t n_da,
                   const int32_t *in, float *x, const float *w, double *y)
{
    int32_t Hp = d->H + d->pt + d->pb, Ow = sa_ow(d), S = d->S, Oh = oc_out_h(d), Oh1 = Hp - d->R + 1;
    int64_t p = 0, z = 0;
    for (int32_t n = 0; n < d->N; n++)
        for (int32_t ch = 0; ch < d->C; ch++) {
            if (p >= n_ptr) return -1;
            if (ptr[p] == OC_NPC) { p++; continue; }
            for (int32_t t = 0; t < sa_ntypes(d); t++) {
                if (!sa_type_present(d, t)) continue;
                if (p + 1 >= n_ptr || ptr[p] != t + 1) return -1;
                if (ptr[p + 1] == OC_NPF) { p += 2; continue; }
                if (p + Ow >= n_ptr) return -1;
                int32_t prev = 0;
                for (int32_t s = 0; s < Ow; s++) {
                    int32_t cs = ptr[p + 1 + s];
                    if (cs < 0) continue;                     /* partition s owns no type-t column */
                    if (cs < prev || z + cs > n_da) return -1;
                    for (int32_t tx = prev; tx < cs; tx++) {
                        int32_t e = in[z + tx], h = e / S, L = e % S, wcol = s * d->sw + L;
                        double v = (double)da[z + tx];
                        if (e < 0 || h >= Hp || sa_cov(d, wcol) != t + 1 || sa_owner(d, wcol) != s) return -1;
                        if (x) {
                            int32_t hh = h - d->pt, ww = wcol - d->pl;
                            if (hh < 0 || hh >= d->H || ww < 0 || ww >= d->W) return -1;
                            x[(((size_t)n * d->C + ch) * d->H + hh) * d->W + ww] = da[z + tx];
                        } else {
                            /* convSpMv over the t+1 partitions s..s+t that cover column wcol */
                            for (int32_t k = 0; k < d->K; k++) {
                                const float *wkc = w + ((size_t)k * d->C + ch) * d->R * d->S;
                                double *O = y + ((size_t)n * d->K + k) * Oh * Ow;
                                for (int32_t l = 0; l < d->R; l++) {
                                    int32_t y1 = h - l;
                                    if (y1 < 0 || y1 >= Oh1 || y1 % d->sh || y1 / d->sh >= Oh) continue;
                                    for (int32_t i = 0; i <= t; i++) {
                                        int32_t xo = s + i, m = wcol - xo * d->sw;
                                        if (xo >= Ow || m < 0 || m >= S) continue;
                                        O[(size_t)(y1 / d->sh) * Ow + xo] += v * (double)wkc[l * S + m];
                                    }
                                }
                            }
                        }
                    }
                    prev = cs;
                }
                z += prev;
                p += 1 + Ow;
            }
        }
    return (p == n_ptr && z == n_da) ? 0 : -1;
}

int oc_decode_sa(const oc_desc *d, const int32_t *ptr, int64_t n_ptr, const float *da, int64_t n_da,
                 const int32_t *in, float *x)
{
    memset(x, 0, sizeof(float) * (size_t)d->N * d->C * d->H * d->W);
    return sa_walk(d, ptr, n_ptr, da, n_da, in, x, NULL, NULL);
}

int oc_sparse_conv_sa(const oc_desc *d, const int32_t *ptr, int64_t n_ptr, const float *da, int64_t n_da,
                      const int32_t *in, const float *w, double *y)
{
    memset(y, 0, sizeof(double) * (size_t)d->N * d->K * oc_out_h(d) * oc_out_w(d));
    return sa_walk(d, ptr, n_ptr, da, n_da, in, NULL, w, y);
}
