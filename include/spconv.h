/*
 * spconv.h -- C ABI of the B200 (sm_100a) implementation of the hot path of
 * arXiv 2104.08314, "High Performance Convolution Using Sparsity and Patterns
 * for Inference in Deep Convolutional Neural Networks" (CPO / CPS).
 *
 * Citations "PAPER.md:<line>" point into the paper text; "reading Ax" points
 * to DESIGN.md §Readings (the canonical resolution of ambiguous passages).
 *
 * Conventions for every entry point
 *  - Tensor pointers are DEVICE pointers unless the argument says "host".
 *    The caller owns and allocates every buffer; no call allocates or frees
 *    device memory.  Device buffers must be 16-byte aligned.
 *  - Calls are asynchronous on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream) unless documented as synchronising.
 *  - Host-side validation happens before any launch; on a non-OK status no
 *    kernel was launched (except SPC_ECUDA, which reports a launch/runtime
 *    error).  spc_last_error() returns a thread-local message.
 *  - Layouts: activations x are NCHW fp32; weights w are KCRS fp32
 *    (K output channels, C input channels, R = K_h rows, S = K_w columns);
 *    outputs y are NKHW fp32 with Oh = floor((H+pt+pb-R)/sh)+1 and
 *    Ow = floor((W+pl+pr-S)/sw)+1 (reading A14).
 *  - Thread safety: calls on different streams with disjoint buffers and
 *    workspaces may run concurrently.  Kernels go to the caller's CURRENT
 *    device (cudaSetDevice); launch caches (shared-memory attributes, SM
 *    counts) are kept per device.  Kernels whose CTAs wait on one another
 *    (the encoder's cross-tile prefix, the balanced-mode convolution) are
 *    launched cooperatively, so the driver co-schedules the whole grid even
 *    when other streams hold SMs; their waits are bounded and a timeout is
 *    reported through the encoding's overflow word (never a trap or a hang).
 */
#ifndef SPCONV_H
#define SPCONV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SPC_OK = 0,
    SPC_EINVAL = -1,        /* bad argument: null pointer, shape mismatch, bad capacity */
    SPC_EUNSUPPORTED = -2,  /* geometry outside the method's scope (see cpo_encode) */
    SPC_ECAPACITY = -3,     /* a stream capacity was too small (reported by spc_encoding_lengths) */
    SPC_ECUDA = -4,         /* CUDA launch or runtime error */
    SPC_ECORRUPT = -5       /* an encoding failed validation */
} spc_status;

typedef enum { SPC_ALGO_IM2COL = 0, SPC_ALGO_CPO = 1, SPC_ALGO_CPS = 2,
               SPC_ALGO_CSCC = 3,   /* the paper's comparison baseline (cscc_encode), never selected */
               SPC_ALGO_CPO_SA = 4  /* stride-aware CPO layout (cpo_encode_strided, reading A32) */ } spc_algo;

/* Hybrid selection modes: favour time = argmin{im2col, CPO};
 * favour space = argmin{im2col, CPS}; best of three = argmin over all three. */
typedef enum { SPC_FAVOUR_TIME = 0, SPC_FAVOUR_SPACE = 1, SPC_BEST_OF_THREE = 2 } spc_mode;

/* Reserved ptr sentinels (reading A7): NPC = all-zero channel, NPF = all-zero
 * overlap region.  -1 keeps the meaning "partition owns no
 * column of this overlap type" (reading A5). */
#define SPC_NPC ((int32_t)INT32_MIN)
#define SPC_NPF ((int32_t)(INT32_MIN + 1))

/* The paper's problem statement (Table 1): input
 * I_n x I_c x I_h x I_w (here N, C, H, W), kernel K x I_c x K_h x K_w
 * (K, C, R, S), strides s_h, s_w and zero padding. */
typedef struct {
    int32_t N, C, H, W;
    int32_t K, R, S;
    int32_t stride_h, stride_w;
    int32_t pad_top, pad_bottom, pad_left, pad_right;
} spc_conv_desc;

/* One encoded activation tensor (CPO or CPS).  Streams:
 *   ptr  int32  per channel: NPC, or the blocks NOP [0,a,a+b] (iff pad_left
 *               = 0), then for t = max(1,pad_left) .. S-1: [t+1, NPF] or
 *               [t+1, c_0 .. c_{Ow1-1}] with block-relative cumulative NZE
 *               counts per partition (-1 = no column); for S = 1 a single
 *               block [0, c_0 .. c_{Ow1-1}] (SI Alg. 5).  Ow1 = Wp - S + 1.
 *   da   fp32   NZE values, bit copies of x, column-major per block
 *   in   int32  CPO: row-major local index L + h*S (h in the
 *               padded frame); CPS: as CPO except the overlapK_w block, which
 *               holds {first NZE index, 4-bit pattern} per set4 with >= 3
 *               NZEs and negated indices otherwise
 * Channels are concatenated n-major then c (reading A19).  The side tables
 * chan_*_off (GPU-only, not part of the paper's streams or its CR) hold the
 * exclusive prefix offsets of each (n,c) segment, N*C+1 entries each.
 * `lengths` (device int64[4]) receives {ptr_len, da_len, in_len, overflow}
 * at the end of an encode; overflow != 0 means some capacity was too small
 * and the streams are incomplete.  `algo` and `geom` are written by the
 * encoder (host fields). */
typedef struct {
    int32_t *ptr;  int64_t ptr_cap;
    float   *da;   int64_t da_cap;
    int32_t *in;   int64_t in_cap;
    int64_t *chan_ptr_off, *chan_nz_off, *chan_in_off;
    int64_t *lengths;
    int32_t algo;
    spc_conv_desc geom;
} spc_encoding;

/* Host.  Worst-case stream capacities for `d` (dense map) and the workspace
 * bytes every other call below needs at most for this geometry:
 *   ptr <= N*C*(3 + (S-1)*(1+Ow1)) (S > 1) or N*C*(1+Ow1) (S = 1);
 *   da  <= N*C*H*W (pad cells are never NZEs);  in <= da.
 * Returns SPC_EUNSUPPORTED for geometries the encoder rejects. */
spc_status spc_encode_capacity(const spc_conv_desc *d, int64_t *ptr_cap, int64_t *da_cap,
                               int64_t *in_cap, size_t *ws_bytes);

/* Host, synchronous.  Zero a workspace once after allocation.  The encoder's
 * cross-tile state in it is epoch-tagged (tags and counters are per launch, a
 * consumed conv flag is re-zeroed by its consumer), so it is never reset between
 * launches -- and must NOT be re-zeroed, or shared by two streams, in the middle
 * of a sequence of launches: one workspace serves one stream at a time. */
spc_status spc_workspace_init(void *ws, size_t ws_bytes, void *stream);

/* CPO encoding (Alg. 1; SI Alg. 5 for S = 1)
 * of x (device, N*C*H*W fp32) into `out`.  The encoding depends only on x,
 * R, S and the pads, never on the stride or K (reading A15).  One launch.
 * Unsupported (SPC_EUNSUPPORTED): R = S = 1 (pointwise);
 * S > 1 with pad_left != pad_right or pad_left > S-1 or Wp < 2S-1; S = 1 with
 * horizontal padding; pad_top or pad_bottom > R-1; K_h > 32; a plane larger than
 * the encoder's shared-memory stage (H*W*4 > 192 KB = 196608 bytes).
 * ws: >= ws_bytes from spc_encode_capacity, zeroed once (spc_workspace_init). */
spc_status cpo_encode(const spc_conv_desc *d, const float *x, spc_encoding *out, void *ws,
                      size_t ws_bytes, void *stream);

/* CPS encoding (Alg. 3): ptr and da identical to CPO; the
 * overlapK_w block of `in` is pattern-compressed in sets of 4 padded rows
 * anchored at row 0 (readings A9-A12).  For S = 1 CPS equals CPO (reading
 * A13).  Same arguments and errors as cpo_encode. */
spc_status cps_encode(const spc_conv_desc *d, const float *x, spc_encoding *out, void *ws,
                      size_t ws_bytes, void *stream);

/* Offline, once per layer: repack KCRS weights into [C][R][S][K] so that a
 * warp's lanes read consecutive output channels (w_packed: C*R*S*K fp32). */
spc_status spc_pack_weights(const spc_conv_desc *d, const float *w_kcrs, float *w_packed, void *stream);

/* Sparse convolution over an encoding (Alg. 2 CPO / Alg. 4 CPS / SI Alg. 6,
 * PAPER.md:236-309, :376-426, :1395-1435): y = conv(decode(enc), w) in fp32
 * with any stride (reading A15, DESIGN.md A.7).  All-zero channels (NPC) and
 * regions (NPF) are skipped.  fuse_relu != 0 applies max(0, .) to y.
 * For a CPS encoding the pattern sets are expanded into ws first.
 * ws: >= ws_bytes from spc_encode_capacity (may be NULL for CPO; with it, a cluster-split
 * launch reduces its partial sums through L2 instead of distributed shared memory). */
spc_status sparse_conv_forward(const spc_conv_desc *d, const spc_encoding *enc, const float *w_packed,
                               float *y, int32_t fuse_relu, void *ws, size_t ws_bytes, void *stream);

/* ---- Stride-aware CPO layout (reading A32 of DESIGN.md).  SI Eq. 2
 * sizes the overlap pointer with ceil(K_w/s_w) types, i.e. partitions at the
 * real horizontal stride; the paper encodes at stride 1 only.  Here partition s
 * (0 <= s < O_w) covers padded columns [s*s_w, s*s_w + K_w); a column's type t = (number of
 * partitions covering it) - 1, owner = the first of them, local column L = w - owner*s_w.  Per
 * channel: [NPC] if no covered column holds an NZE, else for each type present (ascending)
 * [t+1, c_0 .. c_{O_w-1}] (block-relative cumulative counts through partition s's owned type-t
 * columns, -1 = owns none) or [t+1, NPF]; DA / IN column by column ascending, rows ascending,
 * IN = L + h*K_w.  Columns no partition covers are not stored (no output reads them).  At
 * s_w = 2 a block holds O_w instead of Wp - K_w + 1 partitions (about half the ptr).
 * algo = SPC_ALGO_CPO_SA; sparse_conv_forward accepts it (the encoding's stride_w must equal
 * the descriptor's).  Capacities: ptr <= N*C*max(1, ceil(K_w/s_w)*(1+O_w)), da = in <= N*C*H*W. */
spc_status spc_strided_capacity(const spc_conv_desc *d, int64_t *ptr_cap, int64_t *da_cap, int64_t *in_cap);
/* ws (>= ws_bytes from spc_encode_capacity, zeroed once, shareable with cpo_encode on the same
 * stream) and the canonical preconditions of cpo_encode: one launch -- the canonical encoder's
 * kernel with this layout's column order and ptr blocks (capacity overflow as in cpo_encode).
 * ws = NULL (or a geometry outside those preconditions): three launches (counts, scan, writes);
 * lengths[3] = 1 (nothing written) when a capacity is too small.  The streams are identical.
 * SPC_EUNSUPPORTED: pointwise, K_w > 8, or a plane too large for one CTA. */
spc_status cpo_encode_strided(const spc_conv_desc *d, const float *x, spc_encoding *out, void *ws, size_t ws_bytes,
                              void *stream);

/* ---- CSCC, the paper's comparison method.
 * Encoding = SI Alg. 5, the paper's simplification of the CSCC encoder
 * "designed for any value of K_w and s_w": output column s (stride s_w) owns
 * the K_w-wide submatrix of padded columns [s*s_w, s*s_w+K_w) -- the lowered matrix of SI
 * Eq. 17; its NZEs are stored row-major in the submatrix with
 * IN = (w - s*s_w) + h*K_w (h padded), ptr = [0, c_0 .. c_{O_w-1}] channel-cumulative
 * (O_w + 1 entries per channel; no NPC flag).  Channels n-major then c; the side tables and
 * `lengths` as for CPO (algo = SPC_ALGO_CSCC).  Any R, S, stride and padding. */
/* Host: capacities (ptr = N*C*(O_w+1); da = in = N*C*H*W*ceil(K_w/s_w)). */
spc_status spc_cscc_capacity(const spc_conv_desc *d, int64_t *ptr_cap, int64_t *da_cap, int64_t *in_cap);
/* Three launches (per-plane counts, one-CTA scan, per-plane writes); lengths[3] = 1 (and
 * nothing written) when a capacity is too small.  SPC_EUNSUPPORTED: plane (H*W*4 plus the
 * per-row counts) larger than one CTA's shared memory. */
spc_status cscc_encode(const spc_conv_desc *d, const float *x, spc_encoding *out, void *stream);
/* SI Alg. 6 over a CSCC encoding with packed [C][R][S][K] weights
 * (spc_pack_weights): y = conv(x, w) in fp32 (NKHW), ReLU if fuse_relu.  A flagged encoding
 * (lengths[3] != 0) gives y = 0. */
spc_status cscc_conv_forward(const spc_conv_desc *d, const spc_encoding *enc, const float *w_packed, float *y,
                             int32_t fuse_relu, void *stream);

/* NEXT-1: the convolution emits its output ALREADY CPO-encoded
 * for the next layer.  Computes y exactly as sparse_conv_forward (ReLU if fuse_relu; y is still
 * written) and, in the same kernel's epilogue, a row bitmask per output column of the non-zero
 * outputs; one small launch then builds the CPO streams of y for the layer `next` (whose
 * input is y: next->N == N, next->C == K, next->H == Oh, next->W == Ow) from the masks, reading
 * only y's NZEs -- bit-identical to cpo_encode(next, y) (no dense re-scan of y).  `out` as for
 * cpo_encode (algo = SPC_ALGO_CPO).  ws: >= spc_fused_ws_bytes(d), zeroed once
 * (spc_workspace_init), one stream at a time.  SPC_EUNSUPPORTED: next's padded height > 64 or
 * padded width > 256, or a stride-aware input encoding. */
size_t spc_fused_ws_bytes(const spc_conv_desc *d);
spc_status sparse_conv_encode_forward(const spc_conv_desc *d, const spc_encoding *enc, const float *w_packed,
                                      float *y, int32_t fuse_relu, const spc_conv_desc *next, spc_encoding *out,
                                      void *ws, size_t ws_bytes, void *stream);

/* Dense baseline: im2col lowering of x into ws_lowered (SI Eq. 6
 * elements, fp32), then y[n] = W[K x CRS] * L[n].  Layout: [N][C*R*S][Oh*Ow] for the
 * cuBLAS / SIMT engines, [N*Oh*Ow][C*R*S] (K-major, one GEMM over all images) for the
 * tcgen05 engine.  ws_bytes must be >= 4 * S_im2col. */
spc_status im2col_conv_forward(const spc_conv_desc *d, const float *x, const float *w_kcrs, float *y,
                               int32_t fuse_relu, void *ws_lowered, size_t ws_bytes, void *stream);
/* Recommended ws_bytes for im2col_conv_forward under the current engine: the lowered matrix
 * (4 * S_im2col, 256-byte aligned) plus, for the tcgen05 engine, 4 * K*C*R*S bytes where the
 * weights' lo halves (w minus its tf32 truncation) are formed once per call (with only
 * 4 * S_im2col they are formed per tile in shared memory: same results, slower).  Host only. */
size_t spc_im2col_ws_bytes(const spc_conv_desc *d);

/* GEMM engines of the dense baseline.  im2col_conv_forward uses the process-wide
 * default (spc_set_im2col_gemm; initially SPC_GEMM_AUTO: the tcgen05 3xTF32 kernel for
 * layers of >= 2^28 MACs, or >= 2^26 MACs over >= 20 output tiles of 128 positions x 64
 * (K <= 64) or 128 channels or with C*R*S >= 2048, with C*R*S % 4 == 0 (its TMA row pitches), cuBLAS FP32 otherwise,
 * both within the 1e-4 tolerance).  SPC_GEMM_TC_3XTF32 also falls back to cuBLAS FP32
 * when C*R*S % 4 != 0.  An engine the
 * loaded cuBLAS lacks makes im2col_conv_forward return SPC_EUNSUPPORTED (BF16X9
 * needs cuBLAS >= 12.9; PyTorch 2.11 bundles 12.8).  SPC_GEMM_SIMT is this library's own
 * FP32 FFMA kernel; the cuBLAS engines are plain library GEMMs (cublasGemmStridedBatchedEx):
 * FP32 = CUBLAS_COMPUTE_32F (FFMA), BF16X9 = CUBLAS_COMPUTE_32F_EMULATED_16BFX9
 * (fp32 emulated with three bf16 terms on the tensor cores), TF32 =
 * CUBLAS_COMPUTE_32F_FAST_TF32 (one tf32 term: faster, outside the 1e-4 tolerance;
 * reported for the crossover only). */
typedef enum {
    SPC_GEMM_SIMT = 0, SPC_GEMM_CUBLAS_FP32 = 1, SPC_GEMM_CUBLAS_BF16X9 = 2, SPC_GEMM_CUBLAS_TF32 = 3,
    SPC_GEMM_TC_3XTF32 = 4,  /* this library's tcgen05 kernel: fp32 from three TF32 products, TMEM accumulators */
    SPC_GEMM_AUTO = 5        /* TC_3XTF32 for large layers, CUBLAS_FP32 for small ones */
} spc_gemm;
spc_status spc_set_im2col_gemm(spc_gemm gemm);   /* SPC_EINVAL for an unknown engine */
spc_gemm spc_get_im2col_gemm(void);
/* How sparse_conv_forward decodes a CPS encoding (K_w > 1; Alg. 4), process-wide:
 * 0 (default) = a separate pass expands the CPS IN stream into CPO-form indices in the workspace,
 * then the CPO convolution runs; 1 = on the layers the warp-specialised conv serves (14x14 @ 256,
 * 7x7 @ 512, their stride-2 producers) its producer warps decode the CPS stream inline, per chunk
 * of input channels (one launch; the other layers keep the expansion pass).  Both give identical
 * outputs; the inline form measured slower on B200.  Initial value: the
 * SPC_CPS_INLINE environment variable, else 0.  SPC_EINVAL for a value other than 0 / 1.  Host only. */
spc_status spc_set_cps_inline(int32_t on);
int32_t spc_get_cps_inline(void);
/* The engine im2col_conv_forward runs for this layer under the current default (resolves
 * SPC_GEMM_AUTO and the tcgen05 engine's C*R*S % 4 fallback); host only. */
spc_gemm spc_im2col_engine(const spc_conv_desc *d);

/* Which kernel the calling host thread's last sparse_conv_forward / sparse_conv_encode_forward
 * (CPO, CPS or stride-aware encoding) launched: 2 = warp-specialised (ws_conv_kernel), 1 = strip
 * (strip_conv_kernel), 0 = generic, -1 = none yet.  Host only (benchmarks, tests). */
int spc_last_conv_kernel(void);

/* Host, synchronising (it times).  Per-layer offline selection:
 * over the M sample maps (device, M*N*C*H*W fp32), time encode+conv for CPO
 * and CPS and lowering+GEMM for im2col, `reps` times each, sum per algorithm
 * and return the argmin under `mode` (ties prefer the sparse algorithm,
 * reading A24).  times_ms (host float[3]) = {im2col, CPO, CPS} summed over
 * the M samples, per rep.  Geometries the sparse path rejects choose im2col
 * with times_ms[1..2] = -1.  ws: >= spc_select_ws_bytes(d). */
spc_status select_layer_algo(const spc_conv_desc *d, const float *samples, int32_t M, const float *w_kcrs,
                             spc_mode mode, int32_t reps, spc_algo *choice, float *times_ms, void *ws,
                             size_t ws_bytes, void *stream);
size_t spc_select_ws_bytes(const spc_conv_desc *d);

/* Host, no GPU work: the selection rule of select_layer_algo applied to recorded times
 * (replay, SPEC.md:657 / :741: the plan is the argmin on the profiling data).
 * times_ms = {im2col, CPO, CPS} (any consistent unit); sparse_ok = 0 restricts the choice
 * to im2col (times_ms[1..2] ignored).  Modes as spc_mode; ties prefer the
 * smaller footprint, CPS over CPO over im2col (reading A24).  SPC_EINVAL for negative or
 * NaN times in the considered set or an unknown mode. */
spc_status spc_select_from_times(const float *times_ms, int32_t sparse_ok, spc_mode mode, spc_algo *choice);

/* ---- SI space bounds as a zero-cost pre-selector.
 * All host-only, no GPU work.  Bounds are on the AVERAGE channel density rho_bar =
 * sum_{n,c} rho_{n,c} / (I_n I_c) (reading A29; the printed bounds carry a factor I_n I_c and
 * are then clipped to [0, 1]) in the SI's worst case (M = 1, VALID, no NPC, no NPF):
 *   vs im2col / MEC (:616-640): the stride-agnostic CPO layout (reading
 *     A15): O_w -> Ow1 = Wp - K_w + 1, ceil(K_w / s_w) -> K_w;
 *   vs CSCC: (2 O_w K_w Hp rho_hat_bar + (O_w+1)(2 - ceil(K_w/s_w)) - 3)
 *     / (2 H W), rho_hat_bar = the average per-image density of CSCC's lowered matrix (Eq. 17,
 *     padded frame, readings A30 / A31). */
typedef enum { SPC_SPACE_VS_IM2COL = 0, SPC_SPACE_VS_MEC = 1, SPC_SPACE_VS_CSCC = 2 } spc_space_vs;
/* rho_bar_max = P(rho)'s upper end (rho_hat_bar is used only for SPC_SPACE_VS_CSCC). */
spc_status spc_space_bound(const spc_conv_desc *d, spc_space_vs vs, double rho_hat_bar, double *rho_bar_max);
/* Q(rho_hat): the least rho_hat_bar for which the CSCC bound is >= 0. */
spc_status spc_cscc_q_bound(const spc_conv_desc *d, double *rho_hat_min);
/* favour-space pre-selection without timing: SPC_ALGO_CPO when rho_bar <= the bound, else the
 * dense comparison (SPC_ALGO_IM2COL, or SPC_ALGO_CSCC for vs = CSCC); geometries the sparse
 * path rejects (pointwise, ...) always get the dense one. */
spc_status spc_space_preselect(const spc_conv_desc *d, spc_space_vs vs, double rho_bar, double rho_hat_bar,
                               spc_algo *choice);

/* Host: output extents Oh = floor((H+pt+pb-R)/sh)+1, Ow = floor((W+pl+pr-S)/sw)+1
 * (reading A14) -- the dims every entry point uses for y. */
spc_status spc_output_dims(const spc_conv_desc *d, int32_t *oh, int32_t *ow);

/* Host, synchronising: copy the device `lengths` of an encoding to
 * out_host[3] = {ptr_len, da_len, in_len}; returns SPC_ECAPACITY if the
 * encoder reported an overflow (overflow word bit 0), SPC_ECUDA if a bounded
 * device-side wait timed out (bit 1: encoder, bit 2: balanced-mode conv). */
spc_status spc_encoding_lengths(const spc_encoding *enc, int64_t out_host[3], void *stream);

/* Host, synchronising; a debug validator, off the hot path.  Checks
 * that `enc` is a well-formed canonical CPO / CPS encoding for `d` (DESIGN.md Appendix A):
 * side tables monotone and equal to the device lengths; ptr block sequence, tags, NPC /
 * NPF placement, -1 exactly where a partition owns no column of the type, non-decreasing
 * counts adding up to each channel's NZEs; IN local columns / rows inside the real rows,
 * rows ascending per column; CPS set4 pairs decoding to the block's NZE count; DA values
 * non-zero and finite.  Returns SPC_ECORRUPT (message names the first bad channel
 * segment and the reason), SPC_ECAPACITY / SPC_ECUDA for a flagged encoding, SPC_OK
 * otherwise.  scratch: >= 16 bytes of device memory (overwritten). */
spc_status spc_validate_encoding(const spc_conv_desc *d, const spc_encoding *enc, void *scratch,
                                 size_t scratch_bytes, void *stream);

/* Thread-local message describing the last non-OK status of this thread. */
const char *spc_last_error(void);

/* Library build identification (sm_100a code object, git revision if known). */
const char *spc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPCONV_H */
