// api.cu -- extern "C" entry points of libspconv.so (declared in include/spconv.h).
// Host-side validation, workspace carving, launches and the offline selector.
#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

#include <atomic>

// CPS decode form of sparse_conv_forward (spc_set_cps_inline): 0 = expansion pass, 1 = inline
static std::atomic<int32_t> g_cps_inline{[] {
    const char* v = getenv("SPC_CPS_INLINE");
    return (v && atoi(v) == 1) ? 1 : 0;
}()};

namespace spc {
size_t enc_smem_bytes(const Geom& g);
const char* validate_reason(int code);
size_t cscc_smem_bytes(const Geom& g);
cudaError_t launch_cscc_encode(const Geom& g, const float* x, spc_encoding* e, cudaStream_t st);
cudaError_t launch_cscc_conv(const Geom& g, const spc_encoding* e, const float* w_packed, float* y, int relu,
                             cudaStream_t st);
size_t sa_smem_bytes(const Geom& g);
int sa_types(const Geom& g);
cudaError_t launch_sa_encode(const Geom& g, const float* x, spc_encoding* e, cudaStream_t st);
cudaError_t launch_encode_from_masks(const Geom& gn, const float* y, unsigned long long* omask, spc_encoding* e,
                                     void* state, cudaStream_t st);
size_t fe_state_bytes(const Geom& gn);
cudaError_t launch_sa_conv(const Geom& g, const spc_encoding* e, const float* w_packed, float* y, int relu,
                           cudaStream_t st);
cudaError_t launch_validate(const Geom& g, const spc_encoding* e, void* rec_dev, cudaStream_t st,
                            long long* bad_channel, int* code);
}

namespace {

thread_local std::string g_err;

spc_status fail(spc_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
spc_status fail(spc_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

spc_status cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return SPC_OK;
    return fail(SPC_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

spc_status check_desc(const spc_conv_desc* d) {
    if (!d) return fail(SPC_EINVAL, "null descriptor");
    if (d->N < 1 || d->C < 1 || d->H < 1 || d->W < 1 || d->K < 1 || d->R < 1 || d->S < 1)
        return fail(SPC_EINVAL, "dimensions must be >= 1");
    if (d->stride_h < 1 || d->stride_w < 1) return fail(SPC_EINVAL, "strides must be >= 1");
    if (d->pad_top < 0 || d->pad_bottom < 0 || d->pad_left < 0 || d->pad_right < 0)
        return fail(SPC_EINVAL, "negative padding");
    if (d->H + d->pad_top + d->pad_bottom < d->R || d->W + d->pad_left + d->pad_right < d->S)
        return fail(SPC_EINVAL, "kernel larger than the padded input");
    return SPC_OK;
}

// Preconditions of the canonical encoding (DESIGN.md A.1).
spc_status check_sparse_geometry(const spc_conv_desc* d) {
    spc_status s = check_desc(d);
    if (s != SPC_OK) return s;
    const int Wp = d->W + d->pad_left + d->pad_right;
    if (d->R == 1 && d->S == 1) return fail(SPC_EUNSUPPORTED, "pointwise kernels are routed to im2col (PAPER.md:123)");
    if (d->S > 8) return fail(SPC_EUNSUPPORTED, "K_w > 8 not supported");
    // padded-frame row masks are shifted by pad_top inside 32-bit words (pad_top <= R-1 < 32)
    if (d->R > 32) return fail(SPC_EUNSUPPORTED, "K_h > 32 not supported");
    if (d->S > 1) {
        if (d->pad_left != d->pad_right) return fail(SPC_EUNSUPPORTED, "pad_left != pad_right (reading A16)");
        if (d->pad_left > d->S - 1) return fail(SPC_EUNSUPPORTED, "pad_left >= K_w");
        if (Wp < 2 * d->S - 1) return fail(SPC_EUNSUPPORTED, "padded width < 2*K_w - 1 (reading A17)");
    } else if (d->pad_left || d->pad_right) {
        return fail(SPC_EUNSUPPORTED, "K_w = 1 with horizontal padding");
    }
    if (d->pad_top > d->R - 1 || d->pad_bottom > d->R - 1) return fail(SPC_EUNSUPPORTED, "vertical pad >= K_h");
    if ((long long)d->H * d->W * 4 > spc::kEncMaxPlaneBytes)
        return fail(SPC_EUNSUPPORTED, "channel plane larger than the encoder smem stage");
    const long long Hp = d->H + d->pad_top + d->pad_bottom;
    if ((long long)(d->S - 1) + (Hp - 1) * d->S >= (1ll << 31)) return fail(SPC_EUNSUPPORTED, "index overflow");
    return SPC_OK;
}

void caps_of(const spc::Geom& g, int64_t* pc, int64_t* dc, int64_t* ic) {
    const long long per = (g.S == 1) ? (1 + g.Ow1) : (3 + (long long)(g.S - 1) * (1 + g.Ow1));
    *pc = g.NC * per;
    *dc = g.NC * g.H * g.W;
    *ic = *dc;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

spc_status do_encode(const spc_conv_desc* d, const float* x, spc_encoding* out, void* ws, size_t ws_bytes,
                     void* stream, bool cps) {
    spc_status s = check_sparse_geometry(d);
    if (s != SPC_OK) return s;
    if (!x || !out || !ws) return fail(SPC_EINVAL, "null pointer");
    if (!out->ptr || !out->da || !out->in || !out->chan_ptr_off || !out->chan_nz_off || !out->chan_in_off ||
        !out->lengths)
        return fail(SPC_EINVAL, "null stream pointer in spc_encoding");
    if (!aligned16(x)) return fail(SPC_EINVAL, "x must be 16-byte aligned");
    spc::Geom g = spc::make_geom(*d);
    if ((size_t)spc::ws_layout(g).cps_in > ws_bytes) return fail(SPC_EINVAL, "workspace too small");
    if (out->ptr_cap < 0 || out->da_cap < 0 || out->in_cap < 0) return fail(SPC_EINVAL, "negative capacity");
    out->algo = cps ? SPC_ALGO_CPS : SPC_ALGO_CPO;   // S = 1: CPS streams equal CPO (reading A13)
    out->geom = *d;
    return cuda_status(spc::launch_encode(g, cps && d->S > 1, x, out, ws, (cudaStream_t)stream), "encode");
}

}  // namespace

extern "C" {

const char* spc_last_error(void) { return g_err.c_str(); }


const char* spc_version(void) {
#ifndef SPC_GIT_REV
#define SPC_GIT_REV "unknown"
#endif
    return "spconv-b200 sm_100a rev " SPC_GIT_REV;
}

spc_status spc_encode_capacity(const spc_conv_desc* d, int64_t* ptr_cap, int64_t* da_cap, int64_t* in_cap,
                               size_t* ws_bytes) {
    spc_status s = check_sparse_geometry(d);
    if (s != SPC_OK) return s;
    spc::Geom g = spc::make_geom(*d);
    int64_t pc, dc, ic;
    caps_of(g, &pc, &dc, &ic);
    if (ptr_cap) *ptr_cap = pc;
    if (da_cap) *da_cap = dc;
    if (in_cap) *in_cap = ic;
    if (ws_bytes) *ws_bytes = spc::ws_layout(g).total;
    return SPC_OK;
}

spc_status spc_workspace_init(void* ws, size_t ws_bytes, void* stream) {
    if (!ws) return fail(SPC_EINVAL, "null workspace");
    cudaError_t e = cudaMemsetAsync(ws, 0, ws_bytes, (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
    return cuda_status(e, "spc_workspace_init");
}

spc_status cpo_encode(const spc_conv_desc* d, const float* x, spc_encoding* out, void* ws, size_t ws_bytes,
                      void* stream) {
    return do_encode(d, x, out, ws, ws_bytes, stream, false);
}

spc_status cps_encode(const spc_conv_desc* d, const float* x, spc_encoding* out, void* ws, size_t ws_bytes,
                      void* stream) {
    return do_encode(d, x, out, ws, ws_bytes, stream, true);
}

spc_status spc_pack_weights(const spc_conv_desc* d, const float* w_kcrs, float* w_packed, void* stream) {
    spc_status s = check_desc(d);
    if (s != SPC_OK) return s;
    if (!w_kcrs || !w_packed) return fail(SPC_EINVAL, "null pointer");
    spc::Geom g = spc::make_geom(*d);
    return cuda_status(spc::launch_pack_weights(g, w_kcrs, w_packed, (cudaStream_t)stream), "pack_weights");
}

}  // extern "C"

namespace {
spc_status conv_impl(const spc_conv_desc* d, const spc_encoding* enc, const float* w_packed, float* y,
                     int32_t fuse_relu, void* ws, size_t ws_bytes, void* stream, unsigned long long* omask) {
    spc_status s = check_sparse_geometry(d);
    if (s != SPC_OK) return s;
    if (!enc || !w_packed || !y) return fail(SPC_EINVAL, "null pointer");
    if (enc->algo != SPC_ALGO_CPO && enc->algo != SPC_ALGO_CPS && enc->algo != SPC_ALGO_CPO_SA)
        return fail(SPC_EINVAL, "not a CPO / CPS / stride-aware CPO encoding");
    const spc_conv_desc& e = enc->geom;
    if (e.N != d->N || e.C != d->C || e.H != d->H || e.W != d->W || e.R != d->R || e.S != d->S ||
        e.pad_top != d->pad_top || e.pad_bottom != d->pad_bottom || e.pad_left != d->pad_left ||
        e.pad_right != d->pad_right)
        return fail(SPC_EINVAL, "encoding geometry does not match the descriptor");
    spc::Geom g = spc::make_geom(*d);
    cudaStream_t st = (cudaStream_t)stream;
    if (enc->algo == SPC_ALGO_CPO_SA) {
        // the layout depends on the horizontal stride (reading A32)
        if (e.stride_w != d->stride_w) return fail(SPC_EINVAL, "stride-aware encoding made for another stride");
        if ((size_t)4 * g.Oh * 32 * 8 > 227 * 1024) return fail(SPC_EUNSUPPORTED, "output too tall");
        if (omask) return fail(SPC_EUNSUPPORTED, "fused encode: CPO / CPS input encodings only");
        // the coverage types present in the padded row (which (partition, type) slots exist)
        unsigned types = 0;
        for (int w = 0; w < g.Wp; w++) {
            int cov = 0;
            for (int s2 = 0; s2 < g.Ow; s2++)
                if (s2 * g.sw <= w && w < s2 * g.sw + g.S) cov++;
            if (cov) types |= 1u << (cov - 1);
        }
        static const bool force_simple = [] { const char* e = getenv("SPC_SA_SIMPLE"); return e && atoi(e); }();
        // the strip / ws producers address (partition, type) slots of the window: <= 32 per channel
        const int T = (d->S + d->stride_w - 1) / d->stride_w;
        const int WW = 3 * d->stride_w + d->S;                      // window columns of a 4-output strip
        const bool slots_ok = ((WW + d->S - 2) / d->stride_w + 2) * T <= (WW <= 8 ? 8 : 16);
        if (slots_ok && !force_simple) {
            float* scratch = nullptr;
            size_t scratch_bytes = 0;
            if (ws) {
                const spc::WsLayout L = spc::ws_layout(g);
                if (ws_bytes >= L.total && L.total > L.scratch) {
                    scratch = reinterpret_cast<float*>(static_cast<unsigned char*>(ws) + L.scratch);
                    scratch_bytes = L.total - L.scratch;
                }
            }
            const cudaError_t ce = spc::launch_sparse_conv(g, enc, nullptr, w_packed, y, fuse_relu, scratch, scratch_bytes,
                                                           st, nullptr, types);
            if (ce != cudaErrorNotSupported) return cuda_status(ce, "sparse_conv (stride-aware)");
        }
        return cuda_status(spc::launch_sa_conv(g, enc, w_packed, y, fuse_relu, st), "sparse_conv (stride-aware)");
    }
    float* scratch = nullptr;
    size_t scratch_bytes = 0;
    if (ws) {
        const spc::WsLayout L = spc::ws_layout(g);
        if (ws_bytes >= L.total && L.total > L.scratch) {
            scratch = reinterpret_cast<float*>(static_cast<unsigned char*>(ws) + L.scratch);
            scratch_bytes = L.total - L.scratch;
        }
    }
    const int32_t* in_cpo = nullptr;
    if (enc->algo == SPC_ALGO_CPS && d->S > 1) {
        spc::WsLayout L = spc::ws_layout(g);
        if (!ws || ws_bytes < L.total) return fail(SPC_EINVAL, "CPS convolution needs the workspace");
        int32_t* buf = reinterpret_cast<int32_t*>(static_cast<unsigned char*>(ws) + L.cps_in);
        // the warp-specialised conv decodes the CPS stream itself (Alg. 4 inline, one launch);
        // the other conv kernels read CPO-form indices expanded by a separate pass
        if (g_cps_inline.load(std::memory_order_relaxed)) {
            const cudaError_t ce = spc::launch_sparse_conv(g, enc, buf, w_packed, y, fuse_relu, scratch, scratch_bytes,
                                                           st, omask, 0, 0, true);
            if (ce != cudaErrorNotSupported) return cuda_status(ce, "sparse_conv (CPS inline)");
        }
        spc_status r = cuda_status(spc::launch_cps_expand(g, enc, buf, st), "cps_expand");
        if (r != SPC_OK) return r;
        in_cpo = buf;
    }
    return cuda_status(spc::launch_sparse_conv(g, enc, in_cpo, w_packed, y, fuse_relu, scratch, scratch_bytes, st, omask),
                       "sparse_conv");
}
}  // namespace

extern "C" {

spc_status sparse_conv_forward(const spc_conv_desc* d, const spc_encoding* enc, const float* w_packed, float* y,
                               int32_t fuse_relu, void* ws, size_t ws_bytes, void* stream) {
    return conv_impl(d, enc, w_packed, y, fuse_relu, ws, ws_bytes, stream, nullptr);
}

size_t spc_fused_ws_bytes(const spc_conv_desc* d) {
    if (check_sparse_geometry(d) != SPC_OK) return 0;
    const spc::Geom g = spc::make_geom(*d);
    spc_conv_desc nd = *d;                     // the next layer's planes: N*K of them
    nd.C = d->K; nd.H = g.Oh; nd.W = g.Ow;
    return spc::align_up(spc::ws_layout(g).total, 256) + spc::align_up((size_t)8 * g.N * g.K * g.Ow, 256) +
           spc::align_up(spc::fe_state_bytes(spc::make_geom(nd)), 256);
}

spc_status sparse_conv_encode_forward(const spc_conv_desc* d, const spc_encoding* enc, const float* w_packed,
                                      float* y, int32_t fuse_relu, const spc_conv_desc* next, spc_encoding* out,
                                      void* ws, size_t ws_bytes, void* stream) {
    spc_status s = check_sparse_geometry(next);
    if (s != SPC_OK) return s;
    s = check_sparse_geometry(d);
    if (s != SPC_OK) return s;
    const spc::Geom g = spc::make_geom(*d), gn = spc::make_geom(*next);
    if (next->N != d->N || next->C != d->K || next->H != g.Oh || next->W != g.Ow)
        return fail(SPC_EINVAL, "next layer's input must be this layer's output (N, K, Oh, Ow)");
    if (gn.Hp > 64 || gn.Wp > 256) return fail(SPC_EUNSUPPORTED, "fused encode: padded height <= 64, width <= 256");
    if (!out || !out->ptr || !out->da || !out->in || !out->chan_ptr_off || !out->chan_nz_off || !out->chan_in_off ||
        !out->lengths || !ws)
        return fail(SPC_EINVAL, "null pointer");
    const size_t need = spc_fused_ws_bytes(d);
    if (ws_bytes < need) return fail(SPC_EINVAL, "fused workspace too small (%zu < %zu)", ws_bytes, need);
    const size_t mo = spc::align_up(spc::ws_layout(g).total, 256);
    unsigned long long* omask = reinterpret_cast<unsigned long long*>(static_cast<unsigned char*>(ws) + mo);
    static const int dbg = [] { const char* e = getenv("SPC_FUSE_DEBUG"); return e ? atoi(e) : 0; }();
    s = conv_impl(d, enc, w_packed, y, fuse_relu, ws, mo, stream, dbg == 2 ? nullptr : omask);   // dev A/B: 2 = no masks
    if (s != SPC_OK) return s;
    out->algo = SPC_ALGO_CPO;
    out->geom = *next;
    if (dbg >= 1) return SPC_OK;   // dev A/B: 1 = masks only, no stream build
    void* fstate = static_cast<unsigned char*>(ws) + mo + spc::align_up((size_t)8 * g.N * g.K * g.Ow, 256);
    return cuda_status(spc::launch_encode_from_masks(gn, y, omask, out, fstate, (cudaStream_t)stream),
                       "encode_from_masks");
}

spc_status im2col_conv_forward(const spc_conv_desc* d, const float* x, const float* w_kcrs, float* y,
                               int32_t fuse_relu, void* ws_lowered, size_t ws_bytes, void* stream) {
    spc_status s = check_desc(d);
    if (s != SPC_OK) return s;
    if (!x || !w_kcrs || !y || !ws_lowered) return fail(SPC_EINVAL, "null pointer");
    spc::Geom g = spc::make_geom(*d);
    const size_t need = (size_t)4 * g.N * g.C * g.R * g.S * g.Oh * g.Ow;
    if (ws_bytes < need) return fail(SPC_EINVAL, "lowered-matrix workspace too small (%zu < %zu)", ws_bytes, need);
    cudaStream_t st = (cudaStream_t)stream;
    float* L = static_cast<float*>(ws_lowered);
    spc_status r = cuda_status(spc::launch_im2col(g, x, L, st), "im2col");
    if (r != SPC_OK) return r;
    const size_t lowered = spc::align_up(need, 256);
    float* extra = ws_bytes > lowered ? reinterpret_cast<float*>(static_cast<unsigned char*>(ws_lowered) + lowered) : nullptr;
    const cudaError_t ge = spc::launch_gemm(g, w_kcrs, L, y, fuse_relu, st, extra, extra ? ws_bytes - lowered : 0);
    if (ge == cudaErrorNotSupported)
        return fail(SPC_EUNSUPPORTED, "GEMM engine %d is not supported by the loaded cuBLAS", spc::gemm_engine());
    return cuda_status(ge, "gemm");
}

spc_status spc_set_im2col_gemm(spc_gemm gemm) {
    if (gemm < SPC_GEMM_SIMT || gemm > SPC_GEMM_AUTO) return fail(SPC_EINVAL, "unknown GEMM engine %d", (int)gemm);
    spc::set_gemm_engine((int)gemm);
    return SPC_OK;
}

spc_gemm spc_get_im2col_gemm(void) { return (spc_gemm)spc::gemm_engine(); }

spc_status spc_set_cps_inline(int32_t on) {
    if (on != 0 && on != 1) return fail(SPC_EINVAL, "spc_set_cps_inline: 0 or 1");
    g_cps_inline.store(on);
    return SPC_OK;
}
int32_t spc_get_cps_inline(void) { return g_cps_inline.load(); }

int spc_last_conv_kernel(void) { return spc::last_conv_kernel(); }

size_t spc_im2col_ws_bytes(const spc_conv_desc* d) {
    if (!d || check_desc(d) != SPC_OK) return 0;
    const spc::Geom g = spc::make_geom(*d);
    const size_t lowered = spc::align_up((size_t)4 * g.N * g.C * g.R * g.S * g.Oh * g.Ow, 256);
    const bool tc = spc::gemm_engine_for(g) == SPC_GEMM_TC_3XTF32;
    return lowered + (tc ? spc::align_up((size_t)4 * g.K * g.C * g.R * g.S, 256) : 0);
}

spc_gemm spc_im2col_engine(const spc_conv_desc* d) {
    if (!d || check_desc(d) != SPC_OK) return spc_get_im2col_gemm();
    return (spc_gemm)spc::gemm_engine_for(spc::make_geom(*d));
}

spc_status spc_encoding_lengths(const spc_encoding* enc, int64_t out_host[3], void* stream) {
    if (!enc || !enc->lengths || !out_host) return fail(SPC_EINVAL, "null pointer");
    int64_t h[4];
    cudaError_t e = cudaMemcpyAsync(h, enc->lengths, sizeof h, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "spc_encoding_lengths");
    out_host[0] = h[0]; out_host[1] = h[1]; out_host[2] = h[2];
    if (h[3] & 6) return fail(SPC_ECUDA, "a bounded device-side wait timed out (overflow word %lld: bit 1 encoder, "
                              "bit 2 balanced-mode conv)", (long long)h[3]);
    if (h[3]) return fail(SPC_ECAPACITY, "encoder overflow: needs ptr %lld da %lld in %lld", (long long)h[0],
                          (long long)h[1], (long long)h[2]);
    return SPC_OK;
}

spc_status spc_validate_encoding(const spc_conv_desc* d, const spc_encoding* enc, void* scratch,
                                 size_t scratch_bytes, void* stream) {
    spc_status s = check_sparse_geometry(d);
    if (s != SPC_OK) return s;
    if (!enc || !scratch || scratch_bytes < 16) return fail(SPC_EINVAL, "bad argument");
    if (enc->algo != SPC_ALGO_CPO && enc->algo != SPC_ALGO_CPS) return fail(SPC_EINVAL, "the validator checks CPO / CPS");
    if (!enc->ptr || !enc->da || !enc->in || !enc->chan_ptr_off || !enc->chan_nz_off || !enc->chan_in_off ||
        !enc->lengths)
        return fail(SPC_EINVAL, "null stream pointer in spc_encoding");
    const spc_conv_desc& e = enc->geom;
    if (e.N != d->N || e.C != d->C || e.H != d->H || e.W != d->W || e.R != d->R || e.S != d->S ||
        e.pad_top != d->pad_top || e.pad_bottom != d->pad_bottom || e.pad_left != d->pad_left ||
        e.pad_right != d->pad_right)
        return fail(SPC_EINVAL, "encoding geometry does not match the descriptor");
    int64_t len[3];
    s = spc_encoding_lengths(enc, len, stream);
    if (s != SPC_OK) return s;
    spc::Geom g = spc::make_geom(*d);
    long long bad = -1;
    int code = 0;
    s = cuda_status(spc::launch_validate(g, enc, scratch, (cudaStream_t)stream, &bad, &code), "validate");
    if (s != SPC_OK) return s;
    if (bad >= 0)
        return fail(SPC_ECORRUPT, "encoding corrupt at channel segment %lld (n=%lld, c=%lld): %s", bad, bad / g.C,
                    bad % g.C, spc::validate_reason(code));
    return SPC_OK;
}

// ------------------------------------------------------------ CSCC baseline

namespace {
spc_status check_cscc_geometry(const spc_conv_desc* d) {
    spc_status s = check_desc(d);
    if (s != SPC_OK) return s;
    const spc::Geom g = spc::make_geom(*d);
    if (spc::cscc_smem_bytes(g) > 227 * 1024) return fail(SPC_EUNSUPPORTED, "CSCC: plane too large for one CTA");
    if ((size_t)4 * g.Oh * 32 * 8 > 227 * 1024) return fail(SPC_EUNSUPPORTED, "CSCC: output too tall");
    if ((long long)(d->S - 1) + (long long)(g.Hp - 1) * d->S >= (1ll << 31)) return fail(SPC_EUNSUPPORTED, "index overflow");
    return SPC_OK;
}
}  // namespace

spc_status spc_cscc_capacity(const spc_conv_desc* d, int64_t* ptr_cap, int64_t* da_cap, int64_t* in_cap) {
    spc_status s = check_cscc_geometry(d);
    if (s != SPC_OK) return s;
    const spc::Geom g = spc::make_geom(*d);
    // an NZE is stored once per submatrix holding its column: at most ceil(K_w / s_w) times
    const long long kc = (d->S + d->stride_w - 1) / d->stride_w;
    if (ptr_cap) *ptr_cap = g.NC * (g.Ow + 1);
    if (da_cap) *da_cap = g.NC * g.H * g.W * kc;
    if (in_cap) *in_cap = g.NC * g.H * g.W * kc;
    return SPC_OK;
}

spc_status cscc_encode(const spc_conv_desc* d, const float* x, spc_encoding* out, void* stream) {
    spc_status s = check_cscc_geometry(d);
    if (s != SPC_OK) return s;
    if (!x || !out || !out->ptr || !out->da || !out->in || !out->chan_ptr_off || !out->chan_nz_off ||
        !out->chan_in_off || !out->lengths)
        return fail(SPC_EINVAL, "null pointer");
    if (out->ptr_cap < 0 || out->da_cap < 0 || out->in_cap < 0) return fail(SPC_EINVAL, "negative capacity");
    out->algo = SPC_ALGO_CSCC;
    out->geom = *d;
    return cuda_status(spc::launch_cscc_encode(spc::make_geom(*d), x, out, (cudaStream_t)stream), "cscc_encode");
}

spc_status cscc_conv_forward(const spc_conv_desc* d, const spc_encoding* enc, const float* w_packed, float* y,
                             int32_t fuse_relu, void* stream) {
    spc_status s = check_cscc_geometry(d);
    if (s != SPC_OK) return s;
    if (!enc || !w_packed || !y) return fail(SPC_EINVAL, "null pointer");
    if (enc->algo != SPC_ALGO_CSCC) return fail(SPC_EINVAL, "not a CSCC encoding");
    const spc_conv_desc& e = enc->geom;
    if (e.N != d->N || e.C != d->C || e.H != d->H || e.W != d->W || e.R != d->R || e.S != d->S ||
        e.stride_w != d->stride_w || e.pad_top != d->pad_top || e.pad_bottom != d->pad_bottom ||
        e.pad_left != d->pad_left || e.pad_right != d->pad_right)
        return fail(SPC_EINVAL, "encoding geometry does not match the descriptor");
    // the strip kernel reads CSCC's submatrices as window slots (NZE column = s*s_w + IN % K_w;
    // an NZE held by several submatrices lands on the same window cell) where a per-channel
    // configuration exists and the slots fit a warp; else the plain SI Alg. 6 kernel
    static const bool force_simple = [] { const char* e = getenv("SPC_CSCC_SIMPLE"); return e && atoi(e); }();
    const spc::Geom g = spc::make_geom(*d);
    const int WW = 3 * d->stride_w + d->S;
    if (!force_simple && d->S <= 8 && d->R <= 32 && (WW + d->S - 2) / d->stride_w + 2 <= 32 &&
        check_sparse_geometry(d) == SPC_OK) {
        const cudaError_t ce = spc::launch_sparse_conv(g, enc, nullptr, w_packed, y, fuse_relu, nullptr, 0,
                                                       (cudaStream_t)stream, nullptr, 0, 1);
        if (ce != cudaErrorNotSupported) return cuda_status(ce, "cscc_conv (strip)");
    }
    g_err.clear();
    return cuda_status(spc::launch_cscc_conv(g, enc, w_packed, y, fuse_relu, (cudaStream_t)stream), "cscc_conv");
}

// ------------------------------------------------------------ stride-aware CPO layout (NEXT-4)

spc_status spc_strided_capacity(const spc_conv_desc* d, int64_t* ptr_cap, int64_t* da_cap, int64_t* in_cap) {
    spc_status s = check_desc(d);
    if (s != SPC_OK) return s;
    if (d->R == 1 && d->S == 1) return fail(SPC_EUNSUPPORTED, "pointwise kernels are routed to im2col (PAPER.md:123)");
    if (d->S > 8) return fail(SPC_EUNSUPPORTED, "K_w > 8 not supported");
    const spc::Geom g = spc::make_geom(*d);
    if (spc::sa_smem_bytes(g) * 8 > 227 * 1024) return fail(SPC_EUNSUPPORTED, "plane too large (8 planes per CTA)");
    if ((long long)(d->S - 1) + (long long)(g.Hp - 1) * d->S >= (1ll << 31)) return fail(SPC_EUNSUPPORTED, "index overflow");
    if (ptr_cap) *ptr_cap = g.NC * std::max<long long>(1, (long long)spc::sa_types(g) * (1 + g.Ow));
    if (da_cap) *da_cap = g.NC * g.H * g.W;
    if (in_cap) *in_cap = g.NC * g.H * g.W;
    return SPC_OK;
}

spc_status cpo_encode_strided(const spc_conv_desc* d, const float* x, spc_encoding* out, void* ws, size_t ws_bytes,
                              void* stream) {
    spc_status s = spc_strided_capacity(d, nullptr, nullptr, nullptr);
    if (s != SPC_OK) return s;
    if (!x || !out || !out->ptr || !out->da || !out->in || !out->chan_ptr_off || !out->chan_nz_off ||
        !out->chan_in_off || !out->lengths)
        return fail(SPC_EINVAL, "null pointer");
    if (out->ptr_cap < 0 || out->da_cap < 0 || out->in_cap < 0) return fail(SPC_EINVAL, "negative capacity");
    const spc::Geom g = spc::make_geom(*d);
    // single pass (the canonical encoder's kernel with the layout's column order and blocks) when
    // a workspace is given and the canonical preconditions hold; else the three-launch encoder
    static const bool three = [] { const char* e = getenv("SPC_SA_3PASS"); return e && atoi(e); }();
    const bool one = ws && !three && check_sparse_geometry(d) == SPC_OK && aligned16(x) &&
                     (size_t)spc::ws_layout(g).cps_in <= ws_bytes;
    g_err.clear();
    out->algo = SPC_ALGO_CPO_SA;
    out->geom = *d;
    if (one) return cuda_status(spc::launch_encode(g, false, x, out, ws, (cudaStream_t)stream, true), "cpo_encode_strided");
    return cuda_status(spc::launch_sa_encode(g, x, out, (cudaStream_t)stream), "cpo_encode_strided");
}

// ------------------------------------------------------------ SI space bounds (NEXT-3)

namespace {
double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }
}

spc_status spc_space_bound(const spc_conv_desc* d, spc_space_vs vs, double rho_hat_bar, double* rho_bar_max) {
    spc_status s = check_desc(d);
    if (s != SPC_OK) return s;
    if (!rho_bar_max) return fail(SPC_EINVAL, "null pointer");
    const spc::Geom g = spc::make_geom(*d);
    const double HW = (double)d->H * d->W;
    if (vs == SPC_SPACE_VS_IM2COL || vs == SPC_SPACE_VS_MEC) {
        // PAPER.md:596-640 (reading A29): stride-agnostic encoding (A15), O_w -> Ow1, ceil -> K_w
        const double inner = (vs == SPC_SPACE_VS_IM2COL) ? (double)d->S * d->R * g.Oh1 : (double)d->S * d->H;
        *rho_bar_max = clip01((g.Ow1 * (inner + 1 - d->S) - 2 - d->S) / (2.0 * HW));
        return SPC_OK;
    }
    if (vs == SPC_SPACE_VS_CSCC) {
        // PAPER.md:663-684 (readings A30, A31): S_CSCC of Eq. 17 on the padded frame
        if (!(rho_hat_bar >= 0.0 && rho_hat_bar <= 1.0)) return fail(SPC_EINVAL, "rho_hat_bar outside [0, 1]");
        const int kc = (d->S + d->stride_w - 1) / d->stride_w;
        *rho_bar_max = clip01((2.0 * g.Ow * d->S * g.Hp * rho_hat_bar + (double)(g.Ow + 1) * (2 - kc) - 3) / (2.0 * HW));
        return SPC_OK;
    }
    return fail(SPC_EINVAL, "unknown comparison %d", (int)vs);
}

spc_status spc_cscc_q_bound(const spc_conv_desc* d, double* rho_hat_min) {
    spc_status s = check_desc(d);
    if (s != SPC_OK) return s;
    if (!rho_hat_min) return fail(SPC_EINVAL, "null pointer");
    const spc::Geom g = spc::make_geom(*d);
    const int kc = (d->S + d->stride_w - 1) / d->stride_w;
    // Q(rho_hat), per image (reading A31)
    *rho_hat_min = (3.0 - (double)(g.Ow + 1) * (2 - kc)) / (2.0 * g.Ow * g.Hp * d->S);
    return SPC_OK;
}

spc_status spc_space_preselect(const spc_conv_desc* d, spc_space_vs vs, double rho_bar, double rho_hat_bar,
                               spc_algo* choice) {
    if (!choice) return fail(SPC_EINVAL, "null pointer");
    double b = 0.0;
    spc_status s = spc_space_bound(d, vs, rho_hat_bar, &b);
    if (s != SPC_OK) return s;
    const spc_algo dense = (vs == SPC_SPACE_VS_CSCC) ? SPC_ALGO_CSCC : SPC_ALGO_IM2COL;
    if (check_sparse_geometry(d) != SPC_OK) {   // pointwise etc.: the sparse path does not apply
        g_err.clear();
        *choice = dense;
        return SPC_OK;
    }
    *choice = (rho_bar <= b) ? SPC_ALGO_CPO : dense;
    return SPC_OK;
}

// ------------------------------------------------------------ selection

size_t spc_select_ws_bytes(const spc_conv_desc* d) {
    if (check_desc(d) != SPC_OK) return 0;
    spc::Geom g = spc::make_geom(*d);
    size_t total = 0;
    const size_t lowered = spc_im2col_ws_bytes(d);
    const size_t yb = spc::align_up((size_t)4 * g.N * g.K * g.Oh * g.Ow, 256);
    const size_t wpb = spc::align_up((size_t)4 * g.K * g.C * g.R * g.S, 256);
    total += lowered + yb + wpb;
    if (check_sparse_geometry(d) == SPC_OK) {
        int64_t pc, dc, ic;
        caps_of(g, &pc, &dc, &ic);
        total += spc::align_up(4 * pc, 256) + spc::align_up(4 * dc, 256) + spc::align_up(4 * ic, 256);
        total += 3 * spc::align_up(8 * (g.NC + 1), 256) + 256;
        total += spc::ws_layout(g).total;
    }
    g_err.clear();
    return total;
}

spc_status select_layer_algo(const spc_conv_desc* d, const float* samples, int32_t M, const float* w_kcrs,
                             spc_mode mode, int32_t reps, spc_algo* choice, float* times_ms, void* ws,
                             size_t ws_bytes, void* stream) {
    spc_status s = check_desc(d);
    if (s != SPC_OK) return s;
    if (!samples || !w_kcrs || !choice || !times_ms || !ws || M < 1 || reps < 1)
        return fail(SPC_EINVAL, "bad argument");
    if (ws_bytes < spc_select_ws_bytes(d)) return fail(SPC_EINVAL, "selection workspace too small");
    spc::Geom g = spc::make_geom(*d);
    cudaStream_t st = (cudaStream_t)stream;
    unsigned char* p = static_cast<unsigned char*>(ws);
    auto take = [&](size_t b) { unsigned char* r = p; p += spc::align_up(b, 256); return r; };
    const size_t lowered_bytes = spc_im2col_ws_bytes(d);
    float* lowered = reinterpret_cast<float*>(take(lowered_bytes));
    float* y = reinterpret_cast<float*>(take((size_t)4 * g.N * g.K * g.Oh * g.Ow));
    float* wp = reinterpret_cast<float*>(take((size_t)4 * g.K * g.C * g.R * g.S));
    const bool sparse_ok = check_sparse_geometry(d) == SPC_OK;
    g_err.clear();
    const size_t per_sample = (size_t)g.N * g.C * g.H * g.W;
    cudaEvent_t e0, e1;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
        return fail(SPC_ECUDA, "event create");
    float t[3] = {0.f, -1.f, -1.f};
    spc_status r = SPC_OK;
    // im2col: lowering + GEMM
    for (int rep = 0; rep < reps + 1 && r == SPC_OK; rep++) {
        cudaEventRecord(e0, st);
        for (int m = 0; m < M && r == SPC_OK; m++)
            r = im2col_conv_forward(d, samples + m * per_sample, w_kcrs, y, 0, lowered, lowered_bytes, stream);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0) t[0] += ms;  // rep 0 is warm-up
    }
    if (sparse_ok && r == SPC_OK) {
        spc_encoding enc;
        memset(&enc, 0, sizeof enc);
        int64_t pc, dc, ic;
        caps_of(g, &pc, &dc, &ic);
        enc.ptr = reinterpret_cast<int32_t*>(take(4 * pc)); enc.ptr_cap = pc;
        enc.da = reinterpret_cast<float*>(take(4 * dc)); enc.da_cap = dc;
        enc.in = reinterpret_cast<int32_t*>(take(4 * ic)); enc.in_cap = ic;
        enc.chan_ptr_off = reinterpret_cast<int64_t*>(take(8 * (g.NC + 1)));
        enc.chan_nz_off = reinterpret_cast<int64_t*>(take(8 * (g.NC + 1)));
        enc.chan_in_off = reinterpret_cast<int64_t*>(take(8 * (g.NC + 1)));
        enc.lengths = reinterpret_cast<int64_t*>(take(64));
        const size_t ews = spc::ws_layout(g).total;
        void* ew = take(ews);
        r = cuda_status(cudaMemsetAsync(ew, 0, ews, st), "select ws init");
        if (r == SPC_OK) r = spc_pack_weights(d, w_kcrs, wp, stream);
        for (int a = 0; a < 2 && r == SPC_OK; a++) {
            const bool cps = a == 1;
            float tot = 0.f;
            for (int rep = 0; rep < reps + 1 && r == SPC_OK; rep++) {
                cudaEventRecord(e0, st);
                for (int m = 0; m < M && r == SPC_OK; m++) {
                    r = cps ? cps_encode(d, samples + m * per_sample, &enc, ew, ews, stream)
                            : cpo_encode(d, samples + m * per_sample, &enc, ew, ews, stream);
                    if (r == SPC_OK) r = sparse_conv_forward(d, &enc, wp, y, 0, ew, ews, stream);
                }
                cudaEventRecord(e1, st);
                cudaEventSynchronize(e1);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep > 0) tot += ms;
            }
            t[1 + a] = tot;
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (r != SPC_OK) return r;
    for (int i = 0; i < 3; i++) times_ms[i] = (t[i] >= 0.f) ? t[i] / reps : -1.f;
    return spc_select_from_times(times_ms, sparse_ok ? 1 : 0, mode, choice);
}

spc_status spc_select_from_times(const float* times_ms, int32_t sparse_ok, spc_mode mode, spc_algo* choice) {
    if (!times_ms || !choice) return fail(SPC_EINVAL, "null pointer");
    if (mode < SPC_FAVOUR_TIME || mode > SPC_BEST_OF_THREE) return fail(SPC_EINVAL, "unknown mode %d", (int)mode);
    if (!(times_ms[0] >= 0.f)) return fail(SPC_EINVAL, "im2col time must be >= 0");
    if (sparse_ok && (!(times_ms[1] >= 0.f) || !(times_ms[2] >= 0.f)))
        return fail(SPC_EINVAL, "sparse times must be >= 0 when sparse_ok");
    // argmin; ties prefer the smaller footprint: CPS over CPO over im2col (reading A24)
    spc_algo best = SPC_ALGO_IM2COL;
    float tb = times_ms[0];
    if (sparse_ok) {
        if (mode != SPC_FAVOUR_SPACE && times_ms[1] <= tb) { best = SPC_ALGO_CPO; tb = times_ms[1]; }
        if (mode != SPC_FAVOUR_TIME && times_ms[2] <= tb) { best = SPC_ALGO_CPS; tb = times_ms[2]; }
    }
    *choice = best;
    return SPC_OK;
}

spc_status spc_output_dims(const spc_conv_desc* d, int32_t* oh, int32_t* ow) {
    spc_status s = check_desc(d);
    if (s != SPC_OK) return s;
    if (!oh || !ow) return fail(SPC_EINVAL, "null pointer");
    const spc::Geom g = spc::make_geom(*d);
    *oh = g.Oh;
    *ow = g.Ow;
    return SPC_OK;
}

}  // extern "C"
