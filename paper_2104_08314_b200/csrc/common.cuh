// common.cuh -- internal helpers of the sm_100a CPO/CPS library (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>

#include "../../include/spconv.h"

namespace spc {

constexpr int kWarp = 32;

// Geometry shared by encoder and convolution kernels (host-computed).
struct Geom {
    int N, C, H, W, K, R, S, sh, sw, pt, pb, pl, pr;
    int Hp, Wp;      // padded extents
    int Ow1, Oh1;    // stride-1 partition / output counts
    int Oh, Ow;      // output extents at the real stride (floor, reading A14)
    int nwords;      // 32-bit words per padded column mask = ceil(Hp / 32)
    long long NC;    // N * C channel planes
};

inline Geom make_geom(const spc_conv_desc& d) {
    Geom g;
    g.N = d.N; g.C = d.C; g.H = d.H; g.W = d.W; g.K = d.K; g.R = d.R; g.S = d.S;
    g.sh = d.stride_h; g.sw = d.stride_w;
    g.pt = d.pad_top; g.pb = d.pad_bottom; g.pl = d.pad_left; g.pr = d.pad_right;
    g.Hp = d.H + d.pad_top + d.pad_bottom;
    g.Wp = d.W + d.pad_left + d.pad_right;
    g.Ow1 = g.Wp - d.S + 1;
    g.Oh1 = g.Hp - d.R + 1;
    g.Oh = (g.Hp - d.R) / d.stride_h + 1;
    g.Ow = (g.Wp - d.S) / d.stride_w + 1;
    g.nwords = (g.Hp + 31) / 32;
    g.NC = (long long)d.N * d.C;
    return g;
}

// Encoder: 16 warps per CTA; a tile = P consecutive channel planes staged in smem.
constexpr int kEncWarps = 16;
constexpr int kEncMaxPlaneBytes = 192 * 1024;  // smem stage of one plane

// Cross-CTA prefix state of the single-pass encoder (lives in the workspace).
// Aggregates are tagged with epoch+1, so a launch never has to reset them; the
// CTA that owns the last tile bumps the epoch once every tile has published.
struct EncState {
    unsigned epoch;
    unsigned count[2];   // tiles published in launch e (slot e & 1); the other slot is reset for e+1
    int pad;
};

__host__ __device__ inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// ---- per-device launch caches (host).  Kernel attributes and SM counts belong to one
// device context, so every cache is an array indexed by the current device (the C ABI has
// no device argument: launches go to the caller's current device).  Races between threads
// only repeat an idempotent cudaFuncSetAttribute.
constexpr int kMaxDevices = 64;
inline int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
    return d;
}
inline int device_sm_count() {
    static std::atomic<int> n[kMaxDevices];
    const int dev = current_device();
    int v = n[dev].load(std::memory_order_relaxed);
    if (v <= 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        n[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}
// Raise cudaFuncAttributeMaxDynamicSharedMemorySize of `func` on the current device to at
// least `bytes` (cache: one std::atomic<size_t>[kMaxDevices] per kernel instantiation).
inline cudaError_t ensure_smem_attr(const void* func, size_t bytes, std::atomic<size_t>* cache) {
    std::atomic<size_t>& c = cache[current_device()];
    if (c.load(std::memory_order_relaxed) >= bytes) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) c.store(bytes, std::memory_order_relaxed);
    return e;
}

// Kernels whose CTAs wait on other CTAs of the same grid launch with
// cudaLaunchAttributeCooperative (co-scheduled grid).  SPC_COOPERATIVE=0 disables it
// (development A/B only).
inline bool cooperative_launches() {
    static const int on = [] {
        const char* e = getenv("SPC_COOPERATIVE");
        return (e && atoi(e) == 0) ? 0 : 1;
    }();
    return on != 0;
}

// upper bound on encoder tiles (one plane per tile), for workspace sizing
inline long long enc_tiles(const Geom& g) { return g.NC; }

size_t conv_scratch_bytes(const Geom& g);   // sparse_conv.cu: L2 partials of a cluster split

// Workspace layout: [EncState | flags[ntiles] (u64) | agg[3*ntiles] | cps_in[da_cap] | conv partials]
struct WsLayout {
    size_t state, flags, agg, cps_in, scratch, total;
};

inline WsLayout ws_layout(const Geom& g) {
    WsLayout L;
    long long nt = enc_tiles(g);
    L.state = 0;
    L.flags = align_up(sizeof(EncState), 256);
    L.agg = align_up(L.flags + sizeof(unsigned long long) * (size_t)nt, 256);
    L.cps_in = align_up(L.agg + sizeof(long long) * 3 * (size_t)nt, 256);
    L.scratch = align_up(L.cps_in + sizeof(int32_t) * (size_t)(g.NC * g.H * g.W), 256);
    L.total = align_up(L.scratch + conv_scratch_bytes(g), 256);
    return L;
}

// Development probes (built only with -DSPC_PROBES): thread 0 of every CTA
// stamps %globaltimer and clock64 at phase boundaries into a per-TU buffer;
// spc_debug_probes_<tu>() copies it out.  Compiled out of the product library.
constexpr int kProbeCtas = 1024, kProbeSlots = 16;
#ifdef SPC_PROBES
static __device__ unsigned long long g_probe[kProbeCtas][kProbeSlots][2];
#define SPC_PROBE_ACCESSOR(name)                                                                 \
    extern "C" int name(unsigned long long* host, int clear) {                                   \
        cudaDeviceSynchronize();                                                                 \
        if (cudaMemcpyFromSymbol(host, spc::g_probe, sizeof(spc::g_probe)) != cudaSuccess) return -1; \
        if (clear) {                                                                             \
            void* p = nullptr;                                                                   \
            cudaGetSymbolAddress(&p, spc::g_probe);                                              \
            cudaMemset(p, 0, sizeof(spc::g_probe));                                              \
        }                                                                                        \
        return 0;                                                                                \
    }
__device__ __forceinline__ void probe(int slot) {
    if (threadIdx.x == 0 && blockIdx.x + blockIdx.y * gridDim.x + blockIdx.z * gridDim.x * gridDim.y < kProbeCtas) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        const unsigned b = blockIdx.x + blockIdx.y * gridDim.x + blockIdx.z * gridDim.x * gridDim.y;
        g_probe[b][slot][0] = t;
        g_probe[b][slot][1] = clock64();
    }
}
// any thread may stamp (the caller elects it)
__device__ __forceinline__ void probe_any(int slot) {
    if (blockIdx.x + blockIdx.y * gridDim.x + blockIdx.z * gridDim.x * gridDim.y < kProbeCtas && slot < kProbeSlots) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        const unsigned b = blockIdx.x + blockIdx.y * gridDim.x + blockIdx.z * gridDim.x * gridDim.y;
        g_probe[b][slot][0] = t;
        g_probe[b][slot][1] = clock64();
    }
}
#else
__device__ __forceinline__ void probe(int) {}
__device__ __forceinline__ void probe_any(int) {}
#endif

// Programmatic dependent launch (sm_90+): a secondary kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization starts while its primary
// still runs; pdl_wait() blocks until the primary grid has completed and its
// memory is visible (a no-op when launched without the attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- device helpers --------------------------------------------------------

// 1D TMA bulk copies (cp.async.bulk) into shared memory, completion counted on an
// mbarrier in transaction bytes.  Sizes and addresses are multiples of 16 bytes.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_release32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_exclusive_scan(T v, T* total) {
    const int lane = threadIdx.x & 31;
    T inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    *total = __shfl_sync(0xffffffffu, inc, 31);
    return inc - v;
}

}  // namespace spc

// Internal launchers (defined in the .cu files, called from api.cu).
namespace spc {
cudaError_t launch_encode(const Geom& g, bool cps, const float* x, spc_encoding* e, void* ws, cudaStream_t st,
                          bool sa = false);
cudaError_t launch_pack_weights(const Geom& g, const float* w, float* wp, cudaStream_t st);
cudaError_t launch_cps_expand(const Geom& g, const spc_encoding* e, int32_t* in_cpo, cudaStream_t st);
int last_conv_kernel();   // sparse_conv.cu: kernel of this thread's last sparse-conv launch
cudaError_t launch_sparse_conv(const Geom& g, const spc_encoding* e, const int32_t* in_override,
                               const float* w_packed, float* y, int relu, float* scratch, size_t scratch_bytes,
                               cudaStream_t st, unsigned long long* omask = nullptr, unsigned sa_types = 0,
                               int cscc = 0, bool cps_inline = false);
cudaError_t launch_im2col(const Geom& g, const float* x, float* L, cudaStream_t st);
cudaError_t launch_gemm(const Geom& g, const float* w, const float* L, float* y, int relu, cudaStream_t st,
                        float* extra = nullptr, size_t extra_bytes = 0);   // extra: workspace beyond the lowered matrix
cudaError_t launch_tc_gemm(const Geom& g, const float* w, const float* L, float* y, int relu, cudaStream_t st,
                           float* bsplit);   // bsplit: 2*K*C*R*S floats or null
int gemm_engine();
int gemm_engine_for(const Geom& g);   // effective engine of a layer (AUTO / fallbacks resolved)
void set_gemm_engine(int e);
}  // namespace spc
