// dsmem.cu -- cost of distributed-shared-memory traffic inside an 8-CTA cluster on sm_100a:
// (a) every thread stores N scattered 4-byte words into a peer's smem, then cluster.sync;
// (b) every thread loads N 16-byte words from all 8 peers (8 loads in flight), then sync.
// Reports microseconds per phase (globaltimer), median over CTAs.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__device__ __forceinline__ float4 ld_cluster_v4(const float4* local_ptr, unsigned rank) {
    unsigned a = (unsigned)__cvta_generic_to_shared(local_ptr), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(ra));
    return v;
}
__device__ __forceinline__ void st_cluster_f32(float* local_ptr, unsigned rank, float v) {
    unsigned a = (unsigned)__cvta_generic_to_shared(local_ptr), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f32 [%0], %1;" :: "r"(ra), "f"(v) : "memory");
}

__global__ void __cluster_dims__(8, 1, 1) k(int nst, int nld, unsigned long long* out, float* sink, int explicit_) {
    extern __shared__ float sm[];   // 16K floats
    auto cl = cg::this_cluster();
    const int r = cl.block_rank();
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = (float)i;
    cl.sync();
    unsigned long long t0 = gt();
    // (a) scattered remote stores
    for (int i = 0; i < nst; i++) {
        const int peer = (r + 1 + (threadIdx.x + i) % 7) % 8;
        if (explicit_) {
            st_cluster_f32(sm + ((threadIdx.x * 37 + i * 101) & 16383), peer, (float)i);
        } else {
            float* p = cl.map_shared_rank(sm, peer);
            p[(threadIdx.x * 37 + i * 101) & 16383] = (float)i;
        }
    }
    cl.sync();
    unsigned long long t1 = gt();
    // (b) remote float4 loads from all peers
    float acc = 0.f;
    for (int i = 0; i < nld; i++) {
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; q++)
            v[q] = explicit_ ? ld_cluster_v4(reinterpret_cast<float4*>(sm) + ((threadIdx.x + i * 448) & 4095), q)
                             : reinterpret_cast<float4*>(cl.map_shared_rank(sm, q))[(threadIdx.x + i * 448) & 4095];
#pragma unroll
        for (int q = 0; q < 8; q++) acc += v[q].x + v[q].w;
    }
    cl.sync();
    unsigned long long t2 = gt();
    if (acc == 1234.5f) sink[0] = acc;
    if (threadIdx.x == 0) {
        const int b = blockIdx.x;
        out[3 * b] = t1 - t0; out[3 * b + 1] = t2 - t1;
    }
}

int main() {
    unsigned long long* out; float* sink;
    cudaMalloc(&out, 3 * 112 * 8); cudaMalloc(&sink, 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    int cfgs[][2] = {{0, 0}, {3, 0}, {10, 0}, {0, 1}, {0, 4}};
    for (int ex = 0; ex < 2; ex++)
    for (auto& c : cfgs) {
        for (int rep = 0; rep < 3; rep++) k<<<112, 448, 65536>>>(c[0], c[1], out, sink, ex);
        cudaDeviceSynchronize();
        unsigned long long h[3 * 112];
        cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
        double a = 0, b = 0;
        for (int i = 0; i < 112; i++) { a += h[3 * i]; b += h[3 * i + 1]; }
        printf("%s stores/thread %2d loads(x8 peers)/thread %d: store phase %.2f us, load phase %.2f us  (%s)\n", ex ? "explicit" : "generic ", c[0], c[1],
               a / 112 / 1e3, b / 112 / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
