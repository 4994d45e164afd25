// launch.cu -- fixed cost of one graph-launched kernel on B200 as seen by CUDA events,
// after an L2-flushing write kernel: plain / large dynamic smem / cluster 8 / PDL.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void flush_kernel(float4* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}
__global__ void read_kernel(const float4* p, size_t n, float* out) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc += p[i].x;
    if (acc == 12345.f) out[0] = acc;
}
__global__ void empty_kernel(int* out) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0 && out == nullptr) sm[0] = 1;
}
__global__ void __cluster_dims__(1, 1, 8) empty_cluster(int* out) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0 && out == nullptr) sm[0] = 1;
}

int main() {
    size_t n = (256u << 20) / 16;
    float4* buf;
    cudaMalloc(&buf, n * 16);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(empty_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* names[] = {"plain 148x256", "smem 100KB", "smem 200KB", "cluster8 112 CTAs", "cluster8 + 60KB smem", "PDL attr", "2 kernels plain", "2 kernels 2nd PDL"};
    for (int v = 0; v < 8; v++) {
        cudaGraph_t gr;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int rep = 0; rep < (v >= 6 ? 2 : 1); rep++) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(148);
            cfg.blockDim = dim3(256);
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            cfg.attrs = at;
            cfg.numAttrs = 0;
            if (v == 1) cfg.dynamicSmemBytes = 100 * 1024;
            if (v == 2) cfg.dynamicSmemBytes = 200 * 1024;
            if (v == 5 || (v == 7 && rep == 1)) {
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.numAttrs = 1;
            }
            if (v == 3 || v == 4) {
                cfg.gridDim = dim3(14, 1, 8);
                cfg.blockDim = dim3(448);
                if (v == 4) cfg.dynamicSmemBytes = 60 * 1024;
                cudaLaunchKernelEx(&cfg, empty_cluster, (int*)buf);
            } else {
                cudaLaunchKernelEx(&cfg, empty_kernel, (int*)buf);
            }
        }
        cudaStreamEndCapture(st, &gr);
        cudaGraphInstantiate(&ge, gr, 0);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float tot = 0, best = 1e9;
        for (int i = 0; i < 60; i++) {
            flush_kernel<<<148 * 4, 512, 0, st>>>(buf, n);
            cudaEventRecord(a, st);
            cudaGraphLaunch(ge, st);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (i >= 10) { tot += ms; if (ms < best) best = ms; }
        }
        printf("%-24s median-ish mean %.2f us  best %.2f us\n", names[v], tot / 50 * 1e3, best * 1e3);
    }
    // direct stream launches (no graph) and a graph whose events are captured inside it
    {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int nk = 1; nk <= 2; nk++) {
            float tot = 0;
            for (int i = 0; i < 60; i++) {
                flush_kernel<<<148 * 4, 512, 0, st>>>(buf, n);
                cudaEventRecord(a, st);
                for (int k = 0; k < nk; k++) empty_kernel<<<148, 256, 0, st>>>((int*)buf);
                cudaEventRecord(b, st);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (i >= 10) tot += ms;
            }
            printf("direct %d kernel(s)       mean %.2f us\n", nk, tot / 50 * 1e3);
        }
        const char* fl[] = {"no flush", "write flush", "write flush + dummy kernel", "read flush"};
        for (int f = 0; f < 4; f++) {
            float tot = 0;
            for (int i = 0; i < 60; i++) {
                if (f == 1 || f == 2) flush_kernel<<<148 * 4, 512, 0, st>>>(buf, n);
                if (f == 2) empty_kernel<<<1, 32, 0, st>>>((int*)buf);
                if (f == 3) read_kernel<<<148 * 4, 512, 0, st>>>(buf, n, (float*)buf);
                cudaEventRecord(a, st);
                empty_kernel<<<148, 256, 0, st>>>((int*)buf);
                cudaEventRecord(b, st);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (i >= 10) tot += ms;
            }
            printf("%-28s 1 empty kernel: mean %.2f us\n", fl[f], tot / 50 * 1e3);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
