// Texture-gather throughput probe (B200): TLD4.R.AOFFI gathers per second on an
// L1-resident 64x64 u32 texture, 8 independent gathers in flight per thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tld4_probe tld4_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 g4(cudaTextureObject_t t, float x, float y) {
    uint4 g;
    asm volatile("tld4.r.2d.v4.u32.f32 {%0,%1,%2,%3}, [%4, {%5,%6}], {%7,%8};"
                 : "=r"(g.x), "=r"(g.y), "=r"(g.z), "=r"(g.w)
                 : "l"(t), "f"(x), "f"(y), "r"(1), "r"(1));
    return g;
}

__global__ void probe(cudaTextureObject_t t, int iters, unsigned* out) {
    unsigned acc = 0;
    const float bx = (float)(threadIdx.x & 31), by = (float)((threadIdx.x >> 5) & 7);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint4 g = g4(t, bx + (float)j, by + (float)(i & 15));
            acc += g.x ^ g.w;
        }
    }
    if (acc == 0x12345678u) out[blockIdx.x] = acc;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int W = 64;
    unsigned h[W * W];
    for (int i = 0; i < W * W; ++i) h[i] = i * 2654435761u;
    cudaChannelFormatDesc fd = cudaCreateChannelDesc(32, 0, 0, 0, cudaChannelFormatKindUnsigned);
    cudaArray_t arr;
    cudaMallocArray(&arr, &fd, W, W);
    cudaMemcpy2DToArray(arr, 0, 0, h, W * 4, W * 4, W, cudaMemcpyHostToDevice);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeArray;
    rd.res.array.array = arr;
    cudaTextureDesc td = {};
    td.addressMode[0] = td.addressMode[1] = cudaAddressModeBorder;
    td.filterMode = cudaFilterModePoint;
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t t;
    cudaCreateTextureObject(&t, &rd, &td, nullptr);
    unsigned* o;
    cudaMalloc(&o, 1 << 20);
    const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 2048;
    probe<<<blocks, threads>>>(t, 16, o);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        probe<<<blocks, threads>>>(t, iters, o);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double gathers = double(blocks) * threads * iters * 8;
    const double per_s = gathers / (best * 1e-3);
    printf("{\"tld4_lane_gathers_per_s\": %.4g, \"per_sm_per_clk_at_max\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d, "
           "\"ms\": %.3f, \"err\": \"%s\"}\n",
           per_s, per_s / p.multiProcessorCount / (clk * 1e3), p.multiProcessorCount, clk / 1000, best,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
