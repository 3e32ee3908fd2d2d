// Shared-memory bilinear sampling throughput probe (B200): the T0 per-tap work
// (coordinates, bounds, integer parts, fractions, bilinear, sum) with the 2x2
// footprint read by 4 LDS from an image tile in shared memory, lanes along a
// rotated line (32 consecutive taps per warp instruction), for several angles
// and tile pitches; the same arithmetic with one TLD4 per tap beside it.
// Question answered: can shared-memory tiles beat the texture-gather rate
// (2 lane-gathers / clk / SM) for the Radon path, and what do bank conflicts cost?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_sample_probe smem_sample_probe.cu
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int TW = 96;  // tile side (texels)

template <int P>
__global__ void __launch_bounds__(256, 4) lds_probe(const float* __restrict__ src, float c, float s, int iters,
                                                    float* out) {
    __shared__ float tile[TW * P];
    for (int i = threadIdx.x; i < TW * P; i += blockDim.x) tile[i] = src[i % (TW * TW)];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float o = 48.0f, hib = 94.0f;
    float acc = 0.0f;
    for (int i = 0; i < iters; ++i) {
        const float x = (float)((i * 8 + warp) & 31) - 16.0f;
        const float u = fmaf(x, c, o), w = fmaf(x, s, o);
#pragma unroll 4
        for (int j = 0; j < 2; ++j) {
            const float y = (float)(lane + 32 * j) - 32.0f;
            const float qx = fmaf(-y, s, u), qy = fmaf(y, c, w);
            const bool in = qx >= 0.0f && qy >= 0.0f && qx < hib && qy < hib;
            const float ixf = truncf(qx), iyf = truncf(qy);
            const float fx = qx - ixf, fy = qy - iyf;
            const int a = in ? (int)iyf * P + (int)ixf : 0;
            const float i00 = tile[a], i01 = tile[a + 1], i10 = tile[a + P], i11 = tile[a + P + 1];
            const float top = fmaf(fx, i01 - i00, i00), bot = fmaf(fx, i11 - i10, i10);
            const float v = fmaf(fy, bot - top, top);
            acc += in ? v : 0.0f;
        }
    }
    if (acc == 1.2345f) out[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(256, 4) tex_probe(cudaTextureObject_t t, float c, float s, int iters, float* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float o = 48.0f, hib = 94.0f;
    float acc = 0.0f;
    for (int i = 0; i < iters; ++i) {
        const float x = (float)((i * 8 + warp) & 31) - 16.0f;
        const float u = fmaf(x, c, o), w = fmaf(x, s, o);
#pragma unroll 4
        for (int j = 0; j < 2; ++j) {
            const float y = (float)(lane + 32 * j) - 32.0f;
            const float qx = fmaf(-y, s, u), qy = fmaf(y, c, w);
            const bool in = qx >= 0.0f && qy >= 0.0f && qx < hib && qy < hib;
            const float ixf = truncf(in ? qx : -1e7f), iyf = truncf(qy);
            const float fx = qx - ixf, fy = qy - iyf;
            uint4 g;
            asm volatile("tld4.r.2d.v4.u32.f32 {%0,%1,%2,%3}, [%4, {%5,%6}], {%7,%8};"
                         : "=r"(g.x), "=r"(g.y), "=r"(g.z), "=r"(g.w)
                         : "l"(t), "f"(ixf), "f"(iyf), "r"(1), "r"(1));
            const float i00 = __uint_as_float(g.w), i01 = __uint_as_float(g.z), i10 = __uint_as_float(g.x),
                        i11 = __uint_as_float(g.y);
            const float top = fmaf(fx, i01 - i00, i00), bot = fmaf(fx, i11 - i10, i10);
            const float v = fmaf(fy, bot - top, top);
            acc += in ? v : 0.0f;
        }
    }
    if (acc == 1.2345f) out[blockIdx.x] = acc;
}

template <class F>
static double run(F launch, int iters, int blocks, int clk_khz, int sms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double taps = (double)blocks * 256 * iters * 2;
    return taps / (ms * 1e-3) / ((double)clk_khz * 1e3) / sms;  // taps per clock per SM
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int sms = p.multiProcessorCount, blocks = sms * 4, iters = 4096;
    float* src;
    cudaMalloc(&src, TW * TW * 4);
    float h[TW * TW];
    for (int i = 0; i < TW * TW; ++i) h[i] = (float)((i * 2654435761u) >> 8) * 0x1p-24f;
    cudaMemcpy(src, h, sizeof h, cudaMemcpyHostToDevice);
    cudaChannelFormatDesc fd = cudaCreateChannelDesc(32, 0, 0, 0, cudaChannelFormatKindUnsigned);
    cudaArray_t arr;
    cudaMallocArray(&arr, &fd, TW, TW);
    cudaMemcpy2DToArray(arr, 0, 0, h, TW * 4, TW * 4, TW, cudaMemcpyHostToDevice);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeArray;
    rd.res.array.array = arr;
    cudaTextureDesc td = {};
    td.addressMode[0] = td.addressMode[1] = cudaAddressModeBorder;
    td.filterMode = cudaFilterModePoint;
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t t;
    cudaCreateTextureObject(&t, &rd, &td, nullptr);
    float* o;
    cudaMalloc(&o, 1 << 20);
    printf("{\"sm_clock_khz\": %d, \"sms\": %d, \"unit\": \"taps/clk/SM\", \"rows\": [\n", clk, sms);
    const double degs[] = {0, 5, 15, 30, 45, 60, 75, 85, 90};
    for (int k = 0; k < 9; ++k) {
        const double th = degs[k] * M_PI / 180.0;
        const float c = (float)cos(th), s = (float)sin(th);
        const double r96 = run([&] { lds_probe<96><<<blocks, 256>>>(src, c, s, iters, o); }, iters, blocks, clk, sms);
        const double r97 = run([&] { lds_probe<97><<<blocks, 256>>>(src, c, s, iters, o); }, iters, blocks, clk, sms);
        const double r100 = run([&] { lds_probe<100><<<blocks, 256>>>(src, c, s, iters, o); }, iters, blocks, clk, sms);
        const double rt = run([&] { tex_probe<<<blocks, 256>>>(t, c, s, iters, o); }, iters, blocks, clk, sms);
        printf("  {\"deg\": %.0f, \"lds_pitch96\": %.3f, \"lds_pitch97\": %.3f, \"lds_pitch100\": %.3f, \"tld4\": %.3f}%s\n",
               degs[k], r96, r97, r100, rt, k < 8 ? "," : "");
    }
    printf("]}\n");
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
