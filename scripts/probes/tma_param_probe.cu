// TMA descriptor placement probe: one 2-D tile load (box {P, 8} of a 256 x 256
// f32 image) through a tensor map that is (a) a __grid_constant__ kernel
// parameter, (b) element k of an array of maps inside a __grid_constant__
// struct, (c) in global memory.  Prints which forms load the right texels.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_param_probe tma_param_probe.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

struct Maps {
    CUtensorMap m[4];
};

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// FORM 0: shared::cluster + .tile; 1: shared::cluster (CUTLASS SM90_TMA_LOAD_2D form); 2: shared::cta
template <int FORM>
__device__ void load_tile(const CUtensorMap* map, int x, int y, int P, float* out) {
    __shared__ __align__(1024) float tile[256 * 8];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(P * 8 * 4)
                     : "memory");
        const unsigned long long d = reinterpret_cast<unsigned long long>(map);
        if (FORM == 0)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(su32(tile)), "l"(d), "r"(x), "r"(y), "r"(su32(&bar)) : "memory");
        if (FORM == 1)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(su32(tile)), "l"(d), "r"(x), "r"(y), "r"(su32(&bar)) : "memory");
        if (FORM == 2)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(su32(tile)), "l"(d), "r"(x), "r"(y), "r"(su32(&bar)) : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
            su32(&bar))
        : "memory");
    for (int i = threadIdx.x; i < P * 8; i += blockDim.x) out[i] = tile[i];
}

// non-tensor bulk copy of 8 rows of P floats (one cp.async.bulk per row)
__global__ void k_bulk(const float* img, int n, int x, int y, int P, float* out) {
    __shared__ __align__(1024) float tile[256 * 8];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(P * 8 * 4)
                     : "memory");
        for (int r = 0; r < 8; ++r)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(tile + r * P)),
                         "l"(img + (size_t)(y + r) * n + x), "r"(P * 4), "r"(su32(&bar))
                         : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
            su32(&bar))
        : "memory");
    for (int i = threadIdx.x; i < P * 8; i += blockDim.x) out[i] = tile[i];
}

template <int FORM>
__global__ void k_single(const __grid_constant__ CUtensorMap map, int x, int y, int P, float* out) {
    load_tile<FORM>(&map, x, y, P, out);
}
template <int FORM>
__global__ void k_array(const __grid_constant__ Maps maps, int k, int x, int y, int P, float* out) {
    load_tile<FORM>(&maps.m[k], x, y, P, out);
}
template <int FORM>
__global__ void k_global(const CUtensorMap* maps, int k, int x, int y, int P, float* out) {
    load_tile<FORM>(&maps[k], x, y, P, out);
}

int main(int argc, char** argv) {
    const int only = argc > 1 ? atoi(argv[1]) : -1;
    const int form = argc > 4 ? atoi(argv[4]) : 0;
    const int n = 256, P = argc > 2 ? atoi(argv[2]) : 64, x = argc > 3 ? atoi(argv[3]) : 10, y = 20;
    float* img;
    cudaMalloc(&img, n * n * 4);
    static float h[256 * 256];
    for (int i = 0; i < n * n; ++i) h[i] = (float)i;
    cudaMemcpy(img, h, sizeof h, cudaMemcpyHostToDevice);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    if (argc > 5 && atoi(argv[5]) == 1) enc = cuTensorMapEncodeTiled;  // the driver API symbol (-lcuda)
    if (argc > 5 && atoi(argv[5]) == 2) {  // versioned entry point
        cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q);
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    printf("entry point query %d, fn %p\n", (int)q, (void*)enc);
    Maps maps;
    for (int k = 0; k < 4; ++k) {
        const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
        const cuuint64_t strides[1] = {(cuuint64_t)n * 4};
        const cuuint32_t box[2] = {(cuuint32_t)(P), 8};
        const cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&maps.m[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, img, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) printf("encode %d failed: %d\n", k, (int)r);
    }
    {
        const unsigned* w = reinterpret_cast<const unsigned*>(&maps.m[0]);
        printf("desc:");
        for (int i = 0; i < 32; ++i) printf(" %08x", w[i]);
        printf("\n");
    }
    CUtensorMap* gmaps;
    cudaMalloc(&gmaps, sizeof maps);
    cudaMemcpy(gmaps, &maps, sizeof maps, cudaMemcpyHostToDevice);
    float* out;
    cudaMalloc(&out, P * 8 * 4);
    static float ho[256 * 8];
    const char* names[3] = {"grid_constant single", "grid_constant array[k=2]", "global memory"};
    for (int v = 0; v < 3; ++v) {
        if (only >= 0 && v != only) continue;
        cudaMemset(out, 0, P * 8 * 4);
#define TT_LAUNCH(F)                                                             \
    if (form == F) {                                                             \
        if (v == 0) k_single<F><<<1, 128>>>(maps.m[0], x, y, P, out);            \
        if (v == 1) k_array<F><<<1, 128>>>(maps, 2, x, y, P, out);               \
        if (v == 2) k_global<F><<<1, 128>>>(gmaps, 2, x, y, P, out);             \
    }
        if (argc > 6 && atoi(argv[6]) == 1) {  // cluster launch (1x1x1) through cudaLaunchKernelEx
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(1);
            cfg.blockDim = dim3(128);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 1;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_single<1>, maps.m[0], x, y, P, out);
        } else if (argc > 6 && atoi(argv[6]) == 2) {
            k_bulk<<<1, 128>>>(img, n, x, y, P, out);
        } else {
            TT_LAUNCH(0) TT_LAUNCH(1) TT_LAUNCH(2)
        }
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s form %d: %s\n", names[v], form, cudaGetErrorString(e));
            return 1;  // the context is unusable after a fault
        }
        cudaMemcpy(ho, out, P * 8 * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int r = 0; r < 8; ++r)
            for (int c = 0; c < P; ++c) bad += ho[r * P + c] != ((x + c >= 0 && x + c < n) ? (float)((y + r) * n + x + c) : 0.0f);
        printf("%s form %d: %s (%d wrong)\n", names[v], form, bad ? "WRONG" : "ok", bad);
    }
    return 0;
}
