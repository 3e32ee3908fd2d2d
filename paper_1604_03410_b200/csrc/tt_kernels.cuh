// tt_kernels.cuh — launch interface of the sm_100a trace-transform kernels.
//
// The path: rotate the image through every orientation and reduce each line
// (a, p) with the T-functionals (arXiv 1604.03410 §7,
// /root/reference/PAPER.md:810-829).  Semantics: DESIGN.md §2.  The
// reference executes this path on its emulated device through
// DeviceContext::launch -> run_kernel
// (/root/reference/proj/include/gridjit/driver.hpp:221-247,
// emulator.hpp:747-793); these kernels replace that engine.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tt {

constexpr int kNumF = 6;  // T0..T5

enum class Sampler : int {
    Global = 0,   // 4 x LDG through L1 (row-major image in HBM/L2)
    Texture = 1,  // 1 x TLD4 (tex2Dgather) on a block-linear cudaArray copy
    Tma = 2,      // T0 only (n > 704, NS = 32, n % 4 == 0, one image): TMA-staged shared-memory tiles, 4 x LDS;
                  // other launches fall back to Texture (tex must then be set; tma_radon_ok())
};

struct TraceArgs {
    const float* img = nullptr;   // [n][n] row-major (Sampler::Global)
    cudaTextureObject_t tex = 0;  // same image as a 2-D texture (Sampler::Texture)
    int n = 0;                    // image side == line length == lines per angle
    int a0 = 0;                   // first angle (index into ctab/stab)
    int a_count = 0;              // launch units (angles a0 .. a0+a_count-1)
    int pair_stride = 0;          // >0: unit i also owns angle a0+i+pair_stride (rows partner_row+i)
    int partner_row = -1;         // first output row of the partner angles (-1: a_count; batch == 1 only)
    bool peer_out = false;        // out/med live in another GPU's memory: system-scope fence before exit
    const float* ctab = nullptr;  // [A_total] cos(theta_a), f64 -> f32 on host
    const float* stab = nullptr;  // [A_total] sin(theta_a)
    const float* wtab = nullptr;  // [n][8]: r, r^2, w3re, w3im, w4re, w4im, w5re, w5im (spec §2.2), 16-B aligned
    const float* wsoa = nullptr;  // full: launch_weights_soa(wtab) -- [n] float4 (w3, w4) then [n] float2 (w5)
    float* out = nullptr;         // full: [rows][6][n]; T0-only: [rows][n]; rows = a_count*(1+paired)
    int32_t* med = nullptr;       // full: [rows][2][n] (m, m'), may be null
    bool full = true;             // T0..T5 (else T0 / Radon only)
    Sampler sampler = Sampler::Global;
    int batch = 1;                // images in this launch (same n, same angles)
    int img0 = 0;                 // atlas/array index of the launch's first image (outputs stay launch-relative)
    long long img_stride = 0;     // elements between images (0: n*n) -- Global sampler
    int atlas_cols = 1;           // texture atlas tiles per row -- Texture sampler
    float* circ = nullptr;        // full: [rows][6][3] circus features of the launch's rows (separate circus launch)
    bool fuse_circus = false;     // with circ and the texture sampler: the P stage inside the trace launch
    int* epi = nullptr;           // with circ: epi_state_ints() zeroed ints (left zeroed); one per concurrent launch
};

// True when launch_trace serves a Sampler::Tma launch with the TMA tile kernel itself.
bool tma_radon_ok(const TraceArgs& a);
// ... and worth it: enough taps (units * n^2) to amortise its per-launch cost (the context's default sampler)
bool tma_radon_pays(const TraceArgs& a);
// Size (ints) of the fused P stage's state for a launch: per unit a line counter and a finished-row
// counter (zeroed once; every launch leaves them zeroed).
std::size_t epi_state_ints(const TraceArgs& a);

// Slots (lanes) per line of the fused kernel for side n: 8/16/32 (one warp
// segment) or 32W (W warps); T0-only launches with n > 1024 use 32 -- the
// reduction schedule that oracle/tt_oracle.c TTO_REPLAY mirrors.
int schedule_slots(int n, bool full = true);

// Launch units for a drop-in launch of a_count angles: pairs (i, i+a_count/2)
// when a_count is even (the kernel pairs mirrored angles).
inline void launch_structure(int a_count, int* units, int* pair_stride) {
    if (a_count >= 2 && a_count % 2 == 0) {
        *units = a_count / 2;
        *pair_stride = a_count / 2;
    } else {
        *units = a_count;
        *pair_stride = 0;
    }
}

// Pass-2 weight layout: the complex weights of wtab regrouped as [n] float4
// (w3re, w3im, w4re, w4im) followed by [n] float2 (w5re, w5im), so a warp's
// weight loads for 32 consecutive r are two fully used contiguous spans
// (r and r^2 are formed in registers, bit-identical to wtab's first columns).
inline std::size_t weights_soa_bytes(int n) { return std::size_t(n) * 24; }
cudaError_t launch_weights_soa(const float* wtab, int n, float* wsoa, cudaStream_t s);

// Largest n the fused T0-T5 kernel supports (line buffer must fit in smem).
int max_full_n();

// Enqueue the fused kernel on `stream`.  Returns cudaSuccess or the launch
// error.  Args must already be validated (sizes, n range).
cudaError_t launch_trace(const TraceArgs& a, cudaStream_t stream);

// Number of kernel launches launch_trace() issues (for gpu_launches claims).
int trace_launch_count(const TraceArgs& a);

// Native stand-ins for the reference's sample kernels (boundary tests):
// c[i] = a[i] + b[i], i = block + thread * blocks (0-based form of
// /root/reference/proj/kernels/vadd.krn:3-6).  elem: 4 (f32/i32) or 8 (f64/i64).
enum class ElemKind : int { F32 = 0, F64 = 1, I32 = 2, I64 = 3 };
cudaError_t launch_vadd(ElemKind k, const void* a, const void* b, void* c, uint64_t count, cudaStream_t s);

// a[i] *= k for i < count (/root/reference/proj/kernels/scale.krn:2-5).
cudaError_t launch_scale_f32(float* a, float k, uint64_t count, cudaStream_t s);

// b[i] = a[i] (copy, /root/reference/proj/tests/test_autolaunch.cpp:26-28) and
// out[i] = in[i] + out[i] (add_to, test_autolaunch.cpp:145) for i < count.
cudaError_t launch_copy_f32(const float* a, float* b, uint64_t count, cudaStream_t s);
cudaError_t launch_add_to_f32(const float* in, float* out, uint64_t count, cudaStream_t s);

// Texture object over a cudaArray holding a copy of img (caller owns both).
// true when make_image_texture makes a pitch-linear view of img (no cudaArray: *arr == nullptr)
bool pitch_texture_ok(const float* img, int n);
cudaError_t make_image_texture(const float* img, int n, cudaStream_t s, cudaArray_t* arr,
                               cudaTextureObject_t* tex);

// FP32 roofline probe: blocks x 256 threads x iters x 128 FFMA (2 flop each).
cudaError_t launch_ffma_probe(float* out, int blocks, int iters, cudaStream_t s);
cudaError_t launch_tld4_probe(unsigned* out, int blocks, int iters, cudaStream_t s);

// P-functionals (circus features) of `rows` sinogram rows of length n:
// circ[row][3] = (P1 total variation, P2 weighted-median value, P3 max),
// DESIGN.md §2.7.  One warp per row.
cudaError_t launch_circus(const float* sino, int n, int rows, float* circ, cudaStream_t s);
// Spectral P-functional sum_k |F(s)_k|^4 of each row, n <= max_circus_fft_n().
cudaError_t launch_circus_fft(const float* sino, int n, int rows, double* pout, cudaStream_t s);
int max_circus_fft_n();
// Hermite P-functionals H_0..H_{orders-1} of each row around its weighted median:
// hp[row][orders] (f64), center[row] = the median index (may be null); orders <= max_hermite_orders().
cudaError_t launch_hermite(const float* sino, int n, int rows, int orders, double* hp, int32_t* center, cudaStream_t s);
int max_hermite_orders();
// Orthonormal (square) sinogram input: h x w image resampled to s x s, s = orthonormal_side(A) =
// ceil(A / sqrt 2), centred in an A x A frame.
int orthonormal_side(int angles);
cudaError_t launch_orthonormal(const float* img, int h, int w, int angles, float* out, cudaStream_t s);

// Texture atlas of `batch` images (image b at tile (b % cols, b / cols)),
// 32-bit texels holding the float bits.
cudaError_t make_image_atlas(const float* imgs, int n, int batch, long long stride, cudaStream_t s, cudaArray_t* arr,
                             cudaTextureObject_t* tex, int* cols);

// Refill images [b0, b0 + batch) of an atlas created by make_image_atlas from
// imgs (image b0 first; stream-ordered).
cudaError_t fill_image_atlas(cudaArray_t arr, const float* imgs, int n, int batch, long long stride, int cols,
                             cudaStream_t s, int b0 = 0);
// The same through an existing surface object of the atlas array (no per-call object: graph-capturable).
cudaError_t fill_image_atlas_surf(cudaSurfaceObject_t surf, const float* imgs, int n, int batch, long long stride,
                                  int cols, cudaStream_t s, int b0 = 0);

// 8-bit gray/RGB picture (h x w x ch) -> n x n f32 gray, centred, zero padded.
cudaError_t launch_prep(const uint8_t* pix, int h, int w, int ch, int n, float* img, cudaStream_t s);

// Writes a buffer larger than L2 (timing hygiene between bench iterations).
cudaError_t launch_l2_flush(void* buf, uint64_t bytes, cudaStream_t s);

}  // namespace tt
