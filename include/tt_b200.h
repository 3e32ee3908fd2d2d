/*
 * tt_b200.h — C ABI of the B200-native trace-transform device
 * (libtt_b200.so, built from paper_1604_03410_b200/csrc/).
 *
 * This is the drop-in boundary: every entry point below replaces one
 * operation of the reference's driver-style API,
 *   /root/reference/proj/include/gridjit/driver.hpp  (DeviceContext)
 *   /root/reference/proj/include/gridjit/emulator.hpp (launch/trap types)
 * and is exactly what an FFI binding of that API would bind (plain pointers,
 * sizes and PODs; no C++ or torch types).  The C++ surface of the reference
 * is restored on top of it, source-compatibly, by include/tt/gridjit_b200.hpp;
 * INTEGRATION.md shows the ctypes and C++ bindings.
 *
 * Differences from the emulated device, all deliberate:
 *   - module_load reads only the `.module` / `.kernel name(params)` header of
 *     the VPTX text (/root/reference/proj/include/gridjit/vptx.hpp:398-488) and
 *     binds each kernel to a native sm_100a implementation registered for that
 *     exact signature; kernels with no native implementation fail at
 *     tt_get_function with TT_ERR_FUNCTION_NOT_FOUND.  There is no CPU
 *     fallback of any kind.
 *   - launches are stream-ordered on the context's CUDA stream; copies are
 *     synchronous, so every observable result matches the reference's
 *     synchronous launch.
 *   - kernel faults are detected on the host before the launch (buffer extents
 *     are known) and returned as tt_trap values, like TrapInfo; a trapping
 *     launch has no device side effects.
 */
#ifndef TT_B200_H
#define TT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TT_ABI_VERSION 1

/* One status per exception class of /root/reference/proj/include/gridjit/errors.hpp. */
typedef enum tt_status {
    TT_OK = 0,
    TT_ERR_CONTEXT_DESTROYED = 1, /* ContextDestroyed   errors.hpp:106-109 */
    TT_ERR_VPTX_SYNTAX = 2,       /* VptxSyntaxError    errors.hpp:97-102   */
    TT_ERR_VALIDATION_FAILED = 3, /* ValidationFailed   errors.hpp:111-123 */
    TT_ERR_FUNCTION_NOT_FOUND = 4,/* FunctionNotFound   errors.hpp:125-128 */
    TT_ERR_OUT_OF_BOUNDS = 5,     /* OutOfBounds        errors.hpp:130-133 */
    TT_ERR_DOUBLE_FREE = 6,       /* DoubleFree         errors.hpp:135-138 */
    TT_ERR_USE_AFTER_FREE = 7,    /* UseAfterFree       errors.hpp:140-143 */
    TT_ERR_ARGUMENT_MISMATCH = 8, /* ArgumentMismatch   errors.hpp:145-148 */
    TT_ERR_LAUNCH_CONFIG = 9,     /* LaunchConfigError  errors.hpp:150-153 */
    TT_ERR_ARITY = 10,            /* ArityError         errors.hpp:46-54    */
    TT_ERR_CUDA = 11,             /* CUDA runtime failure (no emulator analogue) */
    TT_ERR_INVALID = 12           /* misuse of the C ABI itself (null pointer, short buffer) */
} tt_status;

typedef struct tt_ctx tt_ctx; /* DeviceContext, driver.hpp:112 */

/* DeviceCaps, emulator.hpp:55-58 (logical launch limits checked by tt_launch). */
typedef struct tt_caps {
    uint32_t max_block_threads; /* default 1024 */
    uint64_t max_shared_bytes;  /* default 48 KiB */
} tt_caps;

/* DevicePtr, driver.hpp:45-49: a value handle; base is a synthetic address in
 * the reference's arena convention (first 4096, 256-B aligned, never reused),
 * mapped to pooled HBM. */
typedef struct tt_devptr {
    uint64_t base;
    uint64_t length; /* bytes */
    uint64_t ctx_id;
} tt_devptr;

/* ModuleHandle / FunctionHandle, driver.hpp:31-43 */
typedef struct tt_module {
    uint64_t ctx_id;
    uint64_t id;
} tt_module;
typedef struct tt_function {
    uint64_t ctx_id;
    uint64_t id;
} tt_function;

/* GridConfig, emulator.hpp:42-53 */
typedef struct tt_grid {
    uint32_t grid[3];
    uint32_t block[3];
    uint64_t shared_bytes_extra;
} tt_grid;

/* LaunchArg = std::variant<int32_t,int64_t,float,double,DevicePtr>, driver.hpp:52 */
typedef enum tt_arg_kind { TT_ARG_I32 = 0, TT_ARG_I64 = 1, TT_ARG_F32 = 2, TT_ARG_F64 = 3, TT_ARG_PTR = 4 } tt_arg_kind;
typedef struct tt_arg {
    int32_t kind; /* tt_arg_kind */
    int32_t _pad;
    union {
        int32_t i32;
        int64_t i64;
        float f32;
        double f64;
        tt_devptr ptr;
    } v;
} tt_arg;

/* TrapInfo::Kind, emulator.hpp:61-68 */
typedef enum tt_trap_kind {
    TT_TRAP_GLOBAL_OUT_OF_BOUNDS = 0,
    TT_TRAP_SHARED_OUT_OF_BOUNDS = 1,
    TT_TRAP_USE_OF_FREED_MEMORY = 2,
    TT_TRAP_DIVISION_BY_ZERO = 3,
    TT_TRAP_BARRIER_DIVERGENCE = 4,
    TT_TRAP_EXPLICIT = 5
} tt_trap_kind;

/* LaunchResult / TrapInfo, emulator.hpp:60-102 (trapped == 0 <=> ok()). */
typedef struct tt_trap {
    int32_t trapped;
    int32_t kind;       /* tt_trap_kind */
    uint32_t thread[3]; /* 1-indexed, source-language convention */
    uint32_t block[3];  /* 1-indexed */
    uint64_t instr_index;
    int64_t code;
} tt_trap;

/* Counters scalars, driver.hpp:54-96 (launch_log / events via the calls below). */
typedef struct tt_counters {
    uint64_t modules_loaded;
    uint64_t functions_resolved;
    uint64_t launches;
    uint64_t allocs;
    uint64_t frees;
    uint64_t bytes_h2d;
    uint64_t bytes_d2h;
    uint64_t launch_log_size;
    uint64_t events_size;
    uint64_t gpu_kernel_launches; /* native CUDA kernels enqueued (extension) */
} tt_counters;

/* Counters::Event, driver.hpp:55 */
typedef enum tt_event {
    TT_EV_MODULE_LOAD = 0,
    TT_EV_FUNCTION_RESOLVE = 1,
    TT_EV_ALLOC = 2,
    TT_EV_FREE = 3,
    TT_EV_H2D = 4,
    TT_EV_D2H = 5,
    TT_EV_LAUNCH = 6
} tt_event;

/* ---- library ------------------------------------------------------------ */
int tt_abi_version(void);
tt_status tt_device_count(int* out);
/* Last error text of ctx, or of the calling thread when ctx is NULL. */
const char* tt_last_error(const tt_ctx* ctx);
/* Registered native kernels, one rendered Signature per line
 * (types.hpp:100-113 rendering, e.g. "trace_t05(f32[],i32,...)"). */
tt_status tt_native_kernels(char* buf, size_t cap, size_t* needed);

/* ---- context (driver.hpp:112-132, 332) -------------------------------------- */
tt_status tt_ctx_create(int device, const tt_caps* caps, tt_ctx** out); /* create_context */
tt_status tt_ctx_destroy(tt_ctx* ctx);  /* DeviceContext::destroy: release + poison */
void tt_ctx_release(tt_ctx* ctx);       /* free the handle object (destroys if alive) */
tt_status tt_ctx_id(const tt_ctx* ctx, uint64_t* out);
tt_status tt_ctx_synchronize(tt_ctx* ctx);
tt_status tt_ctx_stream(tt_ctx* ctx, void** stream_out); /* cudaStream_t for interop */
tt_status tt_ctx_device(const tt_ctx* ctx, int* device_out);
/* Extension: image sampler of this context's trace launches:
 * 0 = global/L1 loads, 1 = texture gather (TLD4) for every launch, 2 =
 * TMA-staged shared-memory tiles for the T0-only launches they serve (n > 704,
 * n % 4 == 0, one image) and the texture gather for every other launch, 3
 * (default) = as 2 for T0 launches of at least 1.5e8 taps (units * n^2), whose
 * per-launch cost the tiles amortise, the texture gather otherwise -- the
 * measured-faster sampler for each.  Every sampler gives the same
 * bits.  Plans always sample through their texture unless the sampler is 0. */
tt_status tt_ctx_set_sampler(tt_ctx* ctx, int sampler);

/* ---- modules and functions (driver.hpp:138-177) ------------------------------ */
tt_status tt_module_load(tt_ctx* ctx, const char* vptx_text, size_t len, tt_module* out);
tt_status tt_module_unload(tt_ctx* ctx, tt_module m);
tt_status tt_get_function(tt_ctx* ctx, tt_module m, const char* kernel_name, tt_function* out);

/* ---- memory (driver.hpp:179-217) --------------------------------------------- */
tt_status tt_mem_alloc(tt_ctx* ctx, uint64_t bytes, tt_devptr* out); /* zero-filled */
tt_status tt_mem_free(tt_ctx* ctx, tt_devptr p);
tt_status tt_memcpy_htod(tt_ctx* ctx, tt_devptr dst, const void* src, uint64_t bytes);
tt_status tt_memcpy_dtoh(tt_ctx* ctx, void* dst, tt_devptr src, uint64_t bytes);
/* Extension: raw CUDA address of a live allocation (interop; no counter). */
tt_status tt_mem_device_pointer(tt_ctx* ctx, tt_devptr p, void** out);
/* Extension: page-locked host staging (fast H2D/D2H); not counted. */
tt_status tt_host_alloc(uint64_t bytes, void** out);
tt_status tt_host_free(void* p);

/* ---- launch (driver.hpp:221-247) ----------------------------------------------- */
tt_status tt_launch(tt_ctx* ctx, tt_function fn, const tt_grid* cfg, const tt_arg* args, int nargs,
                    tt_trap* trap_out);

/* ---- introspection (driver.hpp:251-266) ------------------------------------------ */
tt_status tt_counters_get(tt_ctx* ctx, tt_counters* out);
/* Counters::to_json (driver.hpp:78-95) as UTF-8 JSON; *needed includes the NUL. */
tt_status tt_counters_json(tt_ctx* ctx, char* buf, size_t cap, size_t* needed);
/* Counters::events (driver.hpp:72-74): one tt_event byte per operation. */
tt_status tt_events(tt_ctx* ctx, uint8_t* buf, size_t cap, size_t* needed);

/* ---- trace-transform helpers (spec DESIGN.md §2) ------------------------------------ */
/* Host tables: ctab/stab[a_total], wtab[8*n] = per r: r, r^2, w3re, w3im,
 * w4re, w4im, w5re, w5im (any may be NULL). */
tt_status tt_make_tables(int n, int a_total, float* ctab, float* stab, float* wtab);
/* Deterministic synthetic images: kind 0 disk-noise, 1 phantom, 2 sparse. */
tt_status tt_synth_image(int kind, uint64_t seed, int n, float* img);
/* Slots (lanes) per line of the fused kernel for side n: 8, 16 or 32 (one
 * warp segment) or 32W (W warps); T0-only (full = 0) launches with n > 1024
 * use 32 -- the reduction schedule the replay oracle mirrors. */
int tt_schedule_slots(int n, int full);
/* Largest n the fused T0..T5 kernel supports. */
int tt_max_full_n(void);

/* In-bounds taps of angles [a0, a0+a_count): per line the exact interval of
 * t whose rotated point passes the spec §2.1 bounds test, found by bisection
 * on the same fp32 expressions the kernels evaluate (the algorithmic work
 * count behind the FLOP roofline). */
uint64_t tt_count_inbounds_taps(int n, int a0, int a_count, const float* ctab, const float* stab);

/* ---- input formats (the caller side of the path) ------------------------------
 * A photograph is h x w pixels of 1 (gray) or 3 (RGB) 8-bit channels; the
 * transform wants an n x n f32 image whose inscribed disk holds the whole
 * picture, so no rotation loses mass.  tt_prep_side gives that n (the smallest
 * n with (n-1)^2 >= h^2 + w^2, i.e. the picture's diagonal fits the disk of
 * radius (n-1)/2 around the centre o); tt_prep_device converts and pads on the
 * GPU: gray = ((0.299 r + 0.587 g) + 0.114 b) / 255 in f32 (RGB) or v / 255
 * (gray), placed with its top-left corner at ((n-w)/2, (n-h)/2), zeros
 * elsewhere.  The PNM reader/writer handle binary P5 (gray) / P6 (RGB) 8-bit
 * files. */
int tt_prep_side(int h, int w);
tt_status tt_prep_device(const uint8_t* d_pix, int h, int w, int channels, int n, float* d_img, void* stream);
/* *h = *w = *channels = 0 on entry returns the header only (pix may be NULL). */
tt_status tt_pnm_read(const char* path, int* h, int* w, int* channels, uint8_t* pix, size_t cap);
tt_status tt_pgm_write(const char* path, const float* img, int h, int w, float lo, float hi);

/* FP32 roofline probe: enqueue blocks x 256 threads x iters x 128 FFMA on
 * `stream` (2 flop each); out needs `blocks` floats of device memory. */
tt_status tt_ffma_probe(float* d_out, int blocks, int iters, void* stream);
/* Texture-gather roofline probe: blocks x 256 threads x iters x 8 TLD4 gathers
 * (one lane-gather each) on an L1-resident texture; out needs `blocks` uints. */
tt_status tt_tld4_probe(unsigned* d_out, int blocks, int iters, void* stream);

/* Raw device-pointer entry (multi-GPU driver, benchmarks): enqueue the fused
 * kernel for a_count angles on `stream` (cudaStream_t; NULL = legacy
 * default).  out: full ? [a_count][6][n] : [a_count][n]; med may be NULL.
 * sampler: 0 = global/L1 loads, 1 = texture gather through a cudaArray copy of
 * img that this call makes, 2 = TMA-staged shared-memory tiles read straight
 * from img (T0 only, 704 < n with a 32-lane schedule, n % 4 == 0, batch 1, img 16-B aligned; other
 * launches fall back to 1); all are asynchronous (the call only enqueues):
 * the copy is released once its launch has completed (recorded event, reclaimed
 * by later calls and at exit).  Repeated texture launches on one image should
 * use tt_image_tex_create + tt_trace_device_tex (one copy for all of them);
 * that is what the plans and the multi-GPU driver do.
 * pair_stride: 0 = the drop-in rule (angles [a0, a0+a_count); pairs
 * (a0+i, a0+i+a_count/2) when a_count is even); -1 = no pairing; > 0 = the
 * angles are a0+i and a0+i+pair_stride for i < a_count/2 (rows i and
 * a_count/2+i) — an orientation shard together with its mirror half. */
typedef struct tt_trace_desc {
    const float* img;
    int32_t n;
    int32_t a0;
    int32_t a_count;
    int32_t full;
    const float* ctab;
    const float* stab;
    const float* wtab;
    float* out;
    int32_t* med;
    int32_t sampler;
    int32_t pair_stride;
    int32_t batch;      /* images (0 or 1: one); image b at img + b*img_stride, outputs
                           at out + b*rows*F*n and med + b*rows*2*n (rows = a_count) */
    int32_t _pad2;
    int64_t img_stride; /* elements between images (0: n*n) */
    const float* wsoa;  /* optional pass-2 weight layout of wtab (tt_weights_soa, 24n bytes,
                           16-B aligned); NULL: converted into stream-ordered scratch per call */
    int32_t partner_row; /* paired launches: first out/med row of the partner angles relative to
                            out/med (<= 0: a_count/2, i.e. rows [cnt] + [cnt]).  An orientation
                            shard writing straight into the full [A][F][n] sinogram passes
                            out + a0 rows and partner_row = A/2 (batch 1). */
    int32_t flags;       /* TT_TRACE_PEER_OUT: out/med are another GPU's memory (IPC / NVLink):
                            each thread fences its stores at system scope before it exits.
                            TT_TRACE_FUSED_P (texture sampler): circ is computed inside the trace
                            launch (appended P-CTAs; measured slower) */
    float* circ;         /* optional (full only): circ[row][6][3] = tt_circus_device over the launch's
                            sinogram rows (bit-identical): a separate circus launch after the trace
                            kernel on the same stream, or with TT_TRACE_FUSED_P the P stage fused
                            into the trace launch; NULL: none */
} tt_trace_desc;
#define TT_TRACE_PEER_OUT 1
#define TT_TRACE_FUSED_P 2
tt_status tt_trace_device(const tt_trace_desc* d, void* stream);

/* Regroup a [n][8] weight table (tt_make_tables) on device into the fused
 * kernel's pass-2 layout: [n] x (w3re, w3im, w4re, w4im) then [n] x (w5re,
 * w5im) -- 24n bytes at d_wsoa.  Pass the result as tt_trace_desc.wsoa to
 * reuse it across launches. */
tt_status tt_weights_soa(const float* d_wtab, int n, float* d_wsoa, void* stream);

/* Inter-process device pointers (CUDA IPC; over NVLink / NVSwitch between the
 * GPUs of one node, or between processes on one GPU).  The multi-GPU driver
 * hands rank 0's sinogram buffers to every rank, whose fused kernel then
 * writes its orientation shard's rows straight into them (the gather is the
 * kernel's own stores; the multi-GPU driver exports
 * tt_ipc_alloc buffers).  Export works for any pointer inside
 * a cudaMalloc allocation (the handle carries the offset). */
typedef struct tt_ipc_handle {
    uint8_t bytes[64];
    uint64_t offset;
} tt_ipc_handle;
tt_status tt_ipc_export(const void* d_ptr, tt_ipc_handle* out);
tt_status tt_ipc_import(const tt_ipc_handle* h, int device, void** d_ptr);
tt_status tt_ipc_close(void* d_ptr);
/* A dedicated device allocation for exporting (one cudaMalloc per buffer on
 * `device`): its IPC handle does not depend on any caching allocator's block
 * layout (e.g. PyTorch's expandable segments).  Freed by tt_ipc_free after
 * every importer has closed it. */
tt_status tt_ipc_alloc(int device, size_t bytes, void** d_ptr);
tt_status tt_ipc_free(void* d_ptr);

/* P-functionals (circus features) of `rows` sinogram rows of
 * length n on device: circ[row][3] = (total variation, value at the weighted
 * median, max).  For a trace output [a][6][n], rows = 6a. */
tt_status tt_circus_device(const float* d_sino, int n, int rows, float* d_circ, void* stream);

/* Spectral P-functional (the optional |FFT|^4 functional of the
 * paper's circus stage) of `rows` sinogram rows of length n (1 <= n <= 16384) on
 * device: d_p[row] = sum_k |F(s)_k|^4 (double: the 4th powers of T1/T2 rows exceed
 * the f32 range), F the length-n DFT of the row.  fp32 FFT (power-of-two n) or
 * direct DFT, f64 accumulation of the powers; rtol 1e-4
 * against an f64 FFT.  No reference interface exists for it (the reference has
 * no trace-transform code); it sits beside tt_circus_device. */
tt_status tt_circus_fft_device(const float* d_sino, int n, int rows, double* d_p, void* stream);

/* Hermite P-functionals (the Hermite circus functionals of
 * the cited prior work, PAPER.md:813,817 -- no reference interface exists):
 * for each of `rows` sinogram rows of length n, with centre c = the row's
 * weighted median index (the P2 index of tt_circus_device, bit-identical),
 * d_hp[row][k] = sum_p s_p psi_k(z_p) for k < orders (1..8), psi_k the
 * normalised Hermite functions and z_p = (p-c)*10/c below the centre,
 * (p-c)*10/(n-1-c) above it; f64.  d_center[row] = c (may be NULL). */
tt_status tt_hermite_device(const float* d_sino, int n, int rows, int orders, double* d_hp, int32_t* d_center,
                            void* stream);
/* Orthonormal (square) sinogram input: the h x w image on
 * device resampled bilinearly to s x s, s = tt_orthonormal_side(angles) =
 * ceil(angles / sqrt 2), and centred in an angles x angles frame (d_out), so
 * that the trace transform of d_out over `angles` orientations is square
 * (angles lines per orientation). */
int tt_orthonormal_side(int angles);
tt_status tt_orthonormal_device(const float* d_img, int h, int w, int angles, float* d_out, void* stream);

/* Prepared texture for repeated tt_trace_device calls on one image
 * (sampler 1 without the per-call copy). */
typedef struct tt_image_tex tt_image_tex;
tt_status tt_image_tex_create(const float* d_img, int n, void* stream, tt_image_tex** out);
/* Texture atlas of a batch of n x n images (image b at d_imgs + b*img_stride)
 * for batched tt_trace_device_tex calls (batched feature extraction). */
tt_status tt_image_atlas_create(const float* d_imgs, int n, int batch, int64_t img_stride, void* stream,
                                tt_image_tex** out);
/* Re-copy the image(s) into an existing texture/atlas (stream-ordered). */
tt_status tt_image_tex_update(tt_image_tex* t, const float* d_imgs, int64_t img_stride, void* stream);
tt_status tt_image_tex_destroy(tt_image_tex* t);
tt_status tt_trace_device_tex(const tt_trace_desc* d, const tt_image_tex* t, void* stream);

/* VPTX JIT (kernels without a native implementation are compiled from their
 * VPTX bodies at tt_get_function: VPTX -> CUDA C++ -> NVRTC -> sm_100a).  This
 * returns the generated CUDA C++ for `kernel` without compiling (diagnostics). */
tt_status tt_jit_source(const char* vptx, size_t len, const char* kernel, char* buf, size_t cap, size_t* needed);
/* Fingerprint of a kernel body (FNV-1a over its token stream).  A module whose
 * kernel has a body binds to a native kernel of the same signature only when
 * this fingerprint is one the native kernel is registered for (trace_t05: the
 * reference front end's compilation of the documented DSL trace kernel);
 * any other body is compiled and run as written. */
tt_status tt_vptx_body_fingerprint(const char* vptx, size_t len, const char* kernel, uint64_t* out);

/* ---- plans: the host-to-host form of the path -------------------------------
 * One plan = one (n, angles, functionals, batch) configuration with its device
 * tables, image texture and output buffers resident.  tt_plan_run uploads the
 * image, runs the fused kernel in `chunks` angle chunks over two compute
 * streams while a copy stream downloads each finished chunk's rows (overlapped
 * D2H), runs the P-functional stage once over the sinogram, and returns when
 * every requested host buffer is filled.  Batched plans chunk by images
 * instead: chunk c uploads while chunk c-1 computes (trace + features) and
 * chunk c-2 downloads.  Results equal one whole launch
 * bit-for-bit.  Host buffers should be pinned (tt_host_alloc) for the copies to
 * overlap.  The caller-side flow this replaces is cuda_launch's
 * marshal -> launch -> download sequence (autolaunch.hpp:167-245) repeated per
 * image; counters (bytes_h2d / bytes_d2h / gpu_kernel_launches) are updated. */
typedef struct tt_plan tt_plan;
typedef struct tt_plan_desc {
    int32_t n;        /* image side (= line length = lines per angle) */
    int32_t a_total;  /* angle grid: theta_a = 2 pi a / a_total (tt_make_tables) */
    int32_t a0;       /* first angle of this plan */
    int32_t a_count;  /* angles a0 .. a0 + a_count - 1 */
    int32_t full;     /* 1: T0..T5 (+ medians), 0: T0 (Radon) only */
    int32_t features; /* 1: P-functionals (circus) after the trace (full only) */
    int32_t batch;    /* images per run (0 or 1: one) */
    int32_t chunks;   /* pipeline chunks: angle chunks (one image) or image chunks (batch);
                         0 = automatic */
    int32_t slots;    /* device buffer sets for overlapping submissions (1..4; 0: 2 for one
                         image, 1 for batches) */
    int32_t pair_stride; /* 0: the drop-in pairing over [a0, a0+a_count) (tt_trace_desc rule);
                            > 0: an orientation shard with its mirror half -- a_count even, the
                            angles a0+i and a0+i+pair_stride for i < a_count/2, output rows
                            [a_count/2] + [a_count/2] (shard.orientation_shard: pair_stride = A/2) */
    int32_t graph;       /* 1: capture each slot's submission into a CUDA graph (per set of host
                            buffers) and replay it -- one host call per submit (the latency path for
                            small images, C1); 0: enqueue the calls every time */
} tt_plan_desc;
tt_status tt_plan_create(tt_ctx* ctx, const tt_plan_desc* d, tt_plan** out);
/* h_img [batch][n][n]; h_out [batch][a_count][F][n], h_med [batch][a_count][2][n],
 * h_circ [batch][a_count][6][3] -- each output may be NULL (not downloaded). */
tt_status tt_plan_run(tt_plan* p, const float* h_img, float* h_out, int32_t* h_med, float* h_circ);
/* Asynchronous form: submit enqueues one image (or batch) on the plan's next buffer slot and
 * returns; its host buffers must stay valid until tt_plan_wait, which drains every submission.
 * With two slots consecutive submissions overlap (the next upload with the current kernels,
 * the current downloads with the next kernels).  tt_plan_run = submit + wait. */
tt_status tt_plan_submit(tt_plan* p, const float* h_img, float* h_out, int32_t* h_med, float* h_circ);
tt_status tt_plan_wait(tt_plan* p);
tt_status tt_plan_chunks(const tt_plan* p, int* chunks);
/* Graph mode: submissions captured so far (one per slot and host-buffer set; the rest replayed). */
tt_status tt_plan_captures(const tt_plan* p, int* captures);
tt_status tt_plan_destroy(tt_plan* p);

#ifdef __cplusplus
}
#endif
#endif
