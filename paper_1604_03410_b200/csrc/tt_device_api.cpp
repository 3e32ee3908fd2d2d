// tt_device_api.cpp — the raw device-pointer entries of the C ABI
// (tt_trace_device, textures, weight layouts, probes), the pipelined
// host-to-host plans (tt_plan_*) and the inter-process pointers (tt_ipc_*).
// Shares the context internals of tt_context_impl.h.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <array>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include "tt_context_impl.h"

using namespace ttc;

namespace {

// Texture copies made by tt_trace_device (sampler 1) for one launch: released once the launch has
// completed (its event), by later calls or at exit -- the call itself never blocks the host.
struct DeferredTex {
    cudaArray_t arr = nullptr;
    cudaTextureObject_t tex = 0;
    cudaEvent_t done = nullptr;
    int device = 0;
};
std::mutex g_tex_mu;
std::vector<DeferredTex> g_tex_pending;

void release(const DeferredTex& t) {
    DeviceGuard guard(t.device);
    cudaDestroyTextureObject(t.tex);
    if (t.arr) cudaFreeArray(t.arr);
    cudaEventDestroy(t.done);
}

void reclaim_textures(bool all) {
    std::lock_guard<std::mutex> lk(g_tex_mu);
    auto it = g_tex_pending.begin();
    while (it != g_tex_pending.end()) {
        if (all) cudaEventSynchronize(it->done);
        if (all || cudaEventQuery(it->done) == cudaSuccess) {
            release(*it);
            it = g_tex_pending.erase(it);
        } else {
            ++it;
        }
    }
}

struct TexReaper {
    ~TexReaper() { reclaim_textures(true); }
} g_tex_reaper;

// NVTX range (nvtx3, header-only: a no-op unless a profiler injects itself).
struct Range {
    explicit Range(const char* name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
};

}  // namespace

extern "C" {

// ---- trace-transform helpers -------------------------------------------------

int tt_schedule_slots(int n, int full) { return tt::schedule_slots(n, full != 0); }

tt_status tt_ffma_probe(float* d_out, int blocks, int iters, void* stream) {
    if (!d_out || blocks < 1 || iters < 1) return fail(nullptr, TT_ERR_INVALID, "bad probe arguments");
    cudaError_t e = tt::launch_ffma_probe(d_out, blocks, iters, (cudaStream_t)stream);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "ffma probe");
}
tt_status tt_tld4_probe(unsigned* d_out, int blocks, int iters, void* stream) {
    if (!d_out || blocks < 1 || iters < 1) return fail(nullptr, TT_ERR_INVALID, "bad probe arguments");
    cudaError_t e = tt::launch_tld4_probe(d_out, blocks, iters, (cudaStream_t)stream);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "tld4 probe");
}
int tt_max_full_n(void) { return tt::max_full_n(); }

static tt_status check_desc(const tt_trace_desc* d) {
    if (!d) return fail(nullptr, TT_ERR_INVALID, "null descriptor");
    if (d->n < 1 || d->n > (d->full ? tt::max_full_n() : 32768))
        return fail(nullptr, TT_ERR_LAUNCH_CONFIG, "LaunchConfigError: n out of range for the native kernel");
    if (d->a_count < 0 || d->a0 < 0) return fail(nullptr, TT_ERR_INVALID, "negative angle range");
    if (d->pair_stride > 0 && d->a_count % 2 != 0)
        return fail(nullptr, TT_ERR_INVALID, "explicit pair_stride needs an even a_count");
    if (d->partner_row > 0 && d->batch > 1)
        return fail(nullptr, TT_ERR_INVALID, "partner_row applies to single-image launches");
    if ((long long)d->a_count * d->n >= (1ll << 31)) return fail(nullptr, TT_ERR_INVALID, "launch too large");
    if (d->batch < 0 || d->img_stride < 0) return fail(nullptr, TT_ERR_INVALID, "negative batch or stride");
    if (d->img_stride != 0 && d->img_stride < (long long)d->n * d->n)
        return fail(nullptr, TT_ERR_INVALID, "img_stride smaller than one image");
    if (!d->ctab || !d->stab || !d->out || (d->full && !d->wtab))
        return fail(nullptr, TT_ERR_INVALID, "null table or output pointer");
    if (d->full && ((reinterpret_cast<std::uintptr_t>(d->wtab) | reinterpret_cast<std::uintptr_t>(d->wsoa)) & 15u))
        return fail(nullptr, TT_ERR_INVALID, "wtab / wsoa must be 16-byte aligned");
    return TT_OK;
}

static tt::TraceArgs to_args(const tt_trace_desc* d) {
    tt::TraceArgs ta;
    ta.img = d->img;
    ta.n = d->n;
    ta.a0 = d->a0;
    if (d->pair_stride == 0) {
        tt::launch_structure(d->a_count, &ta.a_count, &ta.pair_stride);
    } else if (d->pair_stride > 0 && d->a_count % 2 == 0) {
        ta.a_count = d->a_count / 2;
        ta.pair_stride = d->pair_stride;
    } else {
        ta.a_count = d->a_count;
        ta.pair_stride = 0;
    }
    ta.ctab = d->ctab;
    ta.stab = d->stab;
    ta.wtab = d->wtab;
    ta.wsoa = d->wsoa;
    if (d->partner_row > 0 && ta.pair_stride > 0) ta.partner_row = d->partner_row;
    ta.peer_out = (d->flags & TT_TRACE_PEER_OUT) != 0;
    ta.out = d->out;
    ta.med = d->med;
    ta.full = d->full != 0;
    ta.batch = d->batch > 1 ? d->batch : 1;
    ta.img_stride = d->img_stride;
    ta.circ = d->full ? d->circ : nullptr;
    ta.fuse_circus = (d->flags & TT_TRACE_FUSED_P) != 0;
    return ta;
}

// Stream-ordered scratch of the raw entries comes from the device's default pool; keep freed blocks in
// it (once per device) so a steady stream of calls never returns memory to the driver and re-maps it
// inside the caller's stream (measured: +0.2..3 ms per call at C2 with the default threshold of 0).
void keep_default_pool() {
    static std::atomic<int> done[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || done[dev & 63].load(std::memory_order_acquire)) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        std::uint64_t thresh = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh);
    }
    done[dev & 63].store(1, std::memory_order_release);
}

// Raw-pointer launches without a prepared weight layout convert wtab into
// stream-ordered scratch around the launch (one extra small kernel).
struct WeightScratch {
    float* d = nullptr;
    cudaStream_t s = nullptr;
    ~WeightScratch() {
        if (d) cudaFreeAsync(d, s);
    }
    cudaError_t prepare(tt::TraceArgs& ta, cudaStream_t stream) {
        if (!ta.full || ta.wsoa) return cudaSuccess;
        keep_default_pool();
        s = stream;
        cudaError_t e = cudaMallocAsync((void**)&d, tt::weights_soa_bytes(ta.n), stream);
        if (e != cudaSuccess) return e;
        ta.wsoa = d;
        return tt::launch_weights_soa(ta.wtab, ta.n, d, stream);
    }
};

// State of the fused P stage for one raw launch (stream-ordered scratch).
struct CounterScratch {
    int* d = nullptr;
    cudaStream_t s = nullptr;
    ~CounterScratch() {
        if (d) cudaFreeAsync(d, s);
    }
    cudaError_t prepare(tt::TraceArgs& ta, cudaStream_t stream) {
        if (!ta.circ || !ta.fuse_circus) return cudaSuccess;
        keep_default_pool();
        s = stream;
        const std::size_t bytes = tt::epi_state_ints(ta) * sizeof(int);
        cudaError_t e = cudaMallocAsync((void**)&d, bytes, stream);
        if (e != cudaSuccess) return e;
        ta.epi = d;
        return cudaMemsetAsync(d, 0, bytes, stream);
    }
};

tt_status tt_weights_soa(const float* d_wtab, int n, float* d_wsoa, void* stream) {
    if (!d_wtab || !d_wsoa || n < 1) return fail(nullptr, TT_ERR_INVALID, "bad weight-table arguments");
    if ((reinterpret_cast<std::uintptr_t>(d_wtab) | reinterpret_cast<std::uintptr_t>(d_wsoa)) & 15u)
        return fail(nullptr, TT_ERR_INVALID, "weight tables must be 16-byte aligned");
    cudaError_t e = tt::launch_weights_soa(d_wtab, n, d_wsoa, (cudaStream_t)stream);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "weight table");
}

tt_status tt_trace_device(const tt_trace_desc* d, void* stream) {
    Range r("tt_trace_device");
    tt_status st = check_desc(d);
    if (st != TT_OK) return st;
    if (!d->img) return fail(nullptr, TT_ERR_INVALID, "null image");
    tt::TraceArgs ta = to_args(d);
    cudaStream_t s = (cudaStream_t)stream;
    WeightScratch ws;
    if (cudaError_t e = ws.prepare(ta, s); e != cudaSuccess) return cuda_fail(nullptr, e, "weight table");
    CounterScratch cs;
    if (cudaError_t e = cs.prepare(ta, s); e != cudaSuccess) return cuda_fail(nullptr, e, "circus counters");
    if (d->sampler == 2) {  // TMA-staged tiles straight from img (T0); other launches: the texture copy below
        ta.sampler = tt::Sampler::Tma;
        if (tt::tma_radon_ok(ta)) {
            cudaError_t e = tt::launch_trace(ta, s);
            return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "trace kernel");
        }
    }
    if (d->sampler == 1 || d->sampler == 2) {
        reclaim_textures(false);  // copies of earlier calls whose launches have completed
        DeferredTex t;
        cudaGetDevice(&t.device);
        ta.sampler = tt::Sampler::Texture;
        cudaError_t e = ta.batch > 1
                            ? tt::make_image_atlas(ta.img, ta.n, ta.batch, ta.img_stride > 0 ? ta.img_stride
                                                                                           : (long long)ta.n * ta.n,
                                                   s, &t.arr, &ta.tex, &ta.atlas_cols)
                            : tt::make_image_texture(ta.img, ta.n, s, &t.arr, &ta.tex);
        t.tex = ta.tex;
        if (e == cudaSuccess) e = tt::launch_trace(ta, s);
        const cudaError_t ev = cudaEventCreateWithFlags(&t.done, cudaEventDisableTiming);
        if (ev == cudaSuccess && cudaEventRecord(t.done, s) == cudaSuccess) {
            std::lock_guard<std::mutex> lk(g_tex_mu);
            g_tex_pending.push_back(t);  // released once the launch has completed
        } else {  // no event: fall back to waiting here
            cudaStreamSynchronize(s);
            if (t.tex) cudaDestroyTextureObject(t.tex);
            if (t.arr) cudaFreeArray(t.arr);
            if (t.done) cudaEventDestroy(t.done);
        }
        return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "trace kernel");
    }
    cudaError_t e = tt::launch_trace(ta, s);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "trace kernel");
}

}  // extern "C"

struct tt_image_tex {
    cudaArray_t arr = nullptr;  // null: pitch-linear views of images (small n), one per image pointer seen
    cudaTextureObject_t tex = 0;
    int n = 0;
    int batch = 1;
    int cols = 1;
    std::vector<std::pair<const float*, cudaTextureObject_t>> views;  // (image, view); tex is one of them
};

extern "C" {

tt_status tt_circus_device(const float* d_sino, int n, int rows, float* d_circ, void* stream) {
    if (!d_sino || !d_circ || n < 1 || rows < 0) return fail(nullptr, TT_ERR_INVALID, "bad circus arguments");
    cudaError_t e = tt::launch_circus(d_sino, n, rows, d_circ, (cudaStream_t)stream);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "circus");
}

tt_status tt_circus_fft_device(const float* d_sino, int n, int rows, double* d_p, void* stream) {
    if (!d_sino || !d_p || n < 1 || n > tt::max_circus_fft_n() || rows < 0)
        return fail(nullptr, TT_ERR_INVALID, "bad circus_fft arguments");
    cudaError_t e = tt::launch_circus_fft(d_sino, n, rows, d_p, (cudaStream_t)stream);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "circus_fft");
}

tt_status tt_hermite_device(const float* d_sino, int n, int rows, int orders, double* d_hp, int32_t* d_center,
                            void* stream) {
    if (!d_sino || !d_hp || n < 1 || rows < 0 || orders < 1 || orders > tt::max_hermite_orders())
        return fail(nullptr, TT_ERR_INVALID, "bad hermite arguments");
    cudaError_t e = tt::launch_hermite(d_sino, n, rows, orders, d_hp, d_center, (cudaStream_t)stream);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "hermite");
}

int tt_orthonormal_side(int angles) { return tt::orthonormal_side(angles); }

tt_status tt_orthonormal_device(const float* d_img, int h, int w, int angles, float* d_out, void* stream) {
    if (!d_img || !d_out || h < 1 || w < 1 || angles < 2) return fail(nullptr, TT_ERR_INVALID, "bad orthonormal arguments");
    cudaError_t e = tt::launch_orthonormal(d_img, h, w, angles, d_out, (cudaStream_t)stream);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "orthonormal");
}

tt_status tt_image_tex_create(const float* d_img, int n, void* stream, tt_image_tex** out) {
    if (!d_img || !out || n < 1) return fail(nullptr, TT_ERR_INVALID, "bad argument");
    auto t = std::make_unique<tt_image_tex>();
    t->n = n;
    cudaError_t e = tt::make_image_texture(d_img, n, (cudaStream_t)stream, &t->arr, &t->tex);
    if (e != cudaSuccess) {
        if (t->arr) cudaFreeArray(t->arr);
        return cuda_fail(nullptr, e, "make_image_texture");
    }
    if (!t->arr) t->views.emplace_back(d_img, t->tex);
    *out = t.release();
    return TT_OK;
}

tt_status tt_image_atlas_create(const float* d_imgs, int n, int batch, std::int64_t img_stride, void* stream,
                                tt_image_tex** out) {
    if (!d_imgs || !out || n < 1 || batch < 1) return fail(nullptr, TT_ERR_INVALID, "bad argument");
    auto t = std::make_unique<tt_image_tex>();
    t->n = n;
    t->batch = batch;
    cudaError_t e = tt::make_image_atlas(d_imgs, n, batch, img_stride > 0 ? img_stride : (long long)n * n,
                                         (cudaStream_t)stream, &t->arr, &t->tex, &t->cols);
    if (e != cudaSuccess) {
        if (t->arr) cudaFreeArray(t->arr);
        return cuda_fail(nullptr, e, "make_image_atlas (batch too large for one 2-D texture?)");
    }
    *out = t.release();
    return TT_OK;
}

tt_status tt_image_tex_update(tt_image_tex* t, const float* d_imgs, std::int64_t img_stride, void* stream) {
    if (!t || !d_imgs) return fail(nullptr, TT_ERR_INVALID, "bad argument");
    const long long stride = img_stride > 0 ? img_stride : (long long)t->n * t->n;
    cudaError_t e;
    if (!t->arr) {  // a view: launches read the image itself; another image gets (or reuses) its own view
        for (const auto& v : t->views)
            if (v.first == d_imgs) {
                t->tex = v.second;
                return TT_OK;
            }
        cudaArray_t arr = nullptr;
        cudaTextureObject_t tex = 0;
        e = tt::make_image_texture(d_imgs, t->n, (cudaStream_t)stream, &arr, &tex);  // a view, or an array copy
        if (e != cudaSuccess) {                                                     // of an unaligned image
            if (arr) cudaFreeArray(arr);
            return cuda_fail(nullptr, e, "image texture view");
        }
        if (arr) {
            t->arr = arr;  // from now on an array-backed handle (later updates copy into it)
        } else {
            t->views.emplace_back(d_imgs, tex);  // kept until destroy: earlier launches may still use the others
        }
        t->tex = tex;
        return TT_OK;
    }
    if (t->batch == 1 && t->cols == 1)
        e = cudaMemcpy2DToArrayAsync(t->arr, 0, 0, d_imgs, std::size_t(t->n) * 4, std::size_t(t->n) * 4,
                                     std::size_t(t->n), cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
    else
        e = tt::fill_image_atlas(t->arr, d_imgs, t->n, t->batch, stride, t->cols, (cudaStream_t)stream);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "image texture update");
}

tt_status tt_image_tex_destroy(tt_image_tex* t) {
    if (!t) return TT_OK;
    bool tex_is_view = false;
    for (const auto& v : t->views) {
        cudaDestroyTextureObject(v.second);
        tex_is_view |= v.second == t->tex;
    }
    if (!tex_is_view) cudaDestroyTextureObject(t->tex);
    if (t->arr) cudaFreeArray(t->arr);
    delete t;
    return TT_OK;
}

tt_status tt_trace_device_tex(const tt_trace_desc* d, const tt_image_tex* t, void* stream) {
    Range r("tt_trace_device_tex");
    tt_status st = check_desc(d);
    if (st != TT_OK) return st;
    if (!t || t->n != d->n) return fail(nullptr, TT_ERR_INVALID, "texture does not match n");
    tt::TraceArgs ta = to_args(d);
    if (ta.batch > t->batch) return fail(nullptr, TT_ERR_INVALID, "batch larger than the texture atlas");
    ta.sampler = tt::Sampler::Texture;
    ta.tex = t->tex;
    ta.atlas_cols = t->cols;
    WeightScratch ws;
    if (cudaError_t e = ws.prepare(ta, (cudaStream_t)stream); e != cudaSuccess)
        return cuda_fail(nullptr, e, "weight table");
    CounterScratch cs;
    if (cudaError_t e = cs.prepare(ta, (cudaStream_t)stream); e != cudaSuccess)
        return cuda_fail(nullptr, e, "circus counters");
    cudaError_t e = tt::launch_trace(ta, (cudaStream_t)stream);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "trace kernel");
}

}  // extern "C"

// ----------------------------------------------------------------- plans
//
// A plan is the host-to-host form of the path (include/tt_b200.h
// tt_plan_*): the device tables live for the plan's lifetime and each of
// its `slots` owns an image texture and output buffers.  tt_plan_submit
// enqueues one image (or batch) on the next slot and returns; tt_plan_wait
// drains everything submitted; tt_plan_run = submit + wait.  One image: the
// fused kernel runs in angle chunks alternating over two compute streams
// while a copy stream downloads each finished chunk's sinogram and median
// rows; the P-functional stage runs once over the sinogram.  With two slots
// the next submission's upload overlaps the current kernels and the current
// downloads overlap the next kernels.  The chunked launches write exactly
// the rows of one whole launch (a chunk is the unit range [u0, u1) plus its
// mirror rows at partner_row = U), so outputs are bit-identical to the
// single-launch path.  Batched plans chunk by images (upload / atlas fill +
// trace + features / download on three streams).

struct PlanSlot {
    float* img = nullptr;  // linear image(s) (LDG sampler, batched atlas fill)
    float *out = nullptr, *circ = nullptr;
    std::int32_t* med = nullptr;
    cudaArray_t arr = nullptr;
    cudaTextureObject_t tex = 0;
    std::vector<cudaEvent_t> done;      // per chunk: its rows are final
    std::vector<cudaEvent_t> uploaded;  // per chunk (batched plans): its images are on the device
    cudaEvent_t ready = nullptr;        // image uploaded (single-image plans)
    cudaEvent_t free = nullptr;         // the slot's last download finished: buffers reusable
    bool used = false;
    int* epi[2] = {nullptr, nullptr};   // fused P stage state per compute stream (zeroed, self-resetting)
    cudaSurfaceObject_t surf = 0;       // batched texture plans: the atlas as a surface (created once)
    // graph mode: the slot's submission captured once per set of host buffers and replayed on the
    // slot's own launch stream (the two slots' graphs overlap like the enqueued submissions do)
    cudaStream_t gs = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t join = nullptr;         // capture: the copy stream joins back into the origin
    std::array<const void*, 4> key{};   // host buffers the captured graph reads / writes
    std::uint64_t g_h2d = 0, g_d2h = 0, g_launches = 0;
};

struct tt_plan {
    tt_ctx* ctx = nullptr;
    tt_plan_desc d{};
    int F = 1, units = 0, pair = 0, chunks = 1, cols = 1, next = 0;
    bool fused_circus = false;  // TT_FUSED_CIRCUS=1: the P stage inside each trace launch (measured slower)
    int captures = 0;           // graph mode: submissions captured (the rest replayed)
    float *ctab = nullptr, *stab = nullptr, *wtab = nullptr, *wsoa = nullptr;
    std::vector<PlanSlot> slot;
    cudaStream_t sc[2] = {nullptr, nullptr}, sx = nullptr, si = nullptr;
};

namespace {

void plan_release(tt_plan* p) {
    if (!p) return;
    DeviceGuard guard(p->ctx->device);
    for (cudaStream_t s : {p->sc[0], p->sc[1], p->sx, p->si})
        if (s) cudaStreamSynchronize(s);
    for (PlanSlot& sl : p->slot) {
        for (auto* evs : {&sl.done, &sl.uploaded})
            for (cudaEvent_t e : *evs)
                if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : {sl.ready, sl.free, sl.join})
            if (e) cudaEventDestroy(e);
        if (sl.exec) cudaGraphExecDestroy(sl.exec);
        if (sl.surf) cudaDestroySurfaceObject(sl.surf);
        if (sl.gs) {
            cudaStreamSynchronize(sl.gs);
            cudaStreamDestroy(sl.gs);
        }
        for (int* b : sl.epi)
            if (b) cudaFree(b);
        if (sl.tex) cudaDestroyTextureObject(sl.tex);
        if (sl.arr) cudaFreeArray(sl.arr);
        for (void* b : {(void*)sl.img, (void*)sl.out, (void*)sl.circ, (void*)sl.med})
            if (b) cudaFree(b);
    }
    for (void* b : {(void*)p->ctab, (void*)p->stab, (void*)p->wtab, (void*)p->wsoa})
        if (b) cudaFree(b);
    for (cudaStream_t s : {p->sc[0], p->sc[1], p->sx, p->si})
        if (s) cudaStreamDestroy(s);
    delete p;
}

}  // namespace

extern "C" {

tt_status tt_plan_create(tt_ctx* ctx, const tt_plan_desc* d, tt_plan** out) {
    if (!ctx || ctx->destroyed || !d || !out) return fail(ctx, TT_ERR_INVALID, "bad plan arguments");
    *out = nullptr;
    const int n = d->n;
    if (n < 1 || n > (d->full ? tt::max_full_n() : 32768))
        return fail(ctx, TT_ERR_LAUNCH_CONFIG, "LaunchConfigError: n out of range for the native kernel");
    if (d->a_total < 1 || d->a0 < 0 || d->a_count < 1 || d->a0 + d->a_count > d->a_total || d->batch < 0 ||
        d->chunks < 0 || d->slots < 0 || d->slots > 4 || (d->features && !d->full))
        return fail(ctx, TT_ERR_INVALID, "bad plan descriptor");
    if ((long long)d->a_count * n * (d->batch > 1 ? d->batch : 1) >= (1ll << 31))
        return fail(ctx, TT_ERR_INVALID, "plan too large");
    if (d->pair_stride < 0 ||
        (d->pair_stride > 0 && (d->a_count % 2 != 0 || d->a0 + d->a_count / 2 + d->pair_stride > d->a_total)))
        return fail(ctx, TT_ERR_INVALID, "explicit pair_stride needs an even a_count inside the angle grid");
    DeviceGuard guard(ctx->device);
    auto p = new tt_plan;
    p->ctx = ctx;
    p->d = *d;
    p->d.batch = d->batch > 1 ? d->batch : 1;
    p->F = d->full ? tt::kNumF : 1;
    if (const char* fc = std::getenv("TT_FUSED_CIRCUS")) p->fused_circus = std::atoi(fc) != 0;
    if (d->pair_stride > 0) {  // orientation shard + mirror half: rows [units] + [units]
        p->units = d->a_count / 2;
        p->pair = d->pair_stride;
    } else {
        tt::launch_structure(d->a_count, &p->units, &p->pair);
    }
    const int B = p->d.batch;
    // chunks: >= ~1.6e7 unit-taps (~40 us of kernel) each so the per-chunk enqueue cost stays hidden,
    // at most 32 (measured on C2: 5 chunks 1.28 ms, 24-32 chunks 1.24 ms; C1 best unchunked)
    int ch = d->chunks;
    // at most 8 for one large image (n >= 2048): its chunks are milliseconds long, the D2H of a chunk's rows
    // hides behind the next chunk either way, and fewer chunk boundaries mean fewer partial waves
    // (C3 e2e 34.68 ms with 32 chunks, 34.18 with 8, graph mode; scripts/plan_chunks_c3.py)
    if (ch == 0) {
        const long long cap = (B == 1 && n >= 2048) ? 8 : 32;
        ch = int(std::max(1LL, std::min(cap, (long long)p->units * B * n * n / 16000000LL)));
    }
    p->chunks = std::max(1, std::min(ch, B > 1 ? B : p->units));  // angle chunks (one image) or image chunks
    const int nslots = d->slots > 0 ? d->slots : (B > 1 ? 1 : 2);
    p->d.slots = nslots;
    p->slot.resize(nslots);
    const std::size_t N2 = std::size_t(n) * n;
    const std::size_t rows = std::size_t(B) * d->a_count;
    cudaError_t e = cudaSuccess;
    auto alloc = [&](auto** ptr, std::size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc((void**)ptr, bytes ? bytes : 4);
    };
    alloc(&p->ctab, std::size_t(d->a_total) * 4);
    alloc(&p->stab, std::size_t(d->a_total) * 4);
    if (d->full) {
        alloc(&p->wtab, std::size_t(n) * 32);
        alloc(&p->wsoa, tt::weights_soa_bytes(n));
    }
    for (cudaStream_t* s : {&p->sc[0], &p->sc[1], &p->sx, &p->si})
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
    tt::TraceArgs big;  // the fused P stage's state, sized for the largest launch: all units of all images
    big.batch = B;
    big.a_count = p->units;
    big.pair_stride = p->pair;
    const std::size_t epi_bytes = tt::epi_state_ints(big) * sizeof(int);
    for (PlanSlot& sl : p->slot) {
        alloc(&sl.img, B * N2 * 4);
        alloc(&sl.out, rows * p->F * n * 4);
        if (d->full) alloc(&sl.med, rows * 2 * n * 4);
        if (d->features) alloc(&sl.circ, rows * tt::kNumF * 3 * 4);
        sl.done.resize(p->chunks, nullptr);
        sl.uploaded.resize(p->chunks, nullptr);
        for (auto* evs : {&sl.done, &sl.uploaded})
            for (auto& ev : *evs)
                if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        for (cudaEvent_t* ev : {&sl.ready, &sl.free, &sl.join})
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
        if (e == cudaSuccess && ctx->sampler != int(tt::Sampler::Global))
            e = B > 1 ? tt::make_image_atlas(sl.img, n, B, (long long)N2, p->sc[0], &sl.arr, &sl.tex, &p->cols)
                      : tt::make_image_texture(sl.img, n, p->sc[0], &sl.arr, &sl.tex);
        if (e == cudaSuccess && B > 1 && sl.arr) {
            cudaResourceDesc rd{};
            rd.resType = cudaResourceTypeArray;
            rd.res.array.array = sl.arr;
            e = cudaCreateSurfaceObject(&sl.surf, &rd);
        }
        if (e == cudaSuccess && d->graph) e = cudaStreamCreateWithFlags(&sl.gs, cudaStreamNonBlocking);
        if (d->features)
            for (int k = 0; k < 2; ++k) {
                alloc(&sl.epi[k], epi_bytes);
                if (e == cudaSuccess) e = cudaMemsetAsync(sl.epi[k], 0, epi_bytes, p->sc[0]);
            }
    }
    if (e != cudaSuccess) {
        plan_release(p);
        return cuda_fail(ctx, e, "plan buffers");
    }
    // tables (host f64 -> f32, spec §2.1-2.2) and the pass-2 weight layout
    std::vector<float> ct(d->a_total), st(d->a_total), wt(d->full ? std::size_t(n) * 8 : 0);
    tt_make_tables(n, d->a_total, ct.data(), st.data(), d->full ? wt.data() : nullptr);
    e = cudaMemcpyAsync(p->ctab, ct.data(), ct.size() * 4, cudaMemcpyHostToDevice, p->sc[0]);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p->stab, st.data(), st.size() * 4, cudaMemcpyHostToDevice, p->sc[0]);
    if (e == cudaSuccess && d->full) {
        e = cudaMemcpyAsync(p->wtab, wt.data(), wt.size() * 4, cudaMemcpyHostToDevice, p->sc[0]);
        if (e == cudaSuccess) e = tt::launch_weights_soa(p->wtab, n, p->wsoa, p->sc[0]);
    }
    if (e == cudaSuccess) {  // set the kernels' launch attributes now (not inside a graph capture later)
        tt::TraceArgs ta;
        ta.n = n;
        ta.a_count = 0;
        ta.full = d->full != 0;
        ta.wsoa = p->wsoa;
        ta.batch = B;
        ta.img0 = B > 1 ? 1 : 0;
        ta.sampler = ctx->sampler != int(tt::Sampler::Global) ? tt::Sampler::Texture : tt::Sampler::Global;
        e = tt::launch_trace(ta, p->sc[0]);
        if (e == cudaSuccess && B > 1) {  // a one-image chunk at the atlas origin uses the plain-texture kernel
            ta.batch = 1;
            ta.img0 = 0;
            e = tt::launch_trace(ta, p->sc[0]);
        }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->sc[0]);
    if (e != cudaSuccess) {
        plan_release(p);
        return cuda_fail(ctx, e, "plan setup");
    }
    *out = p;
    return TT_OK;
}

tt_status tt_plan_submit(tt_plan* p, const float* h_img, float* h_out, std::int32_t* h_med, float* h_circ) {
    Range r("tt_plan_submit");
    if (!p || !h_img) return fail(p ? p->ctx : nullptr, TT_ERR_INVALID, "bad plan run arguments");
    tt_ctx* ctx = p->ctx;
    if (ctx->destroyed) return fail(ctx, TT_ERR_INVALID, "context destroyed");
    DeviceGuard guard(ctx->device);
    const tt_plan_desc& d = p->d;
    const int n = d.n, B = d.batch, F = p->F;
    const std::size_t N2 = std::size_t(n) * n;
    const std::size_t row_f = std::size_t(F) * n, row_m = 2 * std::size_t(n), row_c = std::size_t(tt::kNumF) * 3;
    PlanSlot& sl = p->slot[p->next];
    p->next = (p->next + 1) % int(p->slot.size());
    cudaError_t e = cudaSuccess;
    std::uint64_t h2d = 0, d2h = 0, launches = 0;
    auto ok = [&](cudaError_t x) {
        if (e == cudaSuccess) e = x;
        return e == cudaSuccess;
    };
    const bool tex = ctx->sampler != int(tt::Sampler::Global);  // plans sample through their texture
    // the slot's previous submission must have fully drained (its kernels read the texture,
    // its downloads read the outputs) before this one overwrites them
    const bool graph = d.graph != 0;
    if (sl.used) ok(cudaStreamWaitEvent(graph ? sl.gs : p->si, sl.free, 0));
    sl.used = true;
    // Graph mode (tt_plan_desc.graph): the whole submission below -- upload, chunked launches on two
    // streams, downloads, P stage -- is captured into one CUDA graph per slot and host-buffer set,
    // then replayed with a single cudaGraphLaunch (one host call instead of ~4 + 3 per chunk).
    const std::array<const void*, 4> key{h_img, h_out, h_med, h_circ};
    if (graph && sl.exec && sl.key == key) {
        ok(cudaGraphLaunch(sl.exec, sl.gs));
        ok(cudaEventRecord(sl.free, sl.gs));
        if (e != cudaSuccess) return cuda_fail(ctx, e, "plan graph launch");
        ctx->c.bytes_h2d += sl.g_h2d;
        ctx->c.bytes_d2h += sl.g_d2h;
        ctx->c.gpu_kernel_launches += sl.g_launches;
        return TT_OK;
    }
    if (graph) {
        if (sl.exec) {
            cudaGraphExecDestroy(sl.exec);
            sl.exec = nullptr;
        }
        ok(cudaStreamBeginCapture(p->si, cudaStreamCaptureModeThreadLocal));
    }
    auto trace_args = [&](int u0, int u1, int b0, int b1, int stream_k) {
        tt::TraceArgs ta;
        ta.img = sl.img;
        ta.tex = sl.tex;
        ta.sampler = tex ? tt::Sampler::Texture : tt::Sampler::Global;
        ta.atlas_cols = p->cols;
        ta.n = n;
        ta.a0 = d.a0 + u0;
        ta.a_count = u1 - u0;
        ta.pair_stride = p->pair;
        ta.partner_row = B == 1 ? p->units : -1;  // angle chunks write their mirror rows at U (one image)
        ta.ctab = p->ctab;
        ta.stab = p->stab;
        ta.wtab = p->wtab;
        ta.wsoa = p->wsoa;
        const std::size_t rows0 = std::size_t(b0) * d.a_count + u0;  // first output row of the launch
        ta.out = sl.out + rows0 * row_f;
        ta.med = d.full ? sl.med + rows0 * row_m : nullptr;
        ta.full = d.full != 0;
        ta.batch = b1 - b0;
        ta.img0 = b0;
        if (d.features && p->fused_circus) {  // fused P stage: the rows' circus features
            ta.circ = sl.circ + rows0 * row_c;
            ta.epi = sl.epi[stream_k];  // one state block per slot and compute stream (its launches are ordered)
            ta.fuse_circus = true;
        }
        return ta;
    };
    auto download = [&](std::size_t r0, std::size_t cnt) {  // output rows [r0, r0 + cnt) on the copy stream
        if (h_out) {
            ok(cudaMemcpyAsync(h_out + r0 * row_f, sl.out + r0 * row_f, cnt * row_f * 4, cudaMemcpyDeviceToHost, p->sx));
            d2h += cnt * row_f * 4;
        }
        if (h_med && d.full) {
            ok(cudaMemcpyAsync(h_med + r0 * row_m, sl.med + r0 * row_m, cnt * row_m * 4, cudaMemcpyDeviceToHost, p->sx));
            d2h += cnt * row_m * 4;
        }
    };
    if (B == 1) {
        // 1. image in on the upload stream (straight into the texture array when the sampler reads it)
        if (tex && sl.arr)
            ok(cudaMemcpy2DToArrayAsync(sl.arr, 0, 0, h_img, std::size_t(n) * 4, std::size_t(n) * 4, std::size_t(n),
                                        cudaMemcpyHostToDevice, p->si));
        else
            ok(cudaMemcpyAsync(sl.img, h_img, N2 * 4, cudaMemcpyHostToDevice, p->si));
        h2d += N2 * 4;
        ok(cudaEventRecord(sl.ready, p->si));
        ok(cudaStreamWaitEvent(p->sc[0], sl.ready, 0));
        ok(cudaStreamWaitEvent(p->sc[1], sl.ready, 0));
        // 2. angle chunks alternating over two compute streams; each finished chunk's forward and
        //    mirror rows go out on the copy stream while later chunks compute
        for (int c = 0; c < p->chunks && e == cudaSuccess; ++c) {
            const int u0 = int((long long)p->units * c / p->chunks), u1 = int((long long)p->units * (c + 1) / p->chunks);
            cudaStream_t s = p->sc[c & 1];
            tt::TraceArgs ta = trace_args(u0, u1, 0, 1, c & 1);
            if (!ok(tt::launch_trace(ta, s))) break;
            launches += tt::trace_launch_count(ta);
            ok(cudaEventRecord(sl.done[c], s));
            ok(cudaStreamWaitEvent(p->sx, sl.done[c], 0));
            if (h_out || h_med)
                for (int half = 0; half < (p->pair ? 2 : 1); ++half) download(std::size_t(u0 + half * p->units), u1 - u0);
        }
        if (d.features) {  // 3. P-functionals over the whole sinogram (fused: computed by the trace launches)
            const std::size_t rows = d.a_count;
            if (!p->fused_circus) {
                ok(tt::launch_circus(sl.out, n, int(rows * tt::kNumF), sl.circ, p->sx));
                ++launches;
            }
            if (h_circ) {
                ok(cudaMemcpyAsync(h_circ, sl.circ, rows * row_c * 4, cudaMemcpyDeviceToHost, p->sx));
                d2h += rows * row_c * 4;
            }
        }
    } else {
        // Image chunks: chunk c's upload (upload stream) overlaps chunk c-1's atlas fill + trace +
        // features (compute stream) and chunk c-2's download (copy stream).
        const int units_all = d.a_count;  // rows per image
        for (int c = 0; c < p->chunks && e == cudaSuccess; ++c) {
            const int b0 = int((long long)B * c / p->chunks), b1 = int((long long)B * (c + 1) / p->chunks);
            const std::size_t cnt = std::size_t(b1 - b0);
            ok(cudaMemcpyAsync(sl.img + b0 * N2, h_img + b0 * N2, cnt * N2 * 4, cudaMemcpyHostToDevice, p->si));
            h2d += cnt * N2 * 4;
            ok(cudaEventRecord(sl.uploaded[c], p->si));
            cudaStream_t s = p->sc[0];
            ok(cudaStreamWaitEvent(s, sl.uploaded[c], 0));
            if (tex) {
                ok(tt::fill_image_atlas_surf(sl.surf, sl.img + b0 * N2, n, int(cnt), (long long)N2, p->cols, s, b0));
                ++launches;
            }
            tt::TraceArgs ta = trace_args(0, p->units, b0, b1, 0);
            if (!ok(tt::launch_trace(ta, s))) break;
            launches += tt::trace_launch_count(ta);
            const std::size_t r0 = std::size_t(b0) * units_all, rows = cnt * units_all;
            if (d.features && !p->fused_circus) {
                ok(tt::launch_circus(sl.out + r0 * row_f, n, int(rows * tt::kNumF), sl.circ + r0 * row_c, s));
                ++launches;
            }
            ok(cudaEventRecord(sl.done[c], s));
            ok(cudaStreamWaitEvent(p->sx, sl.done[c], 0));
            download(r0, rows);
            if (d.features && h_circ) {
                ok(cudaMemcpyAsync(h_circ + r0 * row_c, sl.circ + r0 * row_c, rows * row_c * 4, cudaMemcpyDeviceToHost,
                                   p->sx));
                d2h += rows * row_c * 4;
            }
        }
    }
    if (graph) {
        ok(cudaEventRecord(sl.join, p->sx));  // the copy stream (which waited on every chunk) joins the origin
        ok(cudaStreamWaitEvent(p->si, sl.join, 0));
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(p->si, &g);  // always ends the capture
        ok(ce);
        if (e == cudaSuccess) ok(cudaGraphInstantiate(&sl.exec, g, 0));
        if (g) cudaGraphDestroy(g);
        if (e == cudaSuccess) {
            ++p->captures;
            sl.key = key;
            sl.g_h2d = h2d;
            sl.g_d2h = d2h;
            sl.g_launches = launches;
            ok(cudaGraphLaunch(sl.exec, sl.gs));
            ok(cudaEventRecord(sl.free, sl.gs));
        }
    } else {
        ok(cudaEventRecord(sl.free, p->sx));  // every download (and, before them, every kernel) of the slot
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "plan submit");
    ctx->c.bytes_h2d += h2d;
    ctx->c.bytes_d2h += d2h;
    ctx->c.gpu_kernel_launches += launches;
    return TT_OK;
}

tt_status tt_plan_wait(tt_plan* p) {
    Range r("tt_plan_wait");
    if (!p) return fail(nullptr, TT_ERR_INVALID, "null plan");
    DeviceGuard guard(p->ctx->device);
    cudaError_t e = cudaSuccess;
    for (cudaStream_t s : {p->sx, p->si, p->sc[0], p->sc[1]}) {
        const cudaError_t x = cudaStreamSynchronize(s);
        if (e == cudaSuccess) e = x;
    }
    for (const PlanSlot& sl : p->slot)
        if (sl.gs) {
            const cudaError_t x = cudaStreamSynchronize(sl.gs);
            if (e == cudaSuccess) e = x;
        }
    return e == cudaSuccess ? TT_OK : cuda_fail(p->ctx, e, "plan wait");
}

tt_status tt_plan_run(tt_plan* p, const float* h_img, float* h_out, std::int32_t* h_med, float* h_circ) {
    tt_status st = tt_plan_submit(p, h_img, h_out, h_med, h_circ);
    if (st != TT_OK) return st;
    return tt_plan_wait(p);
}

tt_status tt_plan_chunks(const tt_plan* p, int* chunks) {
    if (!p || !chunks) return fail(nullptr, TT_ERR_INVALID, "null argument");
    *chunks = p->chunks;
    return TT_OK;
}

tt_status tt_plan_captures(const tt_plan* p, int* captures) {
    if (!p || !captures) return fail(nullptr, TT_ERR_INVALID, "null argument");
    *captures = p->captures;
    return TT_OK;
}

tt_status tt_plan_destroy(tt_plan* p) {
    plan_release(p);
    return TT_OK;
}

}  // extern "C"

// ------------------------------------------------------------------- IPC

namespace {
std::mutex g_ipc_mu;
std::map<void*, void*> g_ipc_open;  // imported pointer (base + offset) -> mapped base
}  // namespace

extern "C" {

tt_status tt_ipc_export(const void* d_ptr, tt_ipc_handle* out) {
    if (!d_ptr || !out) return fail(nullptr, TT_ERR_INVALID, "null argument");
    static PFN_cuMemGetAddressRange_v3020 range = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(f);
    }();
    if (!range) return fail(nullptr, TT_ERR_CUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, CUdeviceptr(d_ptr)) != CUDA_SUCCESS)
        return fail(nullptr, TT_ERR_INVALID, "pointer is not inside a device allocation");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == sizeof(out->bytes), "IPC handle size");
    std::memcpy(out->bytes, &h, sizeof(h));
    out->offset = std::uint64_t(CUdeviceptr(d_ptr) - base);
    return TT_OK;
}

tt_status tt_ipc_alloc(int device, size_t bytes, void** d_ptr) {
    if (!d_ptr || bytes == 0) return fail(nullptr, TT_ERR_INVALID, "bad IPC allocation arguments");
    DeviceGuard guard(device);
    cudaError_t e = cudaMalloc(d_ptr, bytes);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaMalloc (IPC buffer)");
    e = cudaMemset(*d_ptr, 0, bytes);
    if (e != cudaSuccess) {
        cudaFree(*d_ptr);
        *d_ptr = nullptr;
        return cuda_fail(nullptr, e, "cudaMemset (IPC buffer)");
    }
    return TT_OK;
}

tt_status tt_ipc_free(void* d_ptr) {
    if (!d_ptr) return TT_OK;
    cudaError_t e = cudaFree(d_ptr);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "cudaFree (IPC buffer)");
}

tt_status tt_ipc_import(const tt_ipc_handle* hd, int device, void** d_ptr) {
    if (!hd || !d_ptr) return fail(nullptr, TT_ERR_INVALID, "null argument");
    DeviceGuard guard(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hd->bytes, sizeof(h));
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaIpcOpenMemHandle");
    *d_ptr = static_cast<char*>(base) + hd->offset;
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    g_ipc_open[*d_ptr] = base;
    return TT_OK;
}

tt_status tt_ipc_close(void* d_ptr) {
    void* base = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_ipc_mu);
        auto it = g_ipc_open.find(d_ptr);
        if (it == g_ipc_open.end()) return fail(nullptr, TT_ERR_INVALID, "pointer was not imported");
        base = it->second;
        g_ipc_open.erase(it);
    }
    cudaError_t e = cudaIpcCloseMemHandle(base);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "cudaIpcCloseMemHandle");
}

}  // extern "C"

