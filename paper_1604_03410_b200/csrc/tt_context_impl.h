// tt_context_impl.h — internals shared by the context translation units
// (tt_context.cpp: context, memory, modules, launches; tt_device_api.cpp:
// raw device entries, plans, IPC).  Not part of the C ABI.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "tt_b200.h"
#include "tt_jit.h"
#include "tt_kernels.cuh"

namespace ttc {

// ---------------------------------------------------------------- types

enum class Scalar : std::uint8_t { I32, I64, F32, F64 };

inline const char* scalar_name(Scalar t) {
    switch (t) {
        case Scalar::I32: return "i32";
        case Scalar::I64: return "i64";
        case Scalar::F32: return "f32";
        case Scalar::F64: return "f64";
    }
    return "?";
}

inline std::size_t scalar_bytes(Scalar t) { return (t == Scalar::I64 || t == Scalar::F64) ? 8 : 4; }

// vptx::Param (vptx.hpp:186-199): a by-value scalar or a global pointer.
struct Param {
    bool ptr = false;
    Scalar type = Scalar::I32;
    std::string name;
    bool written = false;  // the native kernel stores through this pointer
    bool operator==(const Param& o) const { return ptr == o.ptr && type == o.type; }
    std::string type_text() const { return ptr ? std::string("ptr.global.") + scalar_name(type) : scalar_name(type); }
    std::string sig_text() const { return ptr ? std::string(scalar_name(type)) + "[]" : scalar_name(type); }
};

struct KernelDecl {
    std::string name;
    std::vector<Param> params;
    std::vector<tt::jit::Line> body;  // instructions / declarations between '{' and '}' (JIT input)
    std::string signature() const {  // Signature::to_string, types.hpp:104-111
        std::string s = name + "(";
        for (std::size_t i = 0; i < params.size(); ++i) {
            if (i) s += ",";
            s += params[i].sig_text();
        }
        return s + ")";
    }
};

struct ResolvedArg {
    tt_arg_kind kind;
    tt_arg value;          // scalars
    void* dptr = nullptr;  // device address for pointers
    std::uint64_t bytes = 0;
    std::uint64_t base = 0;  // synthetic address (allocation key)
    std::uint64_t gen = 0;   // write generation of the allocation
    bool exported = false;   // its raw pointer was handed out (Alloc::exported)
};

struct LaunchOutcome {
    tt_status status = TT_OK;
    std::string error;
    tt_trap trap{};
    int gpu_launches = 0;
};
using LaunchFn = LaunchOutcome (*)(tt_ctx&, const tt_grid&, const std::vector<ResolvedArg>&);

struct NativeKernel {
    KernelDecl decl;
    LaunchFn fn;
    // A module binds to the native kernel when its kernel is header-only, or when its VPTX body
    // is one of the documented DSL bodies the native kernel stands in for, identified by
    // body_fingerprint() (trace_t05: oracle/trace_t05.krn as the reference front end compiles
    // it, tests/golden/trace_t05.vptx).  Any other body runs as written (JIT): a user kernel that
    // merely shares a name and signature is never replaced.
    std::vector<std::uint64_t> body_fingerprints;
};

// FNV-1a 64 over a kernel body's token stream (tokens separated by 0x1f, lines by '\n'):
// invariant under whitespace and comments, sensitive to every instruction and operand.
std::uint64_t body_fingerprint(const std::vector<tt::jit::Line>& body);


// ---------------------------------------------------------------- context

struct Alloc {
    void* dptr = nullptr;
    std::uint64_t bytes = 0;
    bool live = true;
    std::uint64_t gen = 0;  // bumped by every write (H2D copy, written launch argument)
    bool exported = false;  // raw pointer handed out (tt_mem_device_pointer): writes are invisible to
                            // the context, so cached derived copies (texture, weight layout) are
                            // refreshed at every launch that reads this allocation
};

// Texture-gather sampler state cached per image allocation: the block-linear
// cudaArray copy is refreshed only when the allocation's generation changed.
struct TexEntry {
    std::uint64_t gen = ~0ull;
    int n = 0;
    int batch = 1;
    int cols = 1;
    cudaArray_t arr = nullptr;     // null: a pitch-linear view of the image (nothing to refresh)
    cudaTextureObject_t tex = 0;
    const float* bound = nullptr;  // the image pointer the texture was made from
};

// Pass-2 weight layout (tt::launch_weights_soa) cached per wtab allocation,
// rebuilt only when the allocation's generation changed.
struct WeightEntry {
    std::uint64_t gen = ~0ull;
    int n = 0;
    float* d = nullptr;
};

struct LaunchRecord {
    std::string kernel;
    std::uint32_t grid[3] = {1, 1, 1};
    std::uint32_t block[3] = {1, 1, 1};
    std::uint64_t h2d = 0, d2h = 0;
};

struct Module {
    std::string name;
    std::vector<KernelDecl> kernels;
};

// A kernel without a native implementation, compiled from its VPTX body (tt_jit.h).
struct JitFunction {
    KernelDecl decl;
    tt::jit::Program prog;
    ~JitFunction() { tt::jit::release(prog); }
};

struct FunctionEntry {
    std::uint64_t module_id = 0;
    std::string kernel;
    const NativeKernel* native = nullptr;
    std::shared_ptr<JitFunction> jit;  // set when native == nullptr
};


}  // namespace ttc

struct tt_ctx {  // the C ABI's opaque context (include/tt_b200.h)
    std::uint64_t id = 0;
    int device = 0;
    tt_caps caps{1024, 48 * 1024};
    bool destroyed = false;
    cudaStream_t stream = nullptr;
    int sampler = 1;  // tt::Sampler for trace launches (default texture; TT_SAMPLER=ldg -> 0)

    std::map<std::uint64_t, ttc::Module> modules;
    std::map<std::uint64_t, ttc::FunctionEntry> functions;
    std::uint64_t next_handle = 1;

    std::map<std::uint64_t, ttc::Alloc> allocs;  // keyed by synthetic base address
    std::uint64_t bump = 4096;              // GlobalMemory::kBase, emulator.hpp:109

    tt_counters c{};
    std::vector<ttc::LaunchRecord> launch_log;
    std::vector<std::uint8_t> events;
    std::uint64_t h2d_mark = 0, d2h_mark = 0;

    std::string last_error;
    std::map<std::uint64_t, ttc::TexEntry> tex_cache;      // keyed by image allocation base
    std::map<std::uint64_t, ttc::WeightEntry> w_cache;     // keyed by wtab allocation base
    // JIT launches: the device trap record and the allocation table the bounds checks search
    tt::jit::TrapRecord* jit_trap = nullptr;
    unsigned long long* jit_rng = nullptr;
    std::size_t jit_rng_cap = 0;  // entries (3 words each)
};

namespace ttc {

// Error plumbing: records `msg` as the context's (and the thread's) last error.
tt_status fail(const tt_ctx* ctx, tt_status st, const std::string& msg);
tt_status cuda_fail(const tt_ctx* ctx, cudaError_t e, const char* what);
tt_status copy_out_text(const std::string& s, char* buf, std::size_t cap, std::size_t* needed);

// Makes the context's device current for the duration of a call.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};


}  // namespace ttc

#define TT_CHECK_CTX(ctx)                                                                       \
    do {                                                                                        \
        if ((ctx) == nullptr) return fail(nullptr, TT_ERR_INVALID, "null context");            \
        if ((ctx)->destroyed)                                                                   \
            return fail((ctx), TT_ERR_CONTEXT_DESTROYED, "ContextDestroyed: operation on a destroyed context"); \
    } while (0)
