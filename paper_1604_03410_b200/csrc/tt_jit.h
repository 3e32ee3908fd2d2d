// tt_jit.h — VPTX -> CUDA C++ -> sm_100a cubin for kernels without a native
// implementation (the paper's framework-compiled
// kernels running natively behind the same driver API).
//
// The reference runs a VPTX kernel on its emulator (run_kernel,
// /root/reference/proj/include/gridjit/emulator.hpp:747-793) with the
// semantics of /root/reference/proj/docs/vptx-isa.md.  The JIT emits one CUDA
// C++ kernel per VPTX kernel with the same arithmetic (explicit
// round-to-nearest intrinsics, no contraction, wrapping integers, saturating
// float->int, zero-initialised registers) and the same trap taxonomy: every
// ld/st is checked against the context's allocation table (global) or the
// block's shared extent, and the first trap in the emulator's order — blocks
// in lexicographic (x, y, z) order, then barrier phase, then linear thread id —
// is the one reported.  NVRTC compiles it for sm_100a at get_function time
// (once per signature: the caller's method cache).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace tt::jit {

enum class Ty : std::uint8_t { I32, I64, F32, F64, Pred };

struct Param {
    bool ptr = false;  // ptr.global.<elem>: passed as its device address (i64)
    Ty type = Ty::I32;
    std::string name;
};

struct Line {
    int no = 0;
    std::vector<std::string> toks;  // ',' '[' ']' '(' ')' '{' '}' are separate tokens
};

struct Program {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kernel = nullptr;
    std::uint64_t static_shared = 0;  // bytes of the kernel's .shared arrays
    std::string source;               // generated CUDA C++ (diagnostics)
};

// Device-side trap record (one per context).
struct TrapRecord {
    unsigned long long key;  // ~0: no trap
    int lock;
    int kind;
    long long code;
    int instr;
    unsigned tid[3], ctaid[3];
};

// Translates kernel `name` (params, body lines between '{' and '}') and
// compiles it.  Returns false with `err` on unsupported input or a compile
// failure.
bool compile(const std::string& name, const std::vector<Param>& params, const std::vector<Line>& body,
             Program& out, std::string& err);

void release(Program& p);

// The CUDA C++ the JIT would compile (no NVRTC, no device): for diagnostics and CPU tests.
bool translate(const std::string& name, const std::vector<Param>& params, const std::vector<Line>& body,
               std::string& source, std::uint64_t& static_shared, std::string& err);

}  // namespace tt::jit
