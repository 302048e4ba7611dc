// qvg_jit.hpp — JIT-specialised fused tile passes (QVG_OPT_JIT).
//
// k_tile (qvg_tile.cuh) interprets a pass's op records: per op and warp it
// loads the record's fields from the parameter bank, tests them and jumps
// through a table into the op's body. On passes of many cheap ops (the QFT's
// controlled phases) that costs more issue slots than the FP64 work itself:
// ncu of a 128-op QFT pass at n = 28 counts ~52 non-FP64 instructions per op
// and warp against ~31 FP64 ones, with the FP64 pipe at 54% and issue at 64%
// (profiles/r02_ncu_summary.md).
//
// A JIT pass is the same kernel body (k_tile_body) with a generated op
// program (TileOpsJit) in place of the interpreter: every op's body, register
// slots, thread-bit and tile-base tests are compile-time constants, so an op
// costs its FP64 instructions plus at most a uniform branch, and its matrix is
// read as direct constant-bank operands of the very records k_tile reads. The
// arithmetic is the same device functions in the same order, so complex128
// stays bit-identical to k_tile and to the reference.
//
// Source generation and NVRTC compilation are host-only (no GPU needed);
// compiled kernels are cached per pass STRUCTURE (geometry, bits, classes,
// flags; not the matrix values, which stay in the parameter block), so a
// circuit whose angles change reuses them. The kernels an apply needs are
// compiled in parallel before its first launch (jit_prepare).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "qvg_tile.cuh"

namespace qvg {

struct JitVariant {
    int amp_bytes;  // 16 complex128, 8 complex64
    int sub;        // register subcube bits
    bool fma;       // complex128 DFMA arithmetic (QVG_OPT_FMA)
    int maxt;       // threads per CTA the instantiation serves (128 / 256 / 512)
    int cm;         // class-set mask (kClsSet*)
};

// The generated CUDA source of one pass (for tests and tools).
std::string jit_source(const TileGeom &g, const TileOp *recs, const JitVariant &v);

// Compile `src` with NVRTC for sm_100a; returns "" on success (cubin in *out
// if given) or the error log. Host-only.
std::string jit_compile(const std::string &src, std::string *cubin);

// Compile (in parallel, joined before returning) every requested pass whose
// kernel is not cached yet, load it, and set each request's `fn` to its
// function on the CURRENT device (nullptr: NVRTC unavailable or the compile
// failed; the caller then launches k_tile). Not inside a stream capture.
struct JitRequest {
    const TileGeom *g;
    const TileOp *recs;
    JitVariant v;
    void *fn;
};
void jit_prepare(JitRequest *reqs, size_t count);
// The cached, resolved function of a pass (jit_prepare ran for it on this
// device), else nullptr. No compile or module load: safe inside a capture.
void *jit_lookup(const TileGeom &g, const TileOp *recs, const JitVariant &v);

// Launch a function from jit_prepare / jit_lookup (driver API, the kernel's
// parameters are k_tile's: psi, TileParams). Dynamic shared memory above 48 KB
// is opted into once per function.
cudaError_t jit_launch(void *fn, unsigned grid, unsigned threads, size_t smem, cudaStream_t stream, void *psi,
                       const TileParams *prm);
// CTAs per SM of a JIT function at this shape (occupancy).
int jit_occupancy(void *fn, unsigned threads, size_t smem);

struct JitCounters {
    uint64_t compiled, failed;
    double compile_ms;  // summed NVRTC time (compiles of one jit_prepare run in parallel)
};
JitCounters jit_counters();
// True when NVRTC and the driver entry points could be loaded.
bool jit_available();

}  // namespace qvg
