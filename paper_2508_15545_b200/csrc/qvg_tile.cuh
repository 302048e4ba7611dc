// qvg_tile.cuh — K4, the fused tile pass: the B200 replacement for the
// reference's block store + sliding window (reference store.cpp, cache.cpp,
// kernel.cpp:113-146).
//
// A CTA owns a tile of 2^k amplitudes and applies a run of gates to it in
// circuit order, so the whole run costs one HBM round trip instead of one per
// gate. The tile is the set of amplitudes that agree on every qubit outside
// the tile qubit set Q (|Q| = k): its lowest `lowc` qubits are 0..lowc-1
// (contiguous 2^lowc-amplitude segments in HBM, >= 128 B), the other k-lowc
// are arbitrary high qubits, so gates on any qubit can be fused. A control
// outside Q is constant per tile, and a diagonal gate needs no pairing, so its
// qubits may lie anywhere.
//
// Inside the tile the run is cut into groups whose pair ops touch at most SUB
// tile bits. For a group, each of the 2^(k-SUB) threads holds the 2^SUB
// amplitudes of one SUB-bit subcube in registers and applies all the group's
// ops there; shared memory is only the transpose buffer between groups. The
// first group reads HBM directly and the last one writes HBM directly, so a
// run that fits one group never touches the shared tile. The op records (the
// same for every tile) travel in the kernel's parameter bank.
//
// Measured limits (profiles/r01_fused_ab.json, r01_ncu_summary.md): the kernel
// is compute/latency-bound, not HBM-bound (issue slots ~59%, FP64 pipe ~42% on
// a grid pass). DFMA arithmetic (half the FP64 instructions) gains only 10-13%,
// and a cp.async next-tile prefetch (fewer CTAs/SM) loses 10-15%. What helped:
// pair and diagonal ops dispatched at compile time by register slot, one jump
// table per op dispatch, structured-matrix bodies, per-case record loads, and
// 16 register amplitudes per thread.
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda.h>  // CUtensorMap (k_tile_tma's tensor-map descriptor; types only, no driver link)
#include <cuda_runtime.h>
#include <stdint.h>
#else  // NVRTC (qvg_jit.hpp): the descriptor's layout only (128 B, 64-B aligned)
typedef struct alignas(64) { unsigned long long opaque[16]; } CUtensorMap;
#endif

#include "qvg_kernels.cuh"

namespace qvg {

enum TileOpKind : int32_t { TILE_PAIR = 0, TILE_DIAG = 1, TILE_GROUP = 2 };

// One record of a tile pass: a group header followed by its ops.
struct __align__(16) TileOp {
    int32_t kind;      // TileOpKind
    int32_t tbit;      // pair/diag: tile-local target bit (-1: diag target outside Q; diag target
                       // in Q but not in the group: its thread-index bit); group: op count
    int32_t cbit;      // tile-local control bit, -1 if none or outside Q (diag control in Q but
                       // not in the group: its thread-index bit)
    int32_t slot;      // dispatch index | flags (op_dispatch): pair 30*class+6*J+(K+1), diag
                       // 180+36*neg+6*(J+1)+(K+1); J/K: register slots
    uint64_t greq;     // global bits that must be 1 in the tile base (controls outside Q)
    uint64_t gtgt;     // diag: global target bit outside Q; group: packed bits b0 | b1<<8 | b2<<16 | b3<<24
    double u[8];       // group: u[j] holds (as bits) the global offset of tile-local bit b_j; op: matrix (diag uses u00 = u[0..1], u11 = u[6..7]); complex64 passes: the same
                       // 8 values as floats in the first 32 bytes (no per-use conversion)
};
static_assert(sizeof(TileOp) == 96, "TileOp layout");

struct TileGeom {
    int n, k, lowc;       // qubits, tile qubits, contiguous low qubits
    int nhi;              // k - lowc
    int ngroups;          // register groups in this pass
    int nrec;             // records (headers + ops)
    int sub;              // subcube bits per thread (3 or 4)
    int stage;            // bit 0: first group loads through shared memory; bit 1: last group stores through it
    int cls_set;          // structured-matrix classes this pass uses (kClsSetReal / kClsSetHalf)
    int order;            // tiles per CTA: 0 strided (blockIdx.x + i * gridDim.x), 1 contiguous chunks
                          // (successive tiles of a CTA are DRAM neighbours, tile_range)
    int hiq[24];          // tile qubits >= lowc, ascending (tile-local bits lowc..k-1)
    uint64_t ntiles;      // 2^(n-k)
    uint64_t sdep[5];     // global offset of tile-local bit (k - sub + i): the staged (coalesced)
                          // layout's index t + j*blockDim is t | j << (k - sub)
#ifdef QVG_TILE_TRACE     // tools/tile_trace.py (debug build `make trace` only): per-tile phase stamps
    unsigned long long *trace;  // 24 words per tile in [trace_first, trace_first + trace_count)
    uint64_t trace_first, trace_count;
#endif
};

// Phase stamps of one tile (thread 0 of its CTA), compiled in only by the
// debug build (`make trace`, libqvg_trace.so): words 0 smid, 1 globaltimer at
// the tile's start, 2 clock at its start, 3 clock at its end, 4 globaltimer at
// its end, 5 groups, then per register group gi < 6: 6+3gi amplitudes arrived,
// 7+3gi ops done, 8+3gi written back (and the barrier passed); 22 clock after
// the start stamps, 23 clock at kernel entry.
struct TileTrace {
#ifdef QVG_TILE_TRACE
    unsigned long long *p = nullptr;
    unsigned long long entry = 0;
    __device__ __forceinline__ void enter() { entry = clock64(); }
    __device__ __forceinline__ void begin(const TileGeom &g, uint64_t tile) {
        p = nullptr;
        if (g.trace && threadIdx.x == 0 && tile >= g.trace_first && tile - g.trace_first < g.trace_count) {
            p = g.trace + 24 * (tile - g.trace_first);
            const unsigned long long c0 = clock64();
            unsigned smid;
            unsigned long long gt;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
            p[0] = smid;
            p[1] = gt;
            p[2] = c0;
            p[22] = clock64();
            p[23] = entry;
        }
    }
    __device__ __forceinline__ void mark(int w) {
        if (p && w < 22) p[w] = clock64();
    }
    // stamp once `a` and `b` (the group's first and last register amplitude) hold their values
    template <class X>
    __device__ __forceinline__ void mark_after(int w, X a, X b) {
        if (p && w < 22) {
            unsigned long long sink;
            asm volatile("mov.b64 %0, %1;" : "=l"(sink) : "l"(__double_as_longlong((double)a) ^ __double_as_longlong((double)b)));
            p[w] = clock64() | (sink & 0);
        }
    }
    __device__ __forceinline__ void end(int ngroups) {
        if (p) {
            const unsigned long long c1 = clock64();
            unsigned long long gt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
            p[3] = c1;
            p[4] = gt;
            p[5] = (unsigned long long)ngroups;
        }
    }
#else
    __device__ __forceinline__ void enter() {}
    __device__ __forceinline__ void begin(const TileGeom &, uint64_t) {}
    __device__ __forceinline__ void mark(int) {}
    template <class X>
    __device__ __forceinline__ void mark_after(int, X, X) {}
    __device__ __forceinline__ void end(int) {}
#endif
};

// Records per fused pass; they travel as the kernel's parameter block
// (CUDA 12.1+ allows 32 KB of parameters).
// (A 32-record block, 3 KB instead of 25 KB, measured no faster to launch at
// n = 12..22.)
constexpr int kMaxTileRecs = 256;
// k_tile_tma (qvg_tile_pipe.cuh): the tile as ONE box of a <= 5-D tensor map
// over the state. Dim 0 is a 128-B row (the lowest rb = log2(128 / S)
// amplitude bits); dims 1.. are the alternating runs of tile and non-tile
// qubits above it, from bit rb up. A tile dim's box spans the run (its
// coordinate is 0); a non-tile ("gap") dim's box is 1 and its coordinate is
// the tile base's bits in that run. Unused dims have size 1.
struct TileTma {
    CUtensorMap map;  // cuTensorMapEncodeTiled, UINT64 elements, SWIZZLE_128B
    int shift[5];     // first amplitude-index bit of dim d (d >= 1)
    int len[5];       // bits of dim d
    int gap[5];       // 1: coordinate = (base >> shift) & (2^len - 1)
};
struct TileParams {
    TileGeom g;
    TileTma tma;  // k_tile_tma only
    TileOp ops[kMaxTileRecs];
};
static_assert(sizeof(TileParams) < 32000, "kernel parameter block limit");

// The tiles a CTA processes: [first, end) with stride `step`.
struct TileRange {
    uint64_t first, end, step;
};
__device__ __forceinline__ TileRange tile_range(const TileGeom &g) {
    if (!g.order) return {blockIdx.x, g.ntiles, gridDim.x};
    const uint64_t per = (g.ntiles + gridDim.x - 1) / gridDim.x;
    const uint64_t f = (uint64_t)blockIdx.x * per;
    return {f, f + per < g.ntiles ? f + per : g.ntiles, 1};
}

// Shared-tile slot of local index l: the 16-B column within each 128-B row is
// XORed with the row's low bits, so lanes whose amplitudes are 2^3, 2^4 or
// 2^5 apart (a group over the carrier bits) hit different banks.
__device__ __forceinline__ uint32_t swz(uint32_t l) { return l ^ ((l >> 3) & 7u); }

// Pair op over the 2^SUB register amplitudes. Target on register slot J, control on slot K (-1: none / decided per tile):
// both are compile-time, so a controlled op costs exactly its pairs and no
// per-pair tests run (the instruction mix was 60% non-FP64 before this).
// The matrix is read here, straight from the record in the parameter bank,
// so each op loads only what its case uses.
template <class R, int SUB, int J, int K, bool FMA>
__device__ __forceinline__ void group_pair(typename Cplx<R>::T (&v)[1 << SUB], const R *uu) {
    if constexpr (J < SUB && K < SUB && J != K) {
        R u[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) u[x] = uu[x];
#pragma unroll
        for (int r = 0; r < (1 << SUB); ++r) {
            if ((r >> J) & 1) continue;
            if (K >= 0 && !((r >> K) & 1)) continue;
            const typename Cplx<R>::T a = v[r], b = v[r | (1 << J)];
            v[r] = madd2x<FMA>(u[0], u[1], a, u[2], u[3], b);
            v[r | (1 << J)] = madd2x<FMA>(u[4], u[5], a, u[6], u[7], b);
        }
    }
}

// Structured matrices (class chosen by the planner, qvg_plan.hpp
// pair_class). Each computes the reference's value with fewer FP64
// instructions; terms whose matrix entry is 0 contribute +-0, which changes
// at most the sign of an exact-zero result.
//   TILE_CLS_REAL: every imaginary part is 0 (H, real rotations):
//     lo = (u00r*a.re + u01r*b.re, u00r*a.im + u01r*b.im), 12 instead of 28.
//   TILE_CLS_SWAP: [[0,1],[1,0]] (X, the target of CX): a swap, each component
//     moved through one DADD with +0 (mov_opaque).
//   TILE_CLS_HALF: every |re| and |im| is 1/2 (sqrt(X), sqrt(Y), their
//     adjoints): with u00 = (s0, s1)/2, u01 = (s2, s3)/2,
//       lo.re = s0/2 * ((a.re - s0s1 a.im) + s0s2 (b.re - s2s3 b.im)),
//     and likewise for lo.im and hi. Halving is exact and commutes with
//     round-to-nearest, and so does negation, so this equals the
//     reference's (s0/2 a.re - s1/2 a.im) + (s2/2 b.re - s3/2 b.im) bit for
//     bit (unless an intermediate falls below 2^-1021 in magnitude, where
//     halving rounds). 16 FP64 instructions instead of 28.
//   TILE_CLS_SQW: diagonal entries as in HALF, u01 = (0, q) imaginary and
//     u10 = (p, 0) real (sqrt(W) of the grid circuits): with u00 = (s0, s1)/2,
//       lo.re = fma(s0/2, a.re - s0s1 a.im, -(q*b.im)),
//     where s0/2 times the bracket is exact, so the DFMA rounds like the
//     reference's final DADD, and 0*b.re contributes +-0. 12 instead of 28.
//   TILE_CLS_U00R: u00 real (U3: u00 = cos(theta/2)), the rest general:
//     lo.re = u00r*a.re + (u01r*b.re - u01i*b.im), the reference's 0*a.im
//     term being +-0. 24 instead of 28.
enum TileCls : int32_t {
    TILE_CLS_GEN = 0,
    TILE_CLS_REAL = 1,
    TILE_CLS_SWAP = 2,
    TILE_CLS_HALF = 3,
    TILE_CLS_SQW = 4,
    TILE_CLS_U00R = 5
};

__device__ __forceinline__ double xsgn(double x, uint32_t m) {
    return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x));
}
__device__ __forceinline__ float xsgn(float x, uint32_t m) { return __int_as_float(__float_as_int(x) ^ (int)m); }
template <class R> __device__ __forceinline__ R neg_rn(R x) { return xsgn(x, 0x80000000u); }
// The SWAP class moves each component through one DADD with +0 (-0 becomes
// +0, nothing else changes). Plain register renaming or inline-asm moves
// made ptxas spill in the 96-register tile kernel: each switch case then
// leaves the amplitudes in a different register assignment.
__device__ __forceinline__ double2 mov_opaque(double2 x) {
    return make_double2(__dadd_rn(x.x, 0.0), __dadd_rn(x.y, 0.0));
}
__device__ __forceinline__ float2 mov_opaque(float2 x) {
    return make_float2(__fadd_rn(x.x, 0.0f), __fadd_rn(x.y, 0.0f));
}

// HALF-class records carry, per output row x (0 = lo, 1 = hi), four reals
// u[4x..4x+3] = (s0/2, -s0 s1, -s2 s3, s0 s2) instead of the matrix
// (pair_record, qvg_plan.hpp). A DFMA by +-1 is exact before its single
// rounding, so fma(c, y, x) rounds exactly like x + c*y as DADD/DSUB: four
// FP64 instructions per component, no sign-bit moves, and every constant is
// a parameter-bank operand (ptxas reloads rather than spills it).
template <class T, class R>
__device__ __forceinline__ T half_apply(const R *uu, T a, T b) {
    const R h = uu[0], c1 = uu[1], c2 = uu[2], c3 = uu[3];
    T o;
    if constexpr (sizeof(R) == 8) {
        const double xr = __fma_rn(c1, a.y, a.x), yr = __fma_rn(c2, b.y, b.x);
        const double xi = __fma_rn(-c1, a.x, a.y), yi = __fma_rn(-c2, b.x, b.y);
        o.x = __dmul_rn(__fma_rn(c3, yr, xr), h);
        o.y = __dmul_rn(__fma_rn(c3, yi, xi), h);
    } else {
        const R xr = fmaf(c1, a.y, a.x), yr = fmaf(c2, b.y, b.x);
        const R xi = fmaf(-c1, a.x, a.y), yi = fmaf(-c2, b.x, b.y);
        o.x = fmaf(c3, yr, xr) * h;
        o.y = fmaf(c3, yi, xi) * h;
    }
    return o;
}

// REAL class: (m0*a.re + m1*b.re, m0*a.im + m1*b.im); the entries are read
// at the point of use (parameter-bank operands, reloaded under pressure).
template <class T, class R, bool FMA>
__device__ __forceinline__ T real_apply(R m0, R m1, T a, T b) {
    T o;
    if constexpr (sizeof(R) == 8 && !FMA) {
        o.x = __dadd_rn(__dmul_rn(m0, a.x), __dmul_rn(m1, b.x));
        o.y = __dadd_rn(__dmul_rn(m0, a.y), __dmul_rn(m1, b.y));
    } else {
        o.x = (R)m0 * a.x + (R)m1 * b.x;
        o.y = (R)m0 * a.y + (R)m1 * b.y;
    }
    return o;
}

// SQW-class records carry per output row the half entry's (s0/2, -s0 s1)
// and the off-diagonal entry's non-zero part: lo (u00, u01 = (0, q)) in
// u[0..2] = (s0/2, -s0 s1, q), hi (u11, u10 = (p, 0)) in u[4..6] =
// (s0'/2, -s0' s1', p) (sqw_record, qvg_plan.hpp).
template <class T, class R>
__device__ __forceinline__ T sqw_lo(const R *uu, T a, T b) {  // u00 a + (0, q) b
    const R s = uu[0], c1 = uu[1], q = uu[2];
    T r;
    if constexpr (sizeof(R) == 8) {
        r.x = __fma_rn(s, __fma_rn(c1, a.y, a.x), -__dmul_rn(q, b.y));
        r.y = __fma_rn(s, __fma_rn(-c1, a.x, a.y), __dmul_rn(q, b.x));
    } else {
        r.x = fmaf(s, fmaf(c1, a.y, a.x), -(q * b.y));
        r.y = fmaf(s, fmaf(-c1, a.x, a.y), q * b.x);
    }
    return r;
}
template <class T, class R>
__device__ __forceinline__ T sqw_hi(const R *uu, T a, T b) {  // (p, 0) a + u11 b
    const R s = uu[4], c1 = uu[5], p = uu[6];
    T r;
    if constexpr (sizeof(R) == 8) {
        r.x = __fma_rn(s, __fma_rn(c1, b.y, b.x), __dmul_rn(p, a.x));
        r.y = __fma_rn(s, __fma_rn(-c1, b.x, b.y), __dmul_rn(p, a.y));
    } else {
        r.x = fmaf(s, fmaf(c1, b.y, b.x), p * a.x);
        r.y = fmaf(s, fmaf(-c1, b.x, b.y), p * a.y);
    }
    return r;
}

// Class sets a k_tile instantiation compiles (CM: bit per TileCls). With all
// four sets of bodies in one 96-register kernel ptxas spills inside the
// bodies (~1 KB of local traffic per op); with three it does not. The planner
// picks the set per pass (tile_class_set, qvg_plan.hpp).
constexpr int kClsSetReal = (1 << TILE_CLS_GEN) | (1 << TILE_CLS_REAL) | (1 << TILE_CLS_SWAP);
constexpr int kClsSetHalf = (1 << TILE_CLS_GEN) | (1 << TILE_CLS_HALF) | (1 << TILE_CLS_SWAP);
constexpr int kClsSetHalfW = (1 << TILE_CLS_GEN) | (1 << TILE_CLS_HALF) | (1 << TILE_CLS_SQW);
constexpr int kClsSetU3 = (1 << TILE_CLS_GEN) | (1 << TILE_CLS_U00R) | (1 << TILE_CLS_SWAP);
template <class R, int SUB, int J, int K, bool FMA, int CLS, int CM>
__device__ __forceinline__ void group_pair_cls(typename Cplx<R>::T (&v)[1 << SUB], const R *uu) {
    using T = typename Cplx<R>::T;
    if constexpr (J < SUB && K < SUB && J != K && ((CM >> CLS) & 1)) {
        if constexpr (CLS == TILE_CLS_SWAP) {
#pragma unroll
            for (int r = 0; r < (1 << SUB); ++r) {
                if ((r >> J) & 1) continue;
                if (K >= 0 && !((r >> K) & 1)) continue;
                const T a = v[r], b = v[r | (1 << J)];
                v[r] = mov_opaque(b);
                v[r | (1 << J)] = mov_opaque(a);
            }
        } else if constexpr (CLS == TILE_CLS_REAL) {
#pragma unroll
            for (int r = 0; r < (1 << SUB); ++r) {
                if ((r >> J) & 1) continue;
                if (K >= 0 && !((r >> K) & 1)) continue;
                const T a = v[r], b = v[r | (1 << J)];
                v[r] = real_apply<T, R, FMA>(uu[0], uu[2], a, b);
                v[r | (1 << J)] = real_apply<T, R, FMA>(uu[4], uu[6], a, b);
            }
        } else if constexpr (CLS == TILE_CLS_SQW) {
#pragma unroll
            for (int r = 0; r < (1 << SUB); ++r) {
                if ((r >> J) & 1) continue;
                if (K >= 0 && !((r >> K) & 1)) continue;
                const T a = v[r], b = v[r | (1 << J)];
                v[r] = sqw_lo<T, R>(uu, a, b);
                v[r | (1 << J)] = sqw_hi<T, R>(uu, a, b);
            }
        } else if constexpr (CLS == TILE_CLS_U00R) {
#pragma unroll
            for (int r = 0; r < (1 << SUB); ++r) {
                if ((r >> J) & 1) continue;
                if (K >= 0 && !((r >> K) & 1)) continue;
                const T a = v[r], b = v[r | (1 << J)];
                if constexpr (sizeof(R) == 8) {
                    v[r] = make_double2(
                        __dadd_rn(__dmul_rn(uu[0], a.x), __dsub_rn(__dmul_rn(uu[2], b.x), __dmul_rn(uu[3], b.y))),
                        __dadd_rn(__dmul_rn(uu[0], a.y), __dadd_rn(__dmul_rn(uu[2], b.y), __dmul_rn(uu[3], b.x))));
                } else {
                    v[r].x = uu[0] * a.x + (uu[2] * b.x - uu[3] * b.y);
                    v[r].y = uu[0] * a.y + (uu[2] * b.y + uu[3] * b.x);
                }
                v[r | (1 << J)] = madd2x<FMA>(uu[4], uu[5], a, uu[6], uu[7], b);
            }
        } else {  // TILE_CLS_HALF
#pragma unroll
            for (int r = 0; r < (1 << SUB); ++r) {
                if ((r >> J) & 1) continue;
                if (K >= 0 && !((r >> K) & 1)) continue;
                const T a = v[r], b = v[r | (1 << J)];
                v[r] = half_apply<T, R>(uu, a, b);
                v[r | (1 << J)] = half_apply<T, R>(uu + 4, a, b);
            }
        }
    }
}

// Diagonal op diag(d0, d1) over the register subcube. The target is on slot J
// (-1: outside the group, then t1 is its value for this thread's whole
// subcube). The control is on slot K (-1: none, or tested per thread/tile
// before the call). J and K are compile-time, so e.g. a CZ with both bits in
// the group costs 2 complex multiplies, not 8 predicated ones. Whether
// d0 != 1 (target-0 elements change too) is a run-time flag: one body per
// (J, K) keeps the kernel's code small, which measured 2-3% faster than a
// body per (J, K, d0) (i-cache). Each element gets exactly one multiply, so
// the bits are the same either way. NEG (planner class: d0 = 1, d1 = -1, i.e.
// Z and CZ) flips the sign bits instead: (-1)*re - 0*im is -re up to the sign
// of an exact zero, and no FP64 instruction is issued.
template <class R, int SUB, int J, int K, bool FMA, bool NEG>
__device__ __forceinline__ void group_diag_rt(typename Cplx<R>::T (&v)[1 << SUB], const R *uu, bool t1,
                                              bool d0) {
    using T = typename Cplx<R>::T;
    auto neg = [](T x) {
        x.x = neg_rn(x.x);
        x.y = neg_rn(x.y);
        return x;
    };
    if constexpr (J < SUB && K < SUB && (J != K || J < 0)) {
        if constexpr (J >= 0) {
            if constexpr (NEG) {
#pragma unroll
                for (int r = 0; r < (1 << SUB); ++r) {
                    if (K >= 0 && !((r >> K) & 1)) continue;
                    if ((r >> J) & 1) v[r] = neg(v[r]);
                }
                return;
            } else {
                const R d1r = uu[6], d1i = uu[7];
#pragma unroll
                for (int r = 0; r < (1 << SUB); ++r) {
                    if (K >= 0 && !((r >> K) & 1)) continue;
                    if ((r >> J) & 1) v[r] = cmulx<FMA>(d1r, d1i, v[r]);
                }
            }
            if (d0) {
                const R d0r = uu[0], d0i = uu[1];
#pragma unroll
                for (int r = 0; r < (1 << SUB); ++r) {
                    if (K >= 0 && !((r >> K) & 1)) continue;
                    if (!((r >> J) & 1)) v[r] = cmulx<FMA>(d0r, d0i, v[r]);
                }
            }
        } else {
            if (!t1 && !d0) return;
            if constexpr (NEG) {
                if (!t1) return;
#pragma unroll
                for (int r = 0; r < (1 << SUB); ++r) {
                    if (K >= 0 && !((r >> K) & 1)) continue;
                    v[r] = neg(v[r]);
                }
                return;
            } else {
                const R dr = t1 ? uu[6] : uu[0], di = t1 ? uu[7] : uu[1];
#pragma unroll
                for (int r = 0; r < (1 << SUB); ++r) {
                    if (K >= 0 && !((r >> K) & 1)) continue;
                    v[r] = cmulx<FMA>(dr, di, v[r]);
                }
            }
        }
    }
}

// One dense dispatch index per op (TileOp::slot & 0xff), so the switch
// compiles to a single jump table (one indirect branch per op). Sparse codes
// compiled to a compare-and-branch tree, and the instruction-fetch bubbles
// after its branches were the kernel's top stall (no_instruction).
//   pair:     30*class + 6*J + (K+1)              0..179
//   diagonal: 180 + 36*neg + 6*(J+1) + (K+1)     180..251
// (J, K < 5: register slots of up to 32-amplitude subcubes)
constexpr int kDispDiag = 180;
constexpr int kSlotCtlTest = 256;  // diagonal: control in the tile but not in the group: test per thread
constexpr int kSlotT1 = 512;       // diagonal: target not in the group: t1 per thread / tile
constexpr int kSlotD0 = 1024;      // diagonal: d0 != 1
template <class R, int SUB, bool FMA, int CM>
__device__ __forceinline__ void op_dispatch(int d, typename Cplx<R>::T (&v)[1 << SUB], const R *u, bool t1,
                                            bool d0) {
#define QVG_GP(J, K)                                                                          \
    case 30 * TILE_CLS_GEN + 6 * (J) + (K) + 1: group_pair<R, SUB, J, K, FMA>(v, u); break;   \
    case 30 * TILE_CLS_REAL + 6 * (J) + (K) + 1:                                              \
        group_pair_cls<R, SUB, J, K, FMA, TILE_CLS_REAL, CM>(v, u);                           \
        break;                                                                                \
    case 30 * TILE_CLS_SWAP + 6 * (J) + (K) + 1:                                              \
        group_pair_cls<R, SUB, J, K, FMA, TILE_CLS_SWAP, CM>(v, u);                           \
        break;                                                                                \
    case 30 * TILE_CLS_HALF + 6 * (J) + (K) + 1:                                              \
        group_pair_cls<R, SUB, J, K, FMA, TILE_CLS_HALF, CM>(v, u);                           \
        break;                                                                                \
    case 30 * TILE_CLS_SQW + 6 * (J) + (K) + 1:                                               \
        group_pair_cls<R, SUB, J, K, FMA, TILE_CLS_SQW, CM>(v, u);                            \
        break;                                                                                \
    case 30 * TILE_CLS_U00R + 6 * (J) + (K) + 1:                                              \
        group_pair_cls<R, SUB, J, K, FMA, TILE_CLS_U00R, CM>(v, u);                           \
        break;
#define QVG_GD(J, K)                                                  \
    case kDispDiag + 6 * ((J) + 1) + (K) + 1:                         \
        group_diag_rt<R, SUB, J, K, FMA, false>(v, u, t1, d0);        \
        break;                                                        \
    case kDispDiag + 36 + 6 * ((J) + 1) + (K) + 1:                    \
        group_diag_rt<R, SUB, J, K, FMA, true>(v, u, t1, false);      \
        break;
    switch (d) {
        QVG_GP(0, -1) QVG_GP(0, 1) QVG_GP(0, 2) QVG_GP(0, 3) QVG_GP(0, 4)
        QVG_GP(1, -1) QVG_GP(1, 0) QVG_GP(1, 2) QVG_GP(1, 3) QVG_GP(1, 4)
        QVG_GP(2, -1) QVG_GP(2, 0) QVG_GP(2, 1) QVG_GP(2, 3) QVG_GP(2, 4)
        QVG_GP(3, -1) QVG_GP(3, 0) QVG_GP(3, 1) QVG_GP(3, 2) QVG_GP(3, 4)
        QVG_GP(4, -1) QVG_GP(4, 0) QVG_GP(4, 1) QVG_GP(4, 2) QVG_GP(4, 3)
        QVG_GD(-1, -1) QVG_GD(-1, 0) QVG_GD(-1, 1) QVG_GD(-1, 2) QVG_GD(-1, 3) QVG_GD(-1, 4)
        QVG_GD(0, -1) QVG_GD(0, 1) QVG_GD(0, 2) QVG_GD(0, 3) QVG_GD(0, 4)
        QVG_GD(1, -1) QVG_GD(1, 0) QVG_GD(1, 2) QVG_GD(1, 3) QVG_GD(1, 4)
        QVG_GD(2, -1) QVG_GD(2, 0) QVG_GD(2, 1) QVG_GD(2, 3) QVG_GD(2, 4)
        QVG_GD(3, -1) QVG_GD(3, 0) QVG_GD(3, 1) QVG_GD(3, 2) QVG_GD(3, 4)
        QVG_GD(4, -1) QVG_GD(4, 0) QVG_GD(4, 1) QVG_GD(4, 2) QVG_GD(4, 3)
    default: break;
    }
#undef QVG_GP
#undef QVG_GD
}

// MAXT: the largest CTA this instantiation serves (2^(k-SUB) threads). The
// minimum-blocks hint keeps 4 CTAs/SM (64 registers) at 256 threads: measured
// faster than 3 CTAs with 80 registers and no spills (C3 1278 vs 1356 ms).
// PF (SUB = 3 only): each thread loads the next tile's first-group amplitudes
// into registers while it computes the current tile, so the first group's
// HBM latency (the top stall without it: DMULs waiting on those loads,
// long_scoreboard) overlaps compute. It costs 32 registers, so such CTAs run
// at 2 per SM (16 warps, as many as the default 16-amplitude subcubes).
#ifndef QVG_SUB4_MINB
#define QVG_SUB4_MINB 5  // CTAs/SM hint for 128-thread 16-amplitude tiles: 96 registers, no spills.
                         // 5 vs 6 (80 registers, spills): C2 -5%, C0-style -5%, C1 +3%; vs 4 (128): better everywhere
#endif
#ifndef QVG_SUB4_256_MINB
#define QVG_SUB4_256_MINB 3  // 256-thread 16-amplitude tiles (12-qubit tiles): 80 registers, no spills
#endif
#ifndef QVG_C64_SUB4_256_MINB
#define QVG_C64_SUB4_256_MINB 4  // complex64 (its default tile): 64 registers; 4-6% faster than 3 CTAs, 5 spills
#endif
#ifndef QVG_SUB5_MINB
#define QVG_SUB5_MINB 5  // complex64 32-amplitude subcubes, 128 threads: 96 registers
                         // (vs 4 CTAs at 128: C1 -5%, C3 -4%; profiles/r01_sub5_ab.json)
#endif
template <class R, int SUB, int MAXT, bool PF>
constexpr int tile_min_blocks() {
    return PF                           ? 2
           : (SUB == 5)                 ? (MAXT <= 128 ? QVG_SUB5_MINB : 2)
           : (MAXT <= 128 && SUB == 4)  ? QVG_SUB4_MINB
           : (MAXT <= 256 && SUB == 4)  ? (sizeof(R) == 4 ? QVG_C64_SUB4_256_MINB : QVG_SUB4_256_MINB)
           : (MAXT <= 256 && SUB == 3)  ? 4
                                        : 2;
}

// The op program of a register group, run by k_tile_body between the group's
// load and store. TileOpsRuntime interprets the pass's records (one jump-table
// dispatch per op); a JIT-specialised pass (qvg_jit.hpp) supplies a program
// with every op's body, bits and tests fixed at compile time and its matrix
// read from the same parameter-bank record.
struct TileOpsRuntime {
    template <class R, int SUB, bool FMA, int CM>
    static __device__ __forceinline__ void apply(int /*gi*/, typename Cplx<R>::T (&v)[1 << SUB], uint64_t base,
                                                 const TileOp *ops, int rec, int nops) {
        for (int i = 0; i < nops; ++i) {
            const TileOp &op = ops[rec + i];
            if ((base & op.greq) != op.greq) continue;  // control outside the tile is 0
            const int sl = op.slot;
            // tile bits outside the group are bits of the thread index
            // (the planner stores their thread-bit positions)
            if ((sl & kSlotCtlTest) && !((threadIdx.x >> op.cbit) & 1u)) continue;
            bool t1 = false;
            if (sl & kSlotT1) t1 = op.tbit >= 0 ? ((threadIdx.x >> op.tbit) & 1u) != 0 : (base & op.gtgt) != 0;
            // complex64 records carry the matrix as 8 floats (tile_record_precision)
            op_dispatch<R, SUB, FMA, CM>(sl & 0xff, v, reinterpret_cast<const R *>(op.u), t1, (sl & kSlotD0) != 0);
        }
    }
};


template <class R, int SUB, bool FMA, int MAXT, bool PF, int CM, class Ops>
__device__ __forceinline__ void k_tile_body(typename Cplx<R>::T *__restrict__ psi, const TileParams &prm) {
    using T = typename Cplx<R>::T;
    constexpr int E = 1 << SUB;
    const TileGeom &g = prm.g;
    TileTrace trc;
    trc.enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // Op records are read straight from the kernel's parameter (constant)
    // bank: the index is warp-uniform, so they load through the constant
    // cache into uniform registers with no shared-memory traffic.
    const TileOp *ops = prm.ops;
    uint64_t *offhi = reinterpret_cast<uint64_t *>(smem_raw);
    T *sm = reinterpret_cast<T *>(smem_raw + (((sizeof(uint64_t) << g.nhi) + 15) & ~15ull));
    const bool use_sm = g.ngroups > 1 || g.stage != 0;
    const uint32_t nhi = 1u << g.nhi;
    const uint32_t lowm = (1u << g.lowc) - 1u;
    {  // the high-qubit offset table
        for (uint32_t h = threadIdx.x; h < nhi; h += blockDim.x) {
            uint64_t off = 0;
#pragma unroll
            for (int i = 0; i < 24; ++i)
                if (i < g.nhi && ((h >> i) & 1u)) off |= 1ull << g.hiq[i];
            offhi[h] = off;
        }
    }
    __syncthreads();
    // base index of a tile: the tile number spread over the qubits outside Q
    auto tile_base = [&](uint64_t tile) {
        uint64_t base = tile << g.lowc;
#pragma unroll
        for (int i = 0; i < 24; ++i)
            if (i < g.nhi) base = ins0(base, g.hiq[i]);
        return base;
    };
    // The first group's layout is the same for every tile. A staged first
    // group loads local indices t + j*blockDim (coalesced) and transposes
    // through shared memory; otherwise each thread loads its own subcube.
    uint32_t first_l0 = threadIdx.x;
    int first_b[SUB];
    if constexpr (PF) {
        const uint64_t packed = ops[0].gtgt;
#pragma unroll
        for (int j = 0; j < SUB; ++j) first_b[j] = (int)((packed >> (8 * j)) & 0xff);
#pragma unroll
        for (int j = 0; j < SUB; ++j) first_l0 = (uint32_t)ins0(first_l0, first_b[j]);
    }
    auto load_first = [&](uint64_t tb, T(&dst)[E]) {
#pragma unroll
        for (int r = 0; r < E; ++r) {
            uint32_t l = threadIdx.x + (uint32_t)r * blockDim.x;
            if (!(g.stage & 1)) {
                l = first_l0;
#pragma unroll
                for (int j = 0; j < SUB; ++j) l |= ((r >> j) & 1) ? (1u << first_b[j]) : 0u;
            }
            dst[r] = ld_amp(psi + (tb | offhi[l >> g.lowc] | (l & lowm)));
        }
    };
    T nx[E];  // PF: the next tile's first-group amplitudes, in flight (unused otherwise)
    if constexpr (PF) {
        const TileRange r0 = tile_range(g);
        if (r0.first < r0.end) load_first(tile_base(r0.first), nx);
    }
    const TileRange tr = tile_range(g);
    for (uint64_t tile = tr.first; tile < tr.end; tile += tr.step) {
        const uint64_t base = tile_base(tile);
        int rec = 0;
        trc.begin(g, tile);
        for (int gi = 0; gi < g.ngroups; ++gi) {
            const int nops = ops[rec].tbit;
            const uint64_t packed = ops[rec].gtgt;
            // global offsets of the group's bits (the planner's group header):
            // amplitude r of the subcube sits at base | dep(l0) | OR_j r_j gdep[j],
            // so an address needs one shared-memory lookup per group, not one per
            // amplitude (those LDS fed every global load and store address)
            const uint64_t *gdep = reinterpret_cast<const uint64_t *>(ops[rec].u);
            ++rec;
            int b[SUB];
#pragma unroll
            for (int j = 0; j < SUB; ++j) b[j] = (int)((packed >> (8 * j)) & 0xff);
            // this thread's subcube: local indices l0 | sum_j {0, 2^b_j}
            uint32_t l0 = threadIdx.x;
#pragma unroll
            for (int j = 0; j < SUB; ++j) l0 = (uint32_t)ins0(l0, b[j]);
            auto lidx = [&](int r) {
                uint32_t l = l0;
#pragma unroll
                for (int j = 0; j < SUB; ++j) l |= ((r >> j) & 1) ? (1u << b[j]) : 0u;
                return l;
            };
            // Shared slot of subcube amplitude r: swz is XOR-linear and l0 has
            // zeros at the group's bits, so swz(lidx(r)) = swz(l0) ^ XOR_j r_j
            // swz(2^b_j): one XOR per slot. s0 / sb are computed right before
            // each use (slots()), never kept live across the op loop.
            uint32_t s0, sb[SUB];
            auto slots = [&]() {
                s0 = swz(l0);
#pragma unroll
                for (int j = 0; j < SUB; ++j) sb[j] = swz(1u << b[j]);
            };
            auto sidx = [&](int r) {
                uint32_t x = s0;
#pragma unroll
                for (int j = 0; j < SUB; ++j) x ^= ((r >> j) & 1) ? sb[j] : 0u;
                return x;
            };
            // complex128 (FP64-issue bound) takes the offsets; complex64 (ALU-issue
            // bound) measured faster with the per-amplitude lookups (64-bit ORs
            // cost it more than the LDS latency): C3 c64 525 vs 597 ms
            // (loads only: dl0 is computed right before them and is dead after;
            // the last group's stores keep the per-amplitude lookups, which
            // measured no slower and need no register live across the op loop,
            // where the extra two spilled up to 780 bytes in some class sets)
            constexpr bool kDep = sizeof(R) == 8;
            auto dep_l0 = [&]() { return kDep ? base | offhi[l0 >> g.lowc] | (l0 & lowm) : 0; };
            auto gaddr = [&](uint64_t dl0, int r) {  // global index of subcube amplitude r
                if constexpr (kDep) {
                    uint64_t a = dl0;
#pragma unroll
                    for (int j = 0; j < SUB; ++j)
                        if ((r >> j) & 1) a |= gdep[j];
                    return a;
                } else {
                    const uint32_t lr = lidx(r);
                    return base | offhi[lr >> g.lowc] | (lr & lowm);
                }
            };
            // staged (coalesced) layout: index t + j*blockDim = t | j << (k - sub)
            const uint32_t t = threadIdx.x;
            auto saddr = [&](uint64_t dt, int j) {
                if constexpr (kDep) {
                    uint64_t a = dt;
#pragma unroll
                    for (int i = 0; i < SUB; ++i)
                        if ((j >> i) & 1) a |= g.sdep[i];
                    return a;
                } else {
                    const uint32_t l = t + (uint32_t)j * blockDim.x;
                    return base | offhi[l >> g.lowc] | (l & lowm);
                }
            };
            T v[E];
            if (PF && gi == 0) {
#pragma unroll
                for (int r = 0; r < E; ++r) v[r] = nx[r];
                if (tile + tr.step < tr.end) load_first(tile_base(tile + tr.step), nx);
                if (g.stage & 1) {  // v holds coalesced amplitudes: transpose to the group layout
#pragma unroll
                    for (int j = 0; j < E; ++j) sm[swz(threadIdx.x + (uint32_t)j * blockDim.x)] = v[j];
                    __syncthreads();
                    slots();
#pragma unroll
                    for (int r = 0; r < E; ++r) v[r] = sm[sidx(r)];
                }
            } else if (gi == 0 && (g.stage & 1)) {
                // the group's bits include the lowest tile bits, so its lanes
                // would stride through HBM: load the tile coalesced (lane =
                // consecutive amplitudes) into shared memory first
                const uint64_t dt = kDep ? base | offhi[t >> g.lowc] | (t & lowm) : 0;
#pragma unroll
                for (int j = 0; j < E; ++j) v[j] = ld_amp(psi + saddr(dt, j));  // all loads in flight first
#pragma unroll
                for (int j = 0; j < E; ++j) sm[swz(threadIdx.x + (uint32_t)j * blockDim.x)] = v[j];
                __syncthreads();
                slots();
#pragma unroll
                for (int r = 0; r < E; ++r) v[r] = sm[sidx(r)];
            } else if (gi == 0) {
                const uint64_t dl0 = dep_l0();
#pragma unroll
                for (int r = 0; r < E; ++r) v[r] = ld_amp(psi + gaddr(dl0, r));
            } else {
                slots();
#pragma unroll
                for (int r = 0; r < E; ++r) v[r] = sm[sidx(r)];
            }
            trc.mark_after(6 + 3 * gi, v[0].x, v[E - 1].y);
            Ops::template apply<R, SUB, FMA, CM>(gi, v, base, ops, rec, nops);
            rec += nops;
            trc.mark_after(7 + 3 * gi, v[0].x, v[E - 1].y);
            if (gi == g.ngroups - 1 && (g.stage & 2)) {
                // each thread rewrites only the slots it read, then the tile
                // leaves coalesced
                asm volatile("" : "+r"(l0));  // recompute the slots: nothing extra live across the op loop
                slots();
#pragma unroll
                for (int r = 0; r < E; ++r) sm[sidx(r)] = v[r];
                __syncthreads();
#pragma unroll
                for (int j = 0; j < E; ++j) v[j] = sm[swz(threadIdx.x + (uint32_t)j * blockDim.x)];
                const uint64_t dt = kDep ? base | offhi[t >> g.lowc] | (t & lowm) : 0;
#pragma unroll
                for (int j = 0; j < E; ++j) st_amp(psi + saddr(dt, j), v[j]);
            } else if (gi == g.ngroups - 1) {
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    const uint32_t lr = lidx(r);
                    st_amp(psi + (base | offhi[lr >> g.lowc] | (lr & lowm)), v[r]);
                }
            } else {
                asm volatile("" : "+r"(l0));
                slots();
#pragma unroll
                for (int r = 0; r < E; ++r) sm[sidx(r)] = v[r];
                __syncthreads();
            }
            trc.mark(8 + 3 * gi);
        }
        if (use_sm) __syncthreads();  // sm was read this tile; the next tile writes it
        trc.end(g.ngroups);
    }
}

template <class R, int SUB, bool FMA, int MAXT, bool PF, int CM>
__global__ void __launch_bounds__(MAXT, (tile_min_blocks<R, SUB, MAXT, PF>()))
k_tile(typename Cplx<R>::T *__restrict__ psi, const __grid_constant__ TileParams prm) {
    k_tile_body<R, SUB, FMA, MAXT, PF, CM, TileOpsRuntime>(psi, prm);
}

}  // namespace qvg
