// qvg_kernels.cuh — sm_100a gate-application kernels.
//
// Every kernel is an HBM-bound streaming read-modify-write over the amplitude
// array (0.44 flop/B for complex128), so the design targets bytes:
// 16-B vector accesses, enumeration of only the amplitudes a gate changes,
// and a fused tile pass that applies a run of gates per HBM round trip.
//
// Arithmetic parity (reference proj/src/kernel.cpp:14-19): the reference's
// apply_pair is `lo = u00*a + u01*b; hi = u10*a + u11*b` on std::complex<double>
// built at -O2 without -march, i.e. (ac-bd, ad+bc) per product and a plain add,
// no FMA. The complex128 kernels use __dmul_rn/__dsub_rn/__dadd_rn so nvcc
// cannot contract them, which makes the c128 results bit-identical to the
// reference. Complex64 (not in the reference) lets the compiler use FFMA.
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>
#else  // NVRTC (the JIT-specialised tile passes, qvg_jit.hpp): no system headers
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned char uint8_t;
#endif

namespace qvg {

template <class R> struct Cplx;
template <> struct Cplx<double> { using T = double2; };
template <> struct Cplx<float> { using T = float2; };

// Row-major 2x2 matrix as 8 reals: re00 im00 re01 im01 re10 im10 re11 im11.
template <class R> struct Mat { R u[8]; };

// (m0 * a) + (m1 * b), complex128, reference operation order, no contraction.
__device__ __forceinline__ double2 madd2(double m0r, double m0i, double2 a, double m1r,
                                         double m1i, double2 b) {
    const double re = __dadd_rn(__dsub_rn(__dmul_rn(m0r, a.x), __dmul_rn(m0i, a.y)),
                                __dsub_rn(__dmul_rn(m1r, b.x), __dmul_rn(m1i, b.y)));
    const double im = __dadd_rn(__dadd_rn(__dmul_rn(m0r, a.y), __dmul_rn(m0i, a.x)),
                                __dadd_rn(__dmul_rn(m1r, b.y), __dmul_rn(m1i, b.x)));
    return make_double2(re, im);
}
__device__ __forceinline__ float2 madd2(float m0r, float m0i, float2 a, float m1r, float m1i,
                                        float2 b) {
    return make_float2(m0r * a.x - m0i * a.y + (m1r * b.x - m1i * b.y),
                       m0r * a.y + m0i * a.x + (m1r * b.y + m1i * b.x));
}
// d * a. For a diagonal gate the reference computes (0*a) + (d*b); adding the
// +-0 product leaves d*b unchanged (up to the sign of an exact zero), so this
// is value-identical to the reference.
__device__ __forceinline__ double2 cmul(double dr, double di, double2 a) {
    return make_double2(__dsub_rn(__dmul_rn(dr, a.x), __dmul_rn(di, a.y)),
                        __dadd_rn(__dmul_rn(dr, a.y), __dmul_rn(di, a.x)));
}
__device__ __forceinline__ float2 cmul(float dr, float di, float2 a) {
    return make_float2(dr * a.x - di * a.y, dr * a.y + di * a.x);
}

// Opt-in fast variants for complex128 (QVG_OPT_FMA): DFMA-contracted, 8
// instead of 14 FP64 instructions per output, within ~1e-16 relative of the
// exact forms but no longer bit-identical to the reference. complex64 always
// contracts, so both variants are the same there.
template <bool FMA>
__device__ __forceinline__ double2 madd2x(double m0r, double m0i, double2 a, double m1r, double m1i, double2 b) {
    if constexpr (!FMA) return madd2(m0r, m0i, a, m1r, m1i, b);
    const double re = fma(m0r, a.x, fma(-m0i, a.y, fma(m1r, b.x, -(m1i * b.y))));
    const double im = fma(m0r, a.y, fma(m0i, a.x, fma(m1r, b.y, m1i * b.x)));
    return make_double2(re, im);
}
template <bool FMA>
__device__ __forceinline__ float2 madd2x(float m0r, float m0i, float2 a, float m1r, float m1i, float2 b) {
    return madd2(m0r, m0i, a, m1r, m1i, b);
}
template <bool FMA>
__device__ __forceinline__ double2 cmulx(double dr, double di, double2 a) {
    if constexpr (!FMA) return cmul(dr, di, a);
    return make_double2(fma(dr, a.x, -(di * a.y)), fma(dr, a.y, di * a.x));
}
template <bool FMA>
__device__ __forceinline__ float2 cmulx(float dr, float di, float2 a) {
    return cmul(dr, di, a);
}

// Streaming loads/stores: every amplitude is touched once per pass, so mark
// the lines evict-first in L2 (ld.global.cs / st.global.cs).
// (Plain-cached loads/stores measured the same at n = 16..30, also for states
// that fit in L2.)
__device__ __forceinline__ double2 ld_amp(const double2 *p) { return __ldcs(p); }
__device__ __forceinline__ float2 ld_amp(const float2 *p) { return __ldcs(p); }
__device__ __forceinline__ void st_amp(double2 *p, double2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_amp(float2 *p, float2 v) { __stcs(p, v); }

__device__ __forceinline__ double shfl_x(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ float shfl_x(float v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

// Insert a 0 bit at position b (b < 64): the pair-base enumeration of
// reference kernel.cpp:72-73 without the nested loop.
__device__ __forceinline__ uint64_t ins0(uint64_t x, int b) {
    const uint64_t low = (1ull << b) - 1ull;
    return ((x & ~low) << 1) | (x & low);
}

// ---------------------------------------------------------------------------
// K1: pairs kernel, any target. Enumerates pair bases with a 0 inserted at the
// target bit and, for a controlled op, the control bit inserted as 1 — so a
// controlled gate touches only the 2^(n-1) amplitudes whose control bit is 1
// (the reference streams all of them, kernel.cpp:74-76). ins_lo < ins_hi are
// the inserted positions (ins_hi = -1 when only the target is inserted); setm
// is the mask of inserted bits that are 1 (the control).
// When the control-1 runs would be shorter than a 32-B sector (control bit 0
// in c128) inserting it saves no DRAM sectors but halves the lanes' access
// efficiency, so that control is instead a select (c_pred): every pair is
// read and written, control=0 pairs unchanged (the dense pass's bytes, which
// the sector-rounded algorithmic count charges anyway).
// Each thread owns PPT pairs, strided by blockDim so every load instruction of
// a warp covers consecutive bases.
template <class R, int PPT>
__global__ void __launch_bounds__(256)
k_pairs(typename Cplx<R>::T *__restrict__ psi, int q, int ins_lo, int ins_hi, uint64_t setm, int c_pred,
        int pred_store, Mat<R> m) {
    using T = typename Cplx<R>::T;
    const uint64_t qb = 1ull << q;
    const uint64_t first = (uint64_t)blockIdx.x * (blockDim.x * PPT) + threadIdx.x;
    uint64_t lo[PPT];
    T a[PPT], b[PPT];
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        uint64_t x = ins0(first + (uint64_t)k * blockDim.x, ins_lo);
        if (ins_hi >= 0) x = ins0(x, ins_hi);
        lo[k] = x | setm;
        a[k] = ld_amp(psi + lo[k]);
        b[k] = ld_amp(psi + (lo[k] | qb));
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        const bool on = c_pred < 0 || ((lo[k] >> c_pred) & 1ull);
        // control=0 pairs are written back unchanged (whole-sector stores
        // measured faster than 16-B masked ones, profiles/r01_*) unless
        // pred_store asks to skip them.
        if (!on && pred_store) continue;
        st_amp(psi + lo[k], on ? madd2(m.u[0], m.u[1], a[k], m.u[2], m.u[3], b[k]) : a[k]);
        st_amp(psi + (lo[k] | qb), on ? madd2(m.u[4], m.u[5], a[k], m.u[6], m.u[7], b[k]) : b[k]);
    }
}

// ---------------------------------------------------------------------------
// K2: low-target kernel (target < 5). A warp loads 32 consecutive enumerated
// amplitudes (512 B c128 when uncontrolled, one 16-B access per lane) and
// finds each partner with __shfl_xor(lane ^ qm). Each lane writes its own
// amplitude with the reference expression for its role (lo or hi).
// A control is inserted into the enumeration as a 1 bit (c_ins, any position
// whose control-1 runs fill whole sectors), so every lane is active and only
// control=1 amplitudes are read; qm is the partner's lane distance in the
// enumeration (2^q, or 2^(q-1) when c_ins < q). A control whose runs are
// shorter than a sector is a select instead (c_pred; control=0 amplitudes
// are written back unchanged).
template <class R, int APT>
__global__ void __launch_bounds__(256)
k_low(typename Cplx<R>::T *__restrict__ psi, int q, int qm, int c_ins, int c_pred, Mat<R> m) {
    using T = typename Cplx<R>::T;
    const uint64_t first = (uint64_t)blockIdx.x * (blockDim.x * APT) + threadIdx.x;
    uint64_t j[APT];
    T v[APT];
#pragma unroll
    for (int k = 0; k < APT; ++k) {
        uint64_t x = first + (uint64_t)k * blockDim.x;
        if (c_ins >= 0) x = ins0(x, c_ins) | (1ull << c_ins);
        j[k] = x;
        v[k] = ld_amp(psi + x);
    }
#pragma unroll
    for (int k = 0; k < APT; ++k) {
        T p;
        p.x = shfl_x(v[k].x, qm);
        p.y = shfl_x(v[k].y, qm);
        const bool hi = (j[k] >> q) & 1ull;
        const T out = hi ? madd2(m.u[4], m.u[5], p, m.u[6], m.u[7], v[k])
                         : madd2(m.u[0], m.u[1], v[k], m.u[2], m.u[3], p);
        st_amp(psi + j[k], (c_pred < 0 || ((j[k] >> c_pred) & 1ull)) ? out : v[k]);
    }
}

// ---------------------------------------------------------------------------
// K3: phase kernel for gates diag(1, d) with optional control (Z, S, T, CZ,
// CP/R_k): only amplitudes whose target (and control) bits are all 1 change,
// a quarter of the state for CZ/CP and half for Z/S/T. Forced-1 bits whose
// runs fill whole DRAM granules are inserted into the enumeration (ins_lo <
// ins_hi, -1 = unused; setm = their mask); the others (selm) select per
// amplitude, with unselected amplitudes written back unchanged (or not
// stored when pred_store).
template <class R, int APT>
__global__ void __launch_bounds__(256)
k_phase(typename Cplx<R>::T *__restrict__ psi, int ins_lo, int ins_hi, uint64_t setm, uint64_t selm,
        int pred_store, R dr, R di) {
    const uint64_t first = (uint64_t)blockIdx.x * (blockDim.x * APT) + threadIdx.x;
    uint64_t j[APT];
    typename Cplx<R>::T v[APT];
#pragma unroll
    for (int k = 0; k < APT; ++k) {
        uint64_t x = first + (uint64_t)k * blockDim.x;
        if (ins_lo >= 0) x = ins0(x, ins_lo);
        if (ins_hi >= 0) x = ins0(x, ins_hi);
        j[k] = x | setm;
        v[k] = ld_amp(psi + j[k]);
    }
#pragma unroll
    for (int k = 0; k < APT; ++k) {
        const bool on = (j[k] & selm) == selm;
        if (on) st_amp(psi + j[k], cmul(dr, di, v[k]));
        else if (!pred_store) st_amp(psi + j[k], v[k]);
    }
}
// ---------------------------------------------------------------------------
// K5: swap two local qubits a < b in place (pure permutation: amplitudes with
// bits (a,b) = (1,0) trade places with (0,1)). Used to restore the canonical
// qubit order of a sharded state and to move a qubit onto the exchange bit.
template <class R, int APT>
__global__ void __launch_bounds__(256)
k_swap_bits(typename Cplx<R>::T *__restrict__ psi, int a, int b) {
    using T = typename Cplx<R>::T;
    const uint64_t first = (uint64_t)blockIdx.x * (blockDim.x * APT) + threadIdx.x;
    uint64_t i0[APT];
    T x[APT], y[APT];
#pragma unroll
    for (int k = 0; k < APT; ++k) {
        const uint64_t base = ins0(ins0(first + (uint64_t)k * blockDim.x, a), b);
        i0[k] = base;
        x[k] = ld_amp(psi + (base | (1ull << a)));
        y[k] = ld_amp(psi + (base | (1ull << b)));
    }
#pragma unroll
    for (int k = 0; k < APT; ++k) {
        st_amp(psi + (i0[k] | (1ull << a)), y[k]);
        st_amp(psi + (i0[k] | (1ull << b)), x[k]);
    }
}

// K7: half-shard exchange over peer memory, optionally fused with the gate
// that triggered it. Shard a has gpos bit 0 and shard b has gpos bit 1. t
// enumerates local indices x0 whose bit lpos is 0, with x1 = x0 | 2^lpos.
//
// After the exchange:
//   * a holds (a[x0], b[x0]) at (x0, x1);
//   * b holds (a[x1], b[x1]) at (x0, x1).
// The gate on the swapped-in qubit (now local bit lpos) pairs exactly those two
// amplitudes. So each t owns four amplitudes that no other t reads or writes.
// The t range can therefore be split between the two ranks (each rank streams
// one half, with half its bytes local and half over NVLink) with no
// synchronisation inside the kernel.
//
// Parameters:
//   * mode bit 0 / bit 1: apply the gate on a's / b's pairs (each rank's
//     predicate for a global control);
//   * cbit: a local control bit (-1 = none); a pair whose cbit is 0 is only
//     exchanged;
//   * mode 0: the pure exchange a[x1] <-> b[x0], touching only those halves;
//   * fence: the shards are on other GPUs; fence the stores system-wide
//     before the stream-ordered barrier that follows the kernel.
// The pair arithmetic is the reference formula (madd2), so a fused exchange
// is bit-identical to exchange-then-gate.
template <class R, int APT>
__global__ void __launch_bounds__(256)
k_xchg(typename Cplx<R>::T *a, typename Cplx<R>::T *b, int lpos, uint64_t t0, int cbit, int mode, int fence,
       Mat<R> m) {
    using T = typename Cplx<R>::T;
    const uint64_t first = t0 + (uint64_t)blockIdx.x * (blockDim.x * APT) + threadIdx.x;
    const uint64_t lb = 1ull << lpos;
    uint64_t x0[APT];
    if (mode == 0) {
        T u[APT], v[APT];
#pragma unroll
        for (int k = 0; k < APT; ++k) {
            x0[k] = ins0(first + (uint64_t)k * blockDim.x, lpos);
            u[k] = ld_amp(a + (x0[k] | lb));
            v[k] = ld_amp(b + x0[k]);
        }
#pragma unroll
        for (int k = 0; k < APT; ++k) {
            st_amp(a + (x0[k] | lb), v[k]);
            st_amp(b + x0[k], u[k]);
        }
    } else {
        T a0[APT], a1[APT], b0[APT], b1[APT];
#pragma unroll
        for (int k = 0; k < APT; ++k) {
            x0[k] = ins0(first + (uint64_t)k * blockDim.x, lpos);
            a0[k] = ld_amp(a + x0[k]);
            a1[k] = ld_amp(a + (x0[k] | lb));
            b0[k] = ld_amp(b + x0[k]);
            b1[k] = ld_amp(b + (x0[k] | lb));
        }
#pragma unroll
        for (int k = 0; k < APT; ++k) {
            const bool on = cbit < 0 || ((x0[k] >> cbit) & 1ull);
            const bool ga = on && (mode & 1), gb = on && (mode & 2);
            st_amp(a + x0[k], ga ? madd2(m.u[0], m.u[1], a0[k], m.u[2], m.u[3], b0[k]) : a0[k]);
            st_amp(a + (x0[k] | lb), ga ? madd2(m.u[4], m.u[5], a0[k], m.u[6], m.u[7], b0[k]) : b0[k]);
            st_amp(b + x0[k], gb ? madd2(m.u[0], m.u[1], a1[k], m.u[2], m.u[3], b1[k]) : a1[k]);
            st_amp(b + (x0[k] | lb), gb ? madd2(m.u[4], m.u[5], a1[k], m.u[6], m.u[7], b1[k]) : b1[k]);
        }
    }
    if (fence) __threadfence_system();
}

// K8: batched exchange of k global qubits over peer memory (STEP_MULTI_EXCHANGE
// in qvg_schedule.hpp).
//
// This rank's shard `self` has value w on the k swapped rank bits. Round t
// (1..2^k-1) pairs it with the rank whose bits read w^t (shard peer[t]): self's
// amplitudes whose local bits at the k positions read w^t trade places with the
// partner's that read w.
//
// Ownership: a (round, base) item is handled by one rank of its pair, the
// one with the lower value taking the first half of the bases. So all ranks
// run with no synchronisation inside the kernel. One grid row per round.
template <class R>
struct MxParams {
    typename Cplx<R>::T *self;
    typename Cplx<R>::T *peer[16];
    int k;
    int ps[4];     // the k local positions, ascending
    int perm[4];   // value bit carried by ps[j]
    uint32_t w;    // this rank's value on the swapped bits
    uint64_t half; // bases per round owned by one rank: 2^(L-k) / 2
    int fence;
};

template <class R>
__device__ __forceinline__ uint64_t mx_deposit(uint64_t b, const MxParams<R> &p, uint32_t v) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (j < p.k) b = ins0(b, p.ps[j]) | ((uint64_t)((v >> p.perm[j]) & 1u) << p.ps[j]);
    return b;
}

template <class R, int APT>
__global__ void __launch_bounds__(256) k_mxchg(const __grid_constant__ MxParams<R> p) {
    using T = typename Cplx<R>::T;
    const uint32_t t = blockIdx.y + 1;
    const uint32_t wp = p.w ^ t;
    T *peer = p.peer[t];
    const uint64_t first = (p.w < wp ? 0 : p.half) + (uint64_t)blockIdx.x * (blockDim.x * APT) + threadIdx.x;
    uint64_t xs[APT], xp[APT];
    T a[APT], b[APT];
#pragma unroll
    for (int i = 0; i < APT; ++i) {
        const uint64_t base = first + (uint64_t)i * blockDim.x;
        xs[i] = mx_deposit(base, p, wp);
        xp[i] = mx_deposit(base, p, p.w);
        a[i] = ld_amp(p.self + xs[i]);
        b[i] = ld_amp(peer + xp[i]);
    }
#pragma unroll
    for (int i = 0; i < APT; ++i) {
        st_amp(p.self + xs[i], b[i]);
        st_amp(peer + xp[i], a[i]);
    }
    if (p.fence) __threadfence_system();
}

// ---------------------------------------------------------------------------
// Readout.
// Per-block partial sums of |a|^2 with a fixed grid, so the result is
// deterministic run to run (the host sums the partials with Kahan, like
// BlockStore::norm, reference store.cpp:301-316).
template <class R>
__global__ void __launch_bounds__(256)
k_norm_partials(const typename Cplx<R>::T *__restrict__ psi, uint64_t count, double *__restrict__ partial) {
    __shared__ double red[256];
    double acc = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const typename Cplx<R>::T v = psi[i];
        const double x = (double)v.x, y = (double)v.y;
        acc += __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// |a_i|^2 = re*re + im*im (std::norm, reference engine.cpp:518).
template <class R>
__global__ void __launch_bounds__(256)
k_probs(const typename Cplx<R>::T *__restrict__ psi, uint64_t count, double *__restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const typename Cplx<R>::T v = psi[i];
        const double x = (double)v.x, y = (double)v.y;
        out[i] = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    }
}

}  // namespace qvg
