// qvg_readout.cuh — device-side readout reductions: inner
// product / fidelity and max |a_i - b_i| between two states, and the
// top-k amplitude selection of the reference's top_amplitudes
// (reference engine.cpp:511-544) as an exact radix select on the device, so
// a readout at n=30 moves kilobytes over PCIe instead of the 16 GiB state.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "qvg_kernels.cuh"

namespace qvg {

// Per-block partials of <a|b> = sum conj(a_i) b_i (fixed grid => deterministic).
template <class R>
__global__ void __launch_bounds__(256)
k_inner_partials(const typename Cplx<R>::T *__restrict__ a, const typename Cplx<R>::T *__restrict__ b,
                 uint64_t count, double *__restrict__ partial) {
    __shared__ double rr[256], ri[256];
    double sr = 0.0, si = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const typename Cplx<R>::T x = a[i], y = b[i];
        const double xr = x.x, xi = x.y, yr = y.x, yi = y.y;
        sr += xr * yr + xi * yi;
        si += xr * yi - xi * yr;
    }
    rr[threadIdx.x] = sr;
    ri[threadIdx.x] = si;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            rr[threadIdx.x] += rr[threadIdx.x + s];
            ri[threadIdx.x] += ri[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = rr[0];
        partial[2 * blockIdx.x + 1] = ri[0];
    }
}

// Per-block max_i |a_i - b_i| (std::abs of a complex difference = hypot,
// reference dense.cpp:174-183).
template <class R>
__global__ void __launch_bounds__(256)
k_maxdiff_partials(const typename Cplx<R>::T *__restrict__ a, const typename Cplx<R>::T *__restrict__ b,
                   uint64_t count, double *__restrict__ partial) {
    __shared__ double red[256];
    double m = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const typename Cplx<R>::T x = a[i], y = b[i];
        const double d = hypot((double)x.x - (double)y.x, (double)x.y - (double)y.y);
        m = d > m || d != d ? d : m;  // NaN propagates
    }
    red[threadIdx.x] = m;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const double o = red[threadIdx.x + s];
            if (o > red[threadIdx.x] || o != o) red[threadIdx.x] = o;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// ---- chunk checksums (qvg_checksums) ------------------------------------------
// Per chunk of C = 2^cbits amplitudes (global index order), two 64-bit sums
// mod 2^64 of mixed amplitude bit patterns:
//   w0 += mix(re_bits ^ i*K0) + mix(im_bits ^ (i*K1 + K2))
//   w1 += mix(re_bits ^ (i*K3 + K4)) + mix(im_bits ^ i*K5)
// (mix = splitmix64's finaliser; re/im bits of the stored precision,
// complex64 zero-extended). Integer sums are order-independent, so any grid
// gives the same words, and every bit of every amplitude, including the sign
// of a zero, reaches both. A size-independent property for full-size parity:
// G-invariance at n = 32/33 compares 2 x 64 bits per chunk on the device
// instead of hashing 64-128 GiB on the host (tests/test_gpu_fullsize.py;
// numpy restatement in tests/conftest.py).
__host__ __device__ __forceinline__ uint64_t ck_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
constexpr uint64_t kCkK0 = 0x9e3779b97f4a7c15ull, kCkK1 = 0xc2b2ae3d27d4eb4full, kCkK2 = 0x165667b19e3779f9ull,
                   kCkK3 = 0x27d4eb2f165667c5ull, kCkK4 = 0xd6e8feb86659fd93ull, kCkK5 = 0xff51afd7ed558ccdull;
__device__ __forceinline__ void ck_bits(double2 v, uint64_t &re, uint64_t &im) {
    re = (uint64_t)__double_as_longlong(v.x);
    im = (uint64_t)__double_as_longlong(v.y);
}
__device__ __forceinline__ void ck_bits(float2 v, uint64_t &re, uint64_t &im) {
    re = (uint64_t)(uint32_t)__float_as_int(v.x);
    im = (uint64_t)(uint32_t)__float_as_int(v.y);
}

// One block: 4096 consecutive amplitudes (inside one chunk, C >= 4096);
// its two partial words are added to out[2*chunk], out[2*chunk+1].
template <class R>
__global__ void __launch_bounds__(256)
k_checksum(const typename Cplx<R>::T *__restrict__ psi, uint64_t count, uint64_t base_index, int cbits,
           unsigned long long *__restrict__ out) {
    __shared__ unsigned long long r0[256], r1[256];
    const uint64_t start = (uint64_t)blockIdx.x * 4096;
    uint64_t w0 = 0, w1 = 0;
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
        const uint64_t li = start + (uint64_t)k * 256 + threadIdx.x;
        if (li >= count) break;
        uint64_t re, im;
        ck_bits(psi[li], re, im);
        const uint64_t i = base_index + li;
        w0 += ck_mix(re ^ (i * kCkK0)) + ck_mix(im ^ (i * kCkK1 + kCkK2));
        w1 += ck_mix(re ^ (i * kCkK3 + kCkK4)) + ck_mix(im ^ (i * kCkK5));
    }
    r0[threadIdx.x] = w0;
    r1[threadIdx.x] = w1;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            r0[threadIdx.x] += r0[threadIdx.x + s];
            r1[threadIdx.x] += r1[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const uint64_t c = (base_index + start) >> cbits;
        atomicAdd(out + 2 * c, r0[0]);
        atomicAdd(out + 2 * c + 1, r1[0]);
    }
}

// ---- top-k by exact radix select over the IEEE bits of |a|^2 ------------------
// For p >= 0 the bit pattern of p, read as uint64, orders like p. One digit of
// `width` bits (starting at bit `shift`) is histogrammed per pass among the
// keys whose higher bits equal `prefix`.
__device__ __forceinline__ uint64_t prob_key(double2 v) {
    return (uint64_t)__double_as_longlong(__dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)));
}
__device__ __forceinline__ uint64_t prob_key(float2 v) {
    const double x = v.x, y = v.y;
    return (uint64_t)__double_as_longlong(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
}

constexpr int kTopkBins = 2048;

template <class R>
__global__ void __launch_bounds__(256)
k_topk_hist(const typename Cplx<R>::T *__restrict__ psi, uint64_t count, uint64_t prefix, int shift, int width,
            unsigned long long *__restrict__ hist) {
    // per-block counts fit 32 bits (a block visits <= 2^33 / 4096 keys); the
    // global bins are 64-bit: a state of >= 2^32 amplitudes (n >= 32 on one
    // B200, or sharded) can put that many keys in one bin
    __shared__ unsigned int sh[kTopkBins];
    for (int i = threadIdx.x; i < kTopkBins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int top = shift + width;  // bits >= top must equal prefix
    const uint64_t dmask = (1ull << width) - 1ull;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t key = prob_key(psi[i]);
        if (top < 64 && (key >> top) != prefix) continue;
        atomicAdd(&sh[(key >> shift) & dmask], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kTopkBins; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

// Append every amplitude with key > tau (at most k of them by construction).
struct TopkEntry {
    uint64_t index;
    double re, im;
};

template <class R>
__global__ void __launch_bounds__(256)
k_topk_collect(const typename Cplx<R>::T *__restrict__ psi, uint64_t count, uint64_t base_index, uint64_t tau,
               TopkEntry *__restrict__ out, unsigned int *__restrict__ n_out, unsigned int cap) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const typename Cplx<R>::T v = psi[i];
        if (prob_key(v) <= tau) continue;
        const unsigned int slot = atomicAdd(n_out, 1u);
        if (slot < cap) out[slot] = TopkEntry{base_index + i, (double)v.x, (double)v.y};
    }
}

// Number of keys == tau in each contiguous chunk of `chunk` amplitudes (ties
// are resolved by ascending index on the host, within the first chunks).
template <class R>
__global__ void __launch_bounds__(256)
k_topk_tie_counts(const typename Cplx<R>::T *__restrict__ psi, uint64_t count, uint64_t chunk, uint64_t tau,
                  unsigned int *__restrict__ counts) {
    const uint64_t c = blockIdx.x;
    unsigned int n = 0;
    for (uint64_t i = c * chunk + threadIdx.x; i < min(count, (c + 1) * chunk); i += blockDim.x)
        n += prob_key(psi[i]) == tau;
    __shared__ unsigned int red[256];
    red[threadIdx.x] = n;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) counts[c] = red[0];
}

// flags[j] = 1 iff amplitude chunk_off + j has key == tau: the tie test stays
// on the device (the host never recomputes |a|^2, whose rounding could differ
// under FMA contraction on another host ISA).
template <class R>
__global__ void __launch_bounds__(256)
k_topk_tie_flags(const typename Cplx<R>::T *__restrict__ psi, uint64_t chunk_off, uint64_t len, uint64_t tau,
                 unsigned char *__restrict__ flags) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < len; j += (uint64_t)gridDim.x * blockDim.x)
        flags[j] = prob_key(psi[chunk_off + j]) == tau;
}

}  // namespace qvg
