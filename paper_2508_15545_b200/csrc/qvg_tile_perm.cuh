// qvg_tile_perm.cuh — K4d, a fused pass of only permutations and +-1 phases
// (X, CX, the CXs of a SWAP, Z, CZ; PASS_PERM in qvg_plan.hpp).
//
// Such a run moves every amplitude of a tile to another slot of the same tile
// and at most flips its sign, so k_tile's register groups and their shared-
// memory transposes (three groups for the nine CXs of a config-2 pass) reduce
// to ONE scatter: each thread loads its amplitudes coalesced, follows each
// one's index through the run's ops in circuit order (integer work only),
// writes it to its final slot in shared memory, and after one barrier the tile
// leaves coalesced.
//
// Bits: k_tile moves a pair of a SWAP-class op through one DADD with +0 per
// component (mov_opaque: -0 becomes +0, nothing else changes) and flips signs
// for the NEG class. Per amplitude this kernel tracks, in op order, whether it
// was moved and the sign flips before and after its last move, then applies
// the same composition once: flips-before, one DADD +0 if moved, flips-after.
// The result equals k_tile's bit for bit (the DADD commutes with a negation
// except on zeros, which the split handles).
#pragma once

#include "qvg_tile.cuh"

namespace qvg {

// MAXT threads per CTA (2^k / E). The minimum-blocks hint: 16 complex128
// amplitudes in flight per thread plus their 16 indices need ~100 registers
// (4 CTAs of 128 threads per SM; at 5 ptxas spilled the indices); complex64
// fits 5 (128 threads) / 3 (256).
#ifndef QVG_PERM_C128_MINB
#define QVG_PERM_C128_MINB 4
#endif
template <class R, int E, int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT <= 128 ? (sizeof(R) == 8 && E == 16 ? QVG_PERM_C128_MINB : 5) : 3)
k_tile_perm(typename Cplx<R>::T *__restrict__ psi, const __grid_constant__ TileParams prm) {
    using T = typename Cplx<R>::T;
    const TileGeom &g = prm.g;
    const TileOp *ops = prm.ops;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t *offhi = reinterpret_cast<uint64_t *>(smem_raw);
    T *sm = reinterpret_cast<T *>(smem_raw + (((sizeof(uint64_t) << g.nhi) + 15) & ~15ull));
    const uint32_t nhi = 1u << g.nhi;
    const uint32_t lowm = (1u << g.lowc) - 1u;
    for (uint32_t h = threadIdx.x; h < nhi; h += blockDim.x) {
        uint64_t off = 0;
#pragma unroll
        for (int i = 0; i < 24; ++i)
            if (i < g.nhi && ((h >> i) & 1u)) off |= 1ull << g.hiq[i];
        offhi[h] = off;
    }
    __syncthreads();
    const uint32_t nt = blockDim.x;
    const uint32_t t = threadIdx.x;
    const TileRange tr = tile_range(g);
    for (uint64_t tile = tr.first; tile < tr.end; tile += tr.step) {
        uint64_t base = tile << g.lowc;
#pragma unroll
        for (int i = 0; i < 24; ++i)
            if (i < g.nhi) base = ins0(base, g.hiq[i]);
        T v[E];
#pragma unroll
        for (int j = 0; j < E; ++j) {  // coalesced: lanes on consecutive amplitudes
            const uint32_t l = t + (uint32_t)j * nt;
            v[j] = ld_amp(psi + (base | offhi[l >> g.lowc] | (l & lowm)));
        }
        uint32_t l[E];
#pragma unroll
        for (int j = 0; j < E; ++j) l[j] = t + (uint32_t)j * nt;
        uint32_t moved = 0, f1 = 0, f2 = 0;  // bit j: amplitude j moved / flips before / after its last move
        for (int i = 0; i < g.nrec; ++i) {
            const TileOp &o = ops[i];
            if ((base & o.greq) != o.greq) continue;  // control outside the tile is 0 (uniform)
            const int cb = o.cbit, tb = o.tbit;
            if (o.kind == TILE_PAIR) {  // X on tile bit tb, controlled by tile bit cb (or none)
                uint32_t cm = 0;
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    const uint32_t c = cb < 0 ? 1u : (l[j] >> cb) & 1u;
                    l[j] ^= c << tb;
                    cm |= c << j;
                }
                f1 ^= f2 & cm;
                f2 &= ~cm;
                moved |= cm;
            } else {  // sign flip where the target (and control) bits are 1
                const bool tg = tb < 0 && (base & o.gtgt) != 0;  // target outside the tile: per tile
                uint32_t fm = 0;
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    const uint32_t c = cb < 0 ? 1u : (l[j] >> cb) & 1u;
                    const uint32_t x = tb < 0 ? (tg ? 1u : 0u) : (l[j] >> tb) & 1u;
                    fm |= (c & x) << j;
                }
                f2 ^= fm;
            }
        }
#pragma unroll
        for (int j = 0; j < E; ++j) {
            T w = v[j];
            if ((moved >> j) & 1u) {
                if ((f1 >> j) & 1u) w = T{neg_rn(w.x), neg_rn(w.y)};
                w = mov_opaque(w);
            }
            if ((f2 >> j) & 1u) w = T{neg_rn(w.x), neg_rn(w.y)};
            sm[swz(l[j])] = w;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const uint32_t lo = t + (uint32_t)j * nt;
            st_amp(psi + (base | offhi[lo >> g.lowc] | (lo & lowm)), sm[swz(lo)]);
        }
        __syncthreads();  // the next tile's scatter overwrites sm
    }
}

}  // namespace qvg
